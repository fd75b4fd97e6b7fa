"""Dependency floor of the wavefront first run at C3.

Model: the stream arrives at a constant PCIe rate over U ms, in K chunks (a
1/64 first chunk, then K-1 equal ones); pass p of chunk k may run once chunk
k has landed (p = 1) or once pass p-1 is done on every chunk up to the one
holding node end_k + r (rows reach r nodes forward; the reach backwards is
always satisfied first); the GPU runs one chunk-pass at a time, lowest pass
first, C ms per pass over the whole graph, plus a fixed cost per launch.
C3: 486 x 486 row-major grid, visibility radius 87 rows -> r = 87*486/N
= 0.18 N.  Prints the modelled end of the run for several chunk counts, for
the dense union (C = 19.6 ms) and the interval variant (C = 2.94 ms incl.
the sparse tables), against the measured 0.219 / 0.111 s (runs after the
first, `profiles/r02/e2e_breakdown.txt`).  No GPU needed.
"""
import json


def model(K, r, U, C, passes=9, first=1 / 64, launch_ms=0.01):
    b = [0.0, first] + [first + (1 - first) * k / (K - 1) for k in range(1, K)]
    b = b[:K + 1]
    b[-1] = 1.0
    arrive = [U * b[k + 1] for k in range(K)]

    def chunk_of(x):
        x = min(max(x, 0.0), 1 - 1e-12)
        return next(k for k in range(K) if b[k] <= x < b[k + 1])

    reach = [chunk_of(b[k + 1] + r) for k in range(K)]
    done, nxt, t = {}, [0] * (passes + 1), 0.0
    while True:
        cand = []
        for p in range(1, passes + 1):
            k = nxt[p]
            if k >= K:
                continue
            if p == 1:
                cand.append((max(t, arrive[k]), p, k))
            elif nxt[p - 1] > reach[k]:
                cand.append((max(t, done[(p - 1, reach[k])], done[(p - 1, k)]), p, k))
        if not cand:
            return t
        st, p, k = min(cand)
        t = st + C * (b[k + 1] - b[k]) + launch_ms
        done[(p, k)] = t
        nxt[p] += 1


if __name__ == "__main__":
    r = 87 * 486 / (486 * 486)
    out = {"reach_fraction": round(r, 4), "upload_ms": 95.0}
    for name, C, meas in (("dense", 19.6, 219), ("interval", 2.94, 111)):
        out[name] = {"measured_run_ms": meas, "pass_ms": C,
                     "model_ms_by_chunks": {K: round(model(K, r, 95.0, C), 1) for K in (16, 24, 32, 48, 64)},
                     "no_dependency_floor_ms": round(max(95.0, 9 * C), 1)}
    print(json.dumps(out, indent=1))
