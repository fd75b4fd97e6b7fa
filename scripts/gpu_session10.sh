export SB_SYNC_TIMEOUT_S=120 PYTHONUNBUFFERED=1
timeout 900 python -u scripts/sweep.py > gpurun_out/sweeps.json 2> gpurun_out/sweeps.log; echo sweep rc=$?; cat gpurun_out/sweeps.log | grep -v generated
for tool in memcheck racecheck synccheck; do
timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 python -u -c "
import sys; sys.path.insert(0,'.')
import numpy as np
from paper_2604_08374_b200 import CompressedCsr, HyperBall
g = CompressedCsr.synth_grid(24, 24, 6, 2, 5, 7, 0)
for p, kw in ((10, {}), (10, {'skip_unchanged': True}), (10, {'interval': True}), (6, {}), (12, {})):
    h = HyperBall(g, p, None, **kw); h.run(); h.registers()
    s = [HyperBall(g, p, None, node_range=r) for r in ((0, g.n//2), (g.n//2, g.n))]
    while True:
        mx = max(x.step_compute() for x in s); HyperBall.exchange_local(s)
        if s[0].step_finish(mx)[1] | s[1].step_finish(mx)[1]: break
print('ok')
" > gpurun_out/sanitizer_$tool.log 2>&1; echo sanitizer $tool rc=$?; tail -3 gpurun_out/sanitizer_$tool.log
done
