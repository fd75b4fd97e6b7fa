# Builds the product library (sm_100a CUDA + host C++) in-tree, plus the
# parity checker under oracle/ (test infrastructure).
NVCC     ?= nvcc
CXX      ?= g++
ARCH     := -gencode arch=compute_100a,code=sm_100a
PKG      := paper_2604_08374_b200
CSRC     := $(PKG)/csrc
BUILD    := build
CUDA_INC := $(dir $(shell which $(NVCC)))../include
NVEXTRA  ?=
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --fmad=false $(NVEXTRA)
CXXFLAGS := -O3 -std=c++17 -fPIC -Wall -ffp-contract=off -I$(CUDA_INC)
LIB      := $(PKG)/libsieveball_cuda.so
TOOL     := tools/sb_hyperball

OBJS := $(BUILD)/sb_kernels.o $(BUILD)/sb_local.o $(BUILD)/sb_vis.o $(BUILD)/sb_graph_api.o $(BUILD)/sb_hb_api.o $(BUILD)/sb_exact_api.o $(BUILD)/sb_csr.o $(BUILD)/sb_error.o
HDRS := $(CSRC)/sb_device.cuh $(CSRC)/sb_internal.h $(CSRC)/sb_error.h $(CSRC)/sb_handles.h include/sieveball_cuda.h

all: $(LIB) $(TOOL) oracle

$(BUILD):
	mkdir -p $(BUILD)

$(BUILD)/sb_kernels.o: $(CSRC)/sb_kernels.cu $(HDRS) | $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(BUILD)/ptxas_kernels.txt || (cat $(BUILD)/ptxas_kernels.txt; false)

$(BUILD)/sb_local.o: $(CSRC)/sb_local.cu $(HDRS) | $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(BUILD)/ptxas_local.txt || (cat $(BUILD)/ptxas_local.txt; false)

$(BUILD)/sb_vis.o: $(CSRC)/sb_vis.cu $(HDRS) | $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(BUILD)/ptxas_vis.txt || (cat $(BUILD)/ptxas_vis.txt; false)

$(BUILD)/%_api.o: $(CSRC)/%_api.cu $(HDRS) | $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(BUILD)/ptxas_$*_api.txt || (cat $(BUILD)/ptxas_$*_api.txt; false)

$(BUILD)/sb_csr.o: $(CSRC)/sb_csr.cpp $(HDRS) | $(BUILD)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(BUILD)/sb_error.o: $(CSRC)/sb_error.cpp $(CSRC)/sb_error.h | $(BUILD)
	$(CXX) $(CXXFLAGS) -c $< -o $@

# cudart is linked statically (nvcc default); NCCL and zlib from the system.
$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lnccl -lz -lpthread

$(TOOL): tools/sb_hyperball.cpp include/sieveball/hyperball_cuda.hpp $(LIB)
	$(CXX) -O2 -std=c++17 -Wall -Iinclude -o $@ $< -L$(PKG) -lsieveball_cuda -Wl,-rpath,'$$ORIGIN/../$(PKG)'

oracle:
	$(MAKE) -s -C oracle

# Instrumented build for scripts/group_stats.py (per-phase cycles of the group
# path); loaded with SB_LIBRARY=$(STATS_LIB), never by default.
STATS_LIB := $(PKG)/libsieveball_cuda_stats.so
stats: $(STATS_LIB)
$(BUILD)/sb_kernels_stats.o: $(CSRC)/sb_kernels.cu $(HDRS) | $(BUILD)
	$(NVCC) $(NVFLAGS) -DSB_GROUP_STATS -c $< -o $@ 2> $(BUILD)/ptxas_kernels_stats.txt || (cat $(BUILD)/ptxas_kernels_stats.txt; false)
$(STATS_LIB): $(BUILD)/sb_kernels_stats.o $(filter-out $(BUILD)/sb_kernels.o,$(OBJS))
	$(NVCC) $(ARCH) -shared -o $@ $^ -lnccl -lz -lpthread

clean:
	rm -rf $(BUILD) $(LIB) $(TOOL) $(STATS_LIB)
	$(MAKE) -C oracle clean

.PHONY: all oracle clean stats
