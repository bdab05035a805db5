# Builds every native artefact in-tree (they travel to the GPU box with gpurun).
NVCC      ?= nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NCCL_INC  := $(shell python -c "import os,nvidia.nccl as m; print(os.path.join(list(m.__path__)[0],'include'))" 2>/dev/null)
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -Iinclude -I$(NCCL_INC) --expt-relaxed-constexpr $(KDB_NVFLAGS)

KDB_SO    := paper_2009_04552_b200/lib/libkdb.so
KDB_DBG   := paper_2009_04552_b200/lib/libkdb_dbg.so
KNNG_SO   := paper_2009_04552_b200/lib/libknng.so
ORACLE_SO := oracle/liboracle.so

all: $(KDB_SO) $(KDB_DBG) $(ORACLE_SO) $(KNNG_SO)

$(KDB_SO): paper_2009_04552_b200/csrc/kdb.cu $(wildcard paper_2009_04552_b200/csrc/kdb_*.cuh) include/kdb.h
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -o $@ $< -ldl

# debug build: workspace guard bands + device bounds checks (tests/test_gpu_debug.py)
$(KDB_DBG): paper_2009_04552_b200/csrc/kdb.cu $(wildcard paper_2009_04552_b200/csrc/kdb_*.cuh) include/kdb.h
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -DKDB_GUARDS=1 -o $@ $< -ldl

# A/B build: light ELL in planes (tools/ scripts load it with KDB_LIBRARY)
paper_2009_04552_b200/lib/libkdb_ellplanes.so: paper_2009_04552_b200/csrc/kdb.cu $(wildcard paper_2009_04552_b200/csrc/kdb_*.cuh) include/kdb.h
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -DKDB_ELL_PLANES=1 -o $@ $< -ldl

# A/B builds: slim light-round hot loop (KDB_SLIM = 1, 2, 3: see kdb_rows.cuh)
paper_2009_04552_b200/lib/libkdb_slim%.so: paper_2009_04552_b200/csrc/kdb.cu $(wildcard paper_2009_04552_b200/csrc/kdb_*.cuh) include/kdb.h
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -DKDB_SLIM=$* -o $@ $< -ldl

$(KNNG_SO): paper_2009_04552_b200/csrc/knng.cu include/knng.h
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -Iinclude -o $@ $<

$(ORACLE_SO): oracle/kdb_oracle.cpp
	g++ -O2 -std=c++17 -shared -fPIC -o $@ $<

clean:
	rm -f $(KDB_SO) $(KDB_DBG) $(KNNG_SO) $(ORACLE_SO)

.PHONY: all clean
