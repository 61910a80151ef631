# Builds the sm_100a C-ABI library in-tree (travels to the GPU box with the snapshot)
# and the CPU oracle (test infrastructure).
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH ?= -gencode arch=compute_100a,code=sm_100a
NVFLAGS ?= -O3 -std=c++17 -lineinfo $(ARCH) -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr
PKG := paper_2005_12648_b200
SRC := $(PKG)/csrc/pm_engine.cu $(PKG)/csrc/pm_flow.cu $(PKG)/csrc/pm_plan.cu $(PKG)/csrc/pm_rotate.cu $(PKG)/csrc/pm_wide.cu $(PKG)/csrc/pm_small.cu $(PKG)/csrc/pm_peers.cu $(PKG)/csrc/pm_capi.cu
HDR := $(wildcard $(PKG)/csrc/*.cuh) $(PKG)/csrc/pm_launch.h $(PKG)/csrc/pm_hostcache.h include/parmerge_b200.h
OBJ := $(SRC:.cu=.o)
LIB := $(PKG)/libparmerge_b200.so

all: $(LIB) oracle

$(PKG)/csrc/%.o: $(PKG)/csrc/%.cu $(HDR)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcudart

oracle:
	$(MAKE) -s -C oracle

ptxas: $(SRC)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $(PKG)/csrc/pm_engine.cu -o /tmp/pm_engine_v.o

clean:
	rm -f $(OBJ) $(LIB)
	$(MAKE) -s -C oracle clean

.PHONY: all oracle clean ptxas variant

# tuning variant: make variant VNAME=t2 VFLAGS="-DPM_ENGINE_TEAM=2 -DPM_ENGINE_MINB=6 -DPM_TILE_BUDGET=36864"
variant:
	mkdir -p /tmp/pmv_$(VNAME)
	for f in $(SRC); do $(NVCC) $(NVFLAGS) $(VFLAGS) -c $$f -o /tmp/pmv_$(VNAME)/$$(basename $$f .cu).o & done; wait
	$(NVCC) $(ARCH) -shared -o $(PKG)/libparmerge_b200_$(VNAME).so /tmp/pmv_$(VNAME)/*.o -lcudart
