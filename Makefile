# Builds the sm_100a C-ABI library in-tree (travels to the GPU box with the snapshot)
# and the CPU oracle (test infrastructure).
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH ?= -gencode arch=compute_100a,code=sm_100a
NVFLAGS ?= -O3 -std=c++17 -lineinfo $(ARCH) -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr
PKG := paper_2005_12648_b200
SRC := $(PKG)/csrc/pm_engine.cu $(PKG)/csrc/pm_plan.cu $(PKG)/csrc/pm_capi.cu
HDR := $(wildcard $(PKG)/csrc/*.cuh) $(PKG)/csrc/pm_launch.h include/parmerge_b200.h
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

.PHONY: all oracle clean ptxas
