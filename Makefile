# libdma: the B200-native (sm_100a) DMA forward path, built in-tree.
NVCC ?= /usr/local/cuda/bin/nvcc
PKG := paper_2604_03950_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
HDR := $(wildcard $(PKG)/csrc/*.cuh) $(PKG)/csrc/launch.h include/dma.h
OBJ := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRC))
LIB := $(PKG)/libdma.so

NVFLAGS := -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
           -Xcompiler -fPIC --expt-relaxed-constexpr \
           -Xptxas -v -Iinclude

all: $(LIB)

build/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJ)
	$(NVCC) -gencode arch=compute_100a,code=sm_100a -shared -o $@ $(OBJ)

clean:
	rm -rf build $(LIB)

.PHONY: all clean
