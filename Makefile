# Builds the C-ABI shared library for sm_100a (B200) in-tree.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude --cudart static \
           -Xptxas -v,-warn-spills
PKG := paper_2503_09203_b200
LIB := $(PKG)/libuuvb200.so
SRC := $(PKG)/csrc/uuv_b200.cu
HDR := include/uuv_b200.h $(wildcard $(PKG)/csrc/*.cuh)

all: $(LIB)

$(LIB): $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) 2> build/ptxas.log || (cat build/ptxas.log; false)
	@grep -E "spill|registers" build/ptxas.log | sed -n '1,200p' > build/ptxas_summary.txt || true

$(LIB): | build
build:
	mkdir -p build

clean:
	rm -f $(LIB) build/ptxas.log build/ptxas_summary.txt

.PHONY: all clean
