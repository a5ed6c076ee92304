# Builds the C-ABI shared library for sm_100a (B200) in-tree.
# uuv_b200.cu compiles as four translation units (csrc/tu/*.cu set UUV_TU=1..4,
# see the top of uuv_b200.cu) so the kernel families build in parallel: make -j4.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude --cudart static \
           -Xptxas -v,-warn-spills -diag-suppress 177
PKG := paper_2503_09203_b200
LIB := $(PKG)/libuuvb200.so
SRC := $(PKG)/csrc/uuv_b200.cu
HDR := include/uuv_b200.h $(wildcard $(PKG)/csrc/*.cuh)
TUS := main step task policy serve
OBJS := $(TUS:%=build/tu_%.o)

all: $(LIB)

build/tu_%.o: $(PKG)/csrc/tu/%.cu $(SRC) $(HDR) | build
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> build/ptxas_$*.log \
	  || (cat build/ptxas_$*.log; false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) --cudart static -shared -o $@ $(OBJS)
	@cat $(TUS:%=build/ptxas_%.log) > build/ptxas.log
	@grep -E "spill|registers" build/ptxas.log > build/ptxas_summary.txt || true

build:
	mkdir -p build

clean:
	rm -f $(LIB) $(OBJS) build/ptxas*.log build/ptxas_summary.txt

.PHONY: all clean
