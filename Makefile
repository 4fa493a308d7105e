# libzinf: hand-written sm_100a kernels behind the C ABI in include/zinf.h.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVEXTRA ?=
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -Iinclude --expt-relaxed-constexpr $(NVEXTRA)
CSRC := paper_2104_07857_b200/csrc
SRCS := $(wildcard $(CSRC)/*.cu)
OBJS := $(patsubst $(CSRC)/%.cu,build/%.o,$(SRCS))
LIB := paper_2104_07857_b200/libzinf.so

all: $(LIB)

build/%.o: $(CSRC)/%.cu $(CSRC)/common.cuh $(CSRC)/bulk.cuh $(CSRC)/tc.cuh include/zinf.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJS)

clean:
	rm -rf build $(LIB)

.PHONY: all clean
