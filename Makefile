# Build everything in-tree (the .so files travel to the GPU box with the gpurun snapshot).
#   make            -> gen + oracle + cuda
#   make cuda       -> paper_2603_15285_b200/libmatcha.so (sm_100a)
NVCC      ?= /usr/local/cuda/bin/nvcc
CXX       ?= g++
CC        ?= gcc
CUDA_HOME ?= /usr/local/cuda
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
             --expt-relaxed-constexpr -Iinclude -Xptxas -v $(EXTRA)
PKG       := paper_2603_15285_b200
CU_SRCS   := $(wildcard $(PKG)/csrc/*.cu)
CU_HDRS   := $(wildcard $(PKG)/csrc/*.cuh) include/matcha.h

all: gen oracle cuda

gen: gen/libmatcha_gen.so
gen/libmatcha_gen.so: gen/gen.c
	$(CC) -O2 -fPIC -shared -o $@ $< -lm -lpthread

oracle: oracle/liboracle.so
oracle/liboracle.so: oracle/oracle.cpp
	$(CXX) -O2 -std=c++17 -fPIC -shared -o $@ $< -lpthread

CU_OBJS   := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(CU_SRCS))

cuda: $(PKG)/libmatcha.so
build/%.o: $(PKG)/csrc/%.cu $(CU_HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; exit 1)
$(PKG)/libmatcha.so: $(CU_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(CU_OBJS)

clean:
	rm -rf gen/*.so oracle/*.so $(PKG)/*.so build

.PHONY: all gen oracle cuda clean
