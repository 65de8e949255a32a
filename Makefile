# Build everything in-tree (the built .so files travel to the GPU box with gpurun).
#   make            -> gen + oracle + libsx
#   make gen | oracle | sx
NVCC      ?= /usr/local/cuda/bin/nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := -std=c++17 -O3 -lineinfo $(ARCH) -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr
PY_SITE   := $(shell python -c "import site; print(site.getsitepackages()[0])" 2>/dev/null)
NCCL_INC  := $(PY_SITE)/nvidia/nccl/include
NCCL_LIB  := $(PY_SITE)/nvidia/nccl/lib
PKG       := paper_2508_04701_b200
CSRC      := $(wildcard $(PKG)/csrc/*.cu)
CHDR      := $(wildcard $(PKG)/csrc/*.cuh) include/sx.h

all: gen oracle sx

gen: gen/libsxgen.so gen/libsxgen_gpu.so
oracle: oracle/liboracle.so oracle/sx_oracle
sx: $(PKG)/libsx.so

gen/libsxgen.so: gen/gen_cpu.c gen/sxgen.h
	gcc -std=c99 -O2 -fPIC -shared -o $@ gen/gen_cpu.c

gen/libsxgen_gpu.so: gen/gen_gpu.cu gen/sxgen.h
	$(NVCC) $(NVFLAGS) -shared -o $@ gen/gen_gpu.cu

# The oracle: plain single-threaded C++; links only the host generator.
oracle/liboracle.so: oracle/oracle.cpp oracle/oracle.h gen/sxgen.h
	g++ -std=c++17 -O2 -fPIC -shared -o $@ oracle/oracle.cpp

oracle/sx_oracle: oracle/sx_oracle.cpp oracle/oracle.cpp oracle/oracle.h gen/gen_cpu.c gen/sxgen.h
	gcc -std=c99 -O2 -c -o oracle/gen_cpu.o gen/gen_cpu.c
	g++ -std=c++17 -O2 -o $@ oracle/sx_oracle.cpp oracle/oracle.cpp oracle/gen_cpu.o
	rm -f oracle/gen_cpu.o

# The product: C-ABI library libsx.so (kernels + executor), sm_100a only.
OBJS := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(CSRC))
build/%.o: $(PKG)/csrc/%.cu $(CHDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -Iinclude -I$(NCCL_INC) -dc -o $@ $<

$(PKG)/libsx.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -L$(NCCL_LIB) -l:libnccl.so.2 -Xlinker -rpath=$(NCCL_LIB)

clean:
	rm -rf build gen/*.so oracle/*.so oracle/sx_oracle $(PKG)/libsx.so

.PHONY: all gen oracle sx clean
