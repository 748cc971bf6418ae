# Top-level build: the sm_100a CUDA library (product), the synthetic video
# generator (bench/test input) and the CPU checkers under oracle/.
NVCC     ?= /usr/local/cuda/bin/nvcc
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
PKG      := paper_1701_03572_b200
CSRC     := $(wildcard $(PKG)/csrc/*.cu)
OBJS     := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(CSRC))
HDRS     := $(wildcard $(PKG)/csrc/*.cuh) include/stabgpu.h

all: $(PKG)/libstabgpu.so $(PKG)/synth/libvideogen.so oracle shim

build/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(PKG)/libstabgpu.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart_static -lrt -ldl -lpthread

$(PKG)/synth/libvideogen.so: $(PKG)/synth/videogen.c
	gcc -std=gnu11 -O3 -fopenmp -fPIC -shared -Wall -o $@ $< -lm

oracle:
	$(MAKE) -C oracle

shim: $(PKG)/libstabgpu.so
	$(MAKE) -C shim

clean:
	rm -rf build $(PKG)/libstabgpu.so $(PKG)/synth/libvideogen.so
	$(MAKE) -C oracle clean

.PHONY: all oracle shim clean

# test-only native helper (brute-force check of the exact walk emulation)
build/libwalktest.so: tests/native/walk_test.c $(PKG)/csrc/walk.h
	@mkdir -p build
	gcc -O2 -ffp-contract=off -fPIC -shared -o $@ $< -lm

all: build/libwalktest.so
