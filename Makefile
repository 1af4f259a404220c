# Builds the sm_100a kernels into an in-tree shared library (travels to the
# GPU box with the gpurun snapshot) and the oracle's C pieces, if any.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -Xptxas -v --expt-relaxed-constexpr
PKG := paper_1912_12055_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
HDR := $(wildcard $(PKG)/csrc/*.cuh) $(wildcard $(PKG)/csrc/*.h) include/nnab.h
LIB := $(PKG)/libnnab.so

all: $(LIB)

$(LIB): $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) 2> build/ptxas.log || (cat build/ptxas.log; exit 1)
	@grep -E "registers|spill|smem" build/ptxas.log | grep -B1 -E "spill" | grep -v "0 bytes spill" || true

$(LIB): | build
build:
	mkdir -p build

sass: $(LIB)
	cuobjdump -sass $(LIB) > build/libnnab.sass
	@grep -cE "UTCHMMA|UTCMMA|UTC.*MMA" build/libnnab.sass || true

clean:
	rm -f $(LIB) build/*

.PHONY: all clean sass
