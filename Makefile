# Builds the sm_100a kernels into an in-tree shared library (travels to the
# GPU box with the gpurun snapshot): one object per translation unit so `make -j`
# compiles them in parallel, then one shared link.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -Xptxas -v --expt-relaxed-constexpr
PKG := paper_1912_12055_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
OBJ := $(patsubst $(PKG)/csrc/%.cu,build/obj/%.o,$(SRC))
HDR := $(wildcard $(PKG)/csrc/*.cuh) $(wildcard $(PKG)/csrc/*.h) include/nnab.h
LIB := $(PKG)/libnnab.so

all: $(LIB)

build/obj/%.o: $(PKG)/csrc/%.cu $(HDR) | build/obj
	@$(NVCC) $(NVFLAGS) -c -o $@ $< 2> build/obj/$*.ptxas.log || (cat build/obj/$*.ptxas.log; exit 1)
	@grep -B1 -E "spill" build/obj/$*.ptxas.log | grep -v "0 bytes spill" | grep -E "spill" || true

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ)
	@cat build/obj/*.ptxas.log > build/ptxas.log

build/obj:
	mkdir -p build/obj

sass: $(LIB)
	cuobjdump -sass $(LIB) > build/libnnab.sass
	@grep -cE "UTCHMMA|UTCMMA|UTC.*MMA" build/libnnab.sass || true

clean:
	rm -rf $(LIB) build/obj build/ptxas.log

.PHONY: all clean sass
