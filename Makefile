# Builds libfvcuda.so (sm_100a) in-tree so it travels to the GPU box with the snapshot.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
PKG := paper_2306_16541_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
HDR := $(wildcard $(PKG)/csrc/*.cuh) $(wildcard $(PKG)/csrc/*.h) include/fv_api.h
OBJ := $(patsubst $(PKG)/csrc/%.cu,build/obj/%.o,$(SRC))
LIB := $(PKG)/libfvcuda.so

all: $(LIB)

build/obj/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p build/obj
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/obj/$*.ptxas.log || (cat build/obj/$*.ptxas.log; exit 1)

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -cudart static $(OBJ) -o $@

clean:
	rm -rf build/obj $(LIB)

.PHONY: all clean
