# Builds the sm_100a C-ABI library in-tree (it travels to the GPU box with gpurun).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
           -Xptxas -v --expt-relaxed-constexpr
SRC := $(wildcard paper_2501_02573_b200/csrc/*.cu)
HDR := $(wildcard paper_2501_02573_b200/csrc/*.cuh) include/linattn_b200.h
OBJ := $(patsubst paper_2501_02573_b200/csrc/%.cu,build/%.o,$(SRC))
LIB := paper_2501_02573_b200/lib/liblinattn_b200.so

all: $(LIB)

build/%.o: paper_2501_02573_b200/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJ)
	@mkdir -p $(dir $(LIB))
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ)

clean:
	rm -rf build $(LIB)

.PHONY: all clean
