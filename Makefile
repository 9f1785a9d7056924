# Build the sm_100a engine library in-tree (travels to the GPU box with the repo).
NVCC    ?= nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
CFLAGS  := -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude $(ARCH) --expt-relaxed-constexpr
SRC     := $(wildcard paper_2603_08582_b200/csrc/*.cu)
OBJ     := $(patsubst paper_2603_08582_b200/csrc/%.cu,build/%.o,$(SRC))
LIB     := paper_2603_08582_b200/libsarfista_b200.so

all: $(LIB)

build/%.o: paper_2603_08582_b200/csrc/%.cu paper_2603_08582_b200/csrc/*.cuh include/sarfista_b200.h
	@mkdir -p build
	$(NVCC) $(CFLAGS) -Xptxas -v -c $< -o $@ 2> build/$*.ptxas.txt || (cat build/$*.ptxas.txt; false)

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcudart

clean:
	rm -rf build $(LIB)

.PHONY: all clean
