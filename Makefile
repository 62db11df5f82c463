# Builds the sm_100a CUDA library in-tree (it travels to the GPU box with gpurun).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
FLAGS := -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Xptxas -warn-spills
SRC := $(wildcard paper_2001_07289_b200/csrc/*.cu)
HDR := $(wildcard paper_2001_07289_b200/csrc/*.cuh) include/bddcso_b200.h
LIB := paper_2001_07289_b200/libbddcso_b200.so

all: $(LIB)

$(LIB): $(SRC) $(HDR)
	$(NVCC) $(ARCH) $(FLAGS) -shared -o $@ $(SRC)

clean:
	rm -f $(LIB)
