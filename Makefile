# Builds the sm_100a CUDA library in-tree (it travels to the GPU box with gpurun).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
FLAGS := -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Xptxas -warn-spills
SRC := $(wildcard paper_2001_07289_b200/csrc/*.cu)
HDR := $(wildcard paper_2001_07289_b200/csrc/*.cuh) include/bddcso_b200.h
OBJDIR := paper_2001_07289_b200/build
OBJ := $(patsubst paper_2001_07289_b200/csrc/%.cu,$(OBJDIR)/%.o,$(SRC))
LIB := paper_2001_07289_b200/libbddcso_b200.so

all: $(LIB)

$(OBJDIR)/%.o: paper_2001_07289_b200/csrc/%.cu $(HDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(ARCH) $(FLAGS) -c -o $@ $<

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ)

clean:
	rm -rf $(LIB) $(OBJDIR)
