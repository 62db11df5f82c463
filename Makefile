# Builds the sm_100a CUDA library in-tree (it travels to the GPU box with gpurun).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
FLAGS := -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Xptxas -warn-spills
SRC := $(wildcard paper_2001_07289_b200/csrc/*.cu)
HDR := $(wildcard paper_2001_07289_b200/csrc/*.cuh) include/bddcso_b200.h
OBJDIR := paper_2001_07289_b200/build
OBJ := $(patsubst paper_2001_07289_b200/csrc/%.cu,$(OBJDIR)/%.o,$(SRC))
LIB := paper_2001_07289_b200/libbddcso_b200.so
# checked build: device bounds checks on the index-driven gathers / scatters (BDDC_CHECK)
CHKDIR := paper_2001_07289_b200/build_check
CHKOBJ := $(patsubst paper_2001_07289_b200/csrc/%.cu,$(CHKDIR)/%.o,$(SRC))
CHKLIB := paper_2001_07289_b200/libbddcso_b200_check.so

all: $(LIB) $(CHKLIB)

check: $(CHKLIB)

$(CHKDIR)/%.o: paper_2001_07289_b200/csrc/%.cu $(HDR)
	@mkdir -p $(CHKDIR)
	$(NVCC) $(ARCH) $(FLAGS) -DBDDC_CHECKS -c -o $@ $<

$(CHKLIB): $(CHKOBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(CHKOBJ)

$(OBJDIR)/%.o: paper_2001_07289_b200/csrc/%.cu $(HDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(ARCH) $(FLAGS) -c -o $@ $<

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ)

clean:
	rm -rf $(LIB) $(OBJDIR) $(CHKLIB) $(CHKDIR)
