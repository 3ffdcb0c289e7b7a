# Builds the sm_100a CUDA library behind the C ABI (include/hodlr_b200.h).
# `python -c "import __graft_entry__ as g; g.build()"` calls this (parallel make).
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -Xptxas -v
SRC := $(wildcard paper_2208_06290_b200/csrc/*.cu)
HDR := $(wildcard paper_2208_06290_b200/csrc/*.cuh) include/hodlr_b200.h
OBJDIR := build/obj
OBJ := $(patsubst paper_2208_06290_b200/csrc/%.cu,$(OBJDIR)/%.o,$(SRC))
LIB := paper_2208_06290_b200/lib/libhodlr_b200.so

all: $(LIB)

$(OBJDIR)/%.o: paper_2208_06290_b200/csrc/%.cu $(HDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $@.ptxas.log || (cat $@.ptxas.log; exit 1)

$(LIB): $(OBJ)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJ)

clean:
	rm -rf $(LIB) $(OBJDIR)

.PHONY: all clean
