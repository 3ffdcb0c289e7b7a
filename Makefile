# Builds the sm_100a CUDA library behind the C ABI (include/hodlr_b200.h) and the
# C oracle helpers.  `python -c "import __graft_entry__ as g; g.build()"` calls this.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -Xptxas -v
SRC := $(wildcard paper_2208_06290_b200/csrc/*.cu)
HDR := $(wildcard paper_2208_06290_b200/csrc/*.cuh) include/hodlr_b200.h
LIB := paper_2208_06290_b200/lib/libhodlr_b200.so

all: $(LIB)

$(LIB): $(SRC) $(HDR)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -shared -cudart static -o $@ $(SRC) 2> build_ptxas.log || (cat build_ptxas.log; exit 1)

clean:
	rm -f $(LIB)

.PHONY: all clean
