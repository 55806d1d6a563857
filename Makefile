# Builds the in-tree CUDA library (sm_100a).  `python -c "import __graft_entry__ as g; g.build()"`
# runs the same command.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
FLAGS := -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared
LIB := paper_2512_07011_b200/_lib/libbsfa_b200.so
SRC := paper_2512_07011_b200/csrc/bsfa_capi.cu
DEPS := $(wildcard paper_2512_07011_b200/csrc/*.cuh) include/bsfa_b200.h

$(LIB): $(SRC) $(DEPS)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) $(FLAGS) -o $@ $(SRC)

clean:
	rm -f $(LIB)

.PHONY: clean
