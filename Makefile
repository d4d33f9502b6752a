# Builds the C-ABI library in-tree (sm_100a).  `python -c "import __graft_entry__ as g; g.build()"` does the same.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
SRC := paper_2412_17560_b200/csrc
LIB := paper_2412_17560_b200/lib/libgqsa.so
CUFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3,-Wall -Xptxas -v --expt-relaxed-constexpr

$(LIB): $(wildcard $(SRC)/*.cu $(SRC)/*.cuh $(SRC)/*.cpp $(SRC)/*.h) include/gqsa.h
	@mkdir -p $(dir $(LIB))
	$(NVCC) $(CUFLAGS) -shared -o $@ $(SRC)/gqsa_stream.cu $(SRC)/gqsa_tc.cu $(SRC)/gqsa_capi.cu $(SRC)/gqsa_pack.cpp $(SRC)/gqsa_pack_tc.cpp $(SRC)/gqsa_compress.cpp 2> $(dir $(LIB))/ptxas.log || (cat $(dir $(LIB))/ptxas.log; false)

clean:
	rm -f $(LIB)
.PHONY: clean
