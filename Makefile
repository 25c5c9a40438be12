# Builds the product library (libentmaxkv.so, sm_100a) and the test oracle.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
CSRC := paper_2605_21649_b200/csrc
LIB := paper_2605_21649_b200/libentmaxkv.so
NVFLAGS := $(EXTRA) -O3 -lineinfo -std=c++17 $(ARCH) -Xcompiler -fPIC -shared -Iinclude -I$(CSRC) --expt-relaxed-constexpr -Xptxas -v

all: $(LIB) oracle/liboracle.so

$(LIB): $(CSRC)/entmaxkv.cu $(CSRC)/*.cuh include/entmaxkv.h
	$(NVCC) $(NVFLAGS) -o $@ $(CSRC)/entmaxkv.cu -lcudart 2> build_ptxas.log || (cat build_ptxas.log; false)

oracle/liboracle.so: oracle/entmaxkv_oracle.c
	gcc -O2 -std=c11 -D_DEFAULT_SOURCE -fPIC -shared -ffp-contract=off -fno-fast-math -o $@ $< -lm

clean:
	rm -f $(LIB) oracle/liboracle.so build_ptxas.log

.PHONY: all clean
