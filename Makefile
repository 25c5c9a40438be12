# Builds the product library (libentmaxkv.so, sm_100a) and the test oracle.
# The library is several translation units (one per kernel family; the tau kernels once
# per KV dtype) compiled in parallel:  make -j8
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
CSRC := paper_2605_21649_b200/csrc
OBJ := build/obj
LIB := paper_2605_21649_b200/libentmaxkv.so
NVFLAGS := $(EXTRA) -O3 -lineinfo -std=c++17 $(ARCH) -Xcompiler -fPIC -Iinclude -I$(CSRC) --expt-relaxed-constexpr -Xptxas -v
HDRS := $(wildcard $(CSRC)/*.cuh) $(CSRC)/host.h include/entmaxkv.h
OBJS := $(OBJ)/entmaxkv.o $(OBJ)/launch_meta.o $(OBJ)/launch_select.o $(OBJ)/launch_attend.o \
        $(OBJ)/launch_tau_bf16.o $(OBJ)/launch_tau_f32.o $(OBJ)/shard.o

all: $(LIB) oracle/liboracle.so

$(OBJ):
	mkdir -p $(OBJ)

$(OBJ)/%.o: $(CSRC)/%.cu $(HDRS) | $(OBJ)
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $@.ptxas.log || (cat $@.ptxas.log; false)

$(OBJ)/launch_tau_bf16.o: $(CSRC)/launch_tau.cu $(HDRS) | $(OBJ)
	$(NVCC) $(NVFLAGS) -DEKV_TAU_T=__nv_bfloat16 -c -o $@ $< 2> $@.ptxas.log || (cat $@.ptxas.log; false)

$(OBJ)/launch_tau_f32.o: $(CSRC)/launch_tau.cu $(HDRS) | $(OBJ)
	$(NVCC) $(NVFLAGS) -DEKV_TAU_T=float -c -o $@ $< 2> $@.ptxas.log || (cat $@.ptxas.log; false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart
	cat $(OBJ)/*.ptxas.log > build_ptxas.log

oracle/liboracle.so: oracle/entmaxkv_oracle.c
	gcc -O2 -std=c11 -D_DEFAULT_SOURCE -fPIC -shared -ffp-contract=off -fno-fast-math -o $@ $< -lm

clean:
	rm -rf $(LIB) $(OBJ) oracle/liboracle.so build_ptxas.log

.PHONY: all clean
