# Builds the B200 library (sm_100a), the CPU oracle and, when the reference tree is present,
# the reference shim used only as a test checker.  `python -c "import __graft_entry__ as g; g.build()"`
# drives this file.
NVCC ?= /usr/local/cuda/bin/nvcc
CXX := /usr/bin/g++
CC := /usr/bin/gcc
REF_INCLUDE ?= /root/reference/proj/include

PKG := paper_2207_00032_b200
CSRC := $(PKG)/csrc
BUILD := build
LIB := $(PKG)/libdsinf.so
ORACLE_LIB := oracle/liboracle.so
REF_LIB := oracle/_ref/libinfersim_ref.so

ARCH := -gencode arch=compute_100a,code=sm_100a
# DIAG=1: per-CTA / per-phase diagnostics in the SBI-GeMM kernel (tools/phase_trace.py, tools/cta_log.py)
DIAGFLAGS := $(if $(DIAG),-DDSINF_DIAG,)
NVCCFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall -Xcompiler -ffp-contract=off \
             --expt-relaxed-constexpr -Iinclude -I$(CSRC) -Xptxas -warn-spills $(DIAGFLAGS)
CXXFLAGS := -O2 -std=c++17 -fPIC -Wall -Wextra -ffp-contract=off -Iinclude -I$(CSRC) -I/usr/local/cuda/include

CU_SRCS := $(CSRC)/sbi_gemm.cu $(CSRC)/tc_gemm.cu $(CSRC)/step_kernel.cu $(CSRC)/attention.cu $(CSRC)/ops.cu $(CSRC)/prefill.cu $(CSRC)/model.cu $(CSRC)/capi.cu
CPP_SRCS := $(CSRC)/host_api.cpp $(CSRC)/nccl_dl.cpp
CU_OBJS := $(patsubst $(CSRC)/%.cu,$(BUILD)/%.o,$(CU_SRCS))
CPP_OBJS := $(patsubst $(CSRC)/%.cpp,$(BUILD)/%.o,$(CPP_SRCS))
HDRS := $(wildcard $(CSRC)/*.h $(CSRC)/*.cuh) include/dsinf.h

.PHONY: all lib oracle ref clean
all: lib oracle $(if $(wildcard $(REF_INCLUDE)/infersim/gemm.hpp),ref,)

lib: $(LIB)
oracle: $(ORACLE_LIB)
ref: $(REF_LIB)

$(BUILD)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVCCFLAGS) -c $< -o $@

$(BUILD)/%.o: $(CSRC)/%.cpp $(HDRS)
	@mkdir -p $(BUILD)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIB): $(CU_OBJS) $(CPP_OBJS)
	$(NVCC) $(ARCH) -shared -cudart shared -o $@ $^ -ldl

# CPU oracle (test infrastructure): no FMA contraction so the fp64 GEMM order is exactly
# the reference's exec_reference order.
$(ORACLE_LIB): oracle/oracle.c oracle/oracle.h
	$(CC) -O3 -std=c11 -fPIC -shared -fopenmp -ffp-contract=off -fno-fast-math -Wall -o $@ oracle/oracle.c -lm

# Reference headers compiled as-is from the read-only tree (never copied); outputs only
# into oracle/_ref/ (git-ignored, travels to the GPU box with the snapshot).
$(REF_LIB): oracle/ref_shim.cpp
	@mkdir -p oracle/_ref
	$(CXX) -O2 -std=c++20 -fPIC -shared -ffp-contract=off -fopenmp -I$(REF_INCLUDE) -o $@ oracle/ref_shim.cpp

clean:
	rm -rf $(BUILD) $(LIB) $(ORACLE_LIB) oracle/_ref
