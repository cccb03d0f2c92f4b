# libpspgmres (sm_100a) and the CPU oracle.  `make` builds both in-tree.
NVCC      ?= nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr $(EXTRA)
BUILD     ?= build
CSRC      := paper_1308_5626_b200/csrc
LIB       ?= paper_1308_5626_b200/libpspgmres.so
SRCS      := $(CSRC)/api.cu $(CSRC)/comm.cu $(CSRC)/stencil.cu $(CSRC)/krylov.cu $(CSRC)/fused.cu $(CSRC)/mrep.cu $(CSRC)/banded.cu $(CSRC)/resident.cu
OBJS      := $(patsubst $(CSRC)/%.cu,$(BUILD)/%.o,$(SRCS))
HDRS      := $(CSRC)/internal.h $(CSRC)/givens.cuh $(CSRC)/stencil_row.cuh include/pspgmres.h
ORACLE    := oracle/liboracle.so

all: $(LIB) $(ORACLE)

$(BUILD)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $(BUILD)/$*.ptxas.txt || (cat $(BUILD)/$*.ptxas.txt; false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart -ldl

$(ORACLE): oracle/oracle.c oracle/oracle.h
	gcc -O2 -std=c99 -ffp-contract=off -fno-fast-math -fPIC -shared -Wall -Wextra -Wno-unused-parameter -o $@ oracle/oracle.c -lm

clean:
	rm -rf build $(LIB) $(ORACLE)

.PHONY: all clean
