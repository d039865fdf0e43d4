# Builds the sm_100a C-ABI library (libsffn.so, in-tree) and the two host-only helper libraries
# (synth/libsynth.so: input generator; oracle/liboracle.so: CPU oracle, test infrastructure only).
NVCC      ?= /usr/local/cuda/bin/nvcc
PY        ?= python
SITE      := $(shell $(PY) -c "import site; print(site.getsitepackages()[0])")
NCCL_INC  := $(SITE)/nvidia/nccl/include
NCCL_LIB  := $(SITE)/nvidia/nccl/lib
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
PKG       := paper_2603_23198_b200
CSRC      := $(PKG)/csrc
LIB       := $(PKG)/libsffn.so
SRCS      := $(CSRC)/sffn_api.cu $(CSRC)/sffn_comm.cu
HDRS      := $(wildcard $(CSRC)/*.cuh) include/sffn.h

all: $(LIB) synth/libsynth.so oracle/liboracle.so

$(LIB): $(SRCS) $(HDRS)
	$(NVCC) $(NVFLAGS) -I$(NCCL_INC) -shared -o $@ $(SRCS) \
	    -L$(NCCL_LIB) -l:libnccl.so.2 -Xlinker -rpath -Xlinker $(NCCL_LIB) 2> build/ptxas.log || (cat build/ptxas.log; exit 1)
	@grep -E "registers|spill|Compiling entry" build/ptxas.log | sed 's/ptxas info    : //' > build/ptxas_summary.txt || true

synth/libsynth.so: synth/synth.c
	gcc -O2 -fopenmp -shared -fPIC -o $@ $< -lm

oracle/liboracle.so: oracle/oracle.c
	gcc -O2 -fopenmp -fno-fast-math -ffp-contract=off -shared -fPIC -o $@ $< -lm

$(shell mkdir -p build)

clean:
	rm -f $(LIB) synth/libsynth.so oracle/liboracle.so build/*.log build/*.txt

.PHONY: all clean
