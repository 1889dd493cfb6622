# Build the sm_100a library and the CPU oracle (no GPU needed: nvcc cross-compiles).
NVCC ?= nvcc
CUDA_HOME ?= /usr/local/cuda
PKG := paper_2402_07529_b200
SRCS := $(wildcard $(PKG)/csrc/*.cu)
HDRS := $(wildcard $(PKG)/csrc/*.cuh $(PKG)/csrc/*.h) include/lhc.h
NVFLAGS := -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
	-Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr -Xptxas -v

all: $(PKG)/liblhc.so oracle/liblhc_oracle.so

$(PKG)/liblhc.so: $(SRCS) $(HDRS)
	$(NVCC) $(NVFLAGS) -shared $(SRCS) -o $@ 2> build_ptxas.log || (cat build_ptxas.log; rm -f $@; false)

oracle/liblhc_oracle.so: oracle/lhc_oracle.c
	gcc -O2 -std=c11 -Wall -shared -fPIC $< -o $@

# experiment builds: make variant V=name FLAGS=-DLHC_PEEL_THREADS=1024
variant: $(SRCS) $(HDRS)
	$(NVCC) $(NVFLAGS) $(FLAGS) -shared $(SRCS) -o scratch/liblhc_$(V).so 2> scratch/ptxas_$(V).log || (cat scratch/ptxas_$(V).log; false)

clean:
	rm -f $(PKG)/liblhc.so oracle/liblhc_oracle.so build_ptxas.log

.PHONY: all clean
