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
	$(NVCC) $(NVFLAGS) -shared $(SRCS) -o $@ 2> build_ptxas.log || (cat build_ptxas.log; false)

oracle/liblhc_oracle.so: oracle/lhc_oracle.c
	gcc -O2 -std=c11 -Wall -shared -fPIC $< -o $@

clean:
	rm -f $(PKG)/liblhc.so oracle/liblhc_oracle.so build_ptxas.log

.PHONY: all clean
