# Builds libps.so (sm_100a) and the CPU oracle.  __graft_entry__.build() runs the same.
NVCC ?= /usr/local/cuda/bin/nvcc
NVFLAGS = -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo \
          -Xcompiler -fPIC -Xcompiler -Wall -shared -Iinclude
SRC = paper_1904_04048_b200/csrc/ps_device.cu
HDR = include/ps.h $(wildcard paper_1904_04048_b200/csrc/*.cuh)

all: paper_1904_04048_b200/libps.so oracle

paper_1904_04048_b200/libps.so: $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -o $@ $(SRC)

oracle:
	$(MAKE) -C oracle

clean:
	rm -f paper_1904_04048_b200/libps.so
	$(MAKE) -C oracle clean
.PHONY: all oracle clean
