# Builds the sm_100a C-ABI library in-tree (it travels to the GPU box with gpurun).
NVCC     ?= /usr/local/cuda/bin/nvcc
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 $(NVEXTRA) -Xcompiler -fPIC -Iinclude -Ipaper_2605_16058_b200/csrc
SRCS     := $(wildcard paper_2605_16058_b200/csrc/*.cu)
OBJS     := $(SRCS:paper_2605_16058_b200/csrc/%.cu=build/%.o)
LIB      := paper_2605_16058_b200/libstarm.so

all: $(LIB)

build/%.o: paper_2605_16058_b200/csrc/%.cu paper_2605_16058_b200/csrc/common.cuh include/starm.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> build/$*.ptxas.txt || (cat build/$*.ptxas.txt; exit 1)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)

clean:
	rm -rf build $(LIB)

.PHONY: all clean
