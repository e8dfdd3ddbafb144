# Builds paper_2205_05158_b200/libfdpd.so for B200 (sm_100a) only.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -cudart static --expt-relaxed-constexpr
SRC := $(wildcard paper_2205_05158_b200/csrc/*.cu)
HDR := $(wildcard paper_2205_05158_b200/csrc/*.cuh) include/fdpd.h
OBJ := $(patsubst paper_2205_05158_b200/csrc/%.cu,build/%.o,$(SRC))
LIB := paper_2205_05158_b200/libfdpd.so

all: $(LIB)

build/%.o: paper_2205_05158_b200/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJ)

clean:
	rm -rf build $(LIB)

.PHONY: all clean
