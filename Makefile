# Builds the sm_100a shared library behind include/somb200.h.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -Xptxas -v
SRC := $(wildcard paper_1305_1422_b200/csrc/*.cu)
OBJ := $(patsubst paper_1305_1422_b200/csrc/%.cu,build/%.o,$(SRC))
LIB := paper_1305_1422_b200/libsomb200.so

all: $(LIB)

build/%.o: paper_1305_1422_b200/csrc/%.cu paper_1305_1422_b200/csrc/*.cuh include/somb200.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.txt || (cat build/$*.ptxas.txt; exit 1)

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcuda

clean:
	rm -rf build $(LIB)

.PHONY: all clean
