# Build libicepop_b200.so (sm_100a) and the C oracle helpers. `make` is what
# __graft_entry__.build() runs; the .so is git-ignored but travels with gpurun.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -shared --expt-extended-lambda -Xptxas -v
PKG := paper_2510_18855_b200
SRC := $(PKG)/csrc/icepop_abi.cu
DEPS := $(wildcard $(PKG)/csrc/*.cuh) include/icepop.h
LIB := $(PKG)/libicepop_b200.so

TESTLIB := tests/native/libicepop_testhelpers.so

all: $(LIB) $(TESTLIB)

# test-only helpers (tests/native): never loaded by the product package
$(TESTLIB): tests/native/occupy.cu
	$(NVCC) $(ARCH) -O2 -std=c++17 -Xcompiler -fPIC -shared -o $@ $<

$(LIB): $(SRC) $(DEPS)
	$(NVCC) $(NVFLAGS) -o $@ $(SRC) 2> build/ptxas.log || (cat build/ptxas.log; false)
	@grep -E "spill|Used" build/ptxas.log | sort | uniq -c | sort -rn | head -5 || true

build:
	mkdir -p build

$(LIB): | build

clean:
	rm -f $(LIB) $(TESTLIB) build/ptxas.log

.PHONY: all clean
