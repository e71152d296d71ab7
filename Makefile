# Build libsieve.so (sm_100a) and the test-only oracle library.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v
PKG := paper_1205_4883_b200
SRC := $(PKG)/csrc/kernels.cu $(PKG)/csrc/primality.cu $(PKG)/csrc/peer.cu $(PKG)/csrc/runtime.cu
HDR := $(PKG)/csrc/internal.h $(PKG)/csrc/peer.cuh include/sieve.h

all: $(PKG)/libsieve.so $(PKG)/libsieve_check.so oracle/liboracle.so

$(PKG)/libsieve.so: $(SRC) $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -shared $(SRC) -o $@ 2> build/ptxas.log || (cat build/ptxas.log; false)

# bounds-check build (include/sieve.h sieve_debug_violations):
# same sources, every out-of-bounds mark/store counted in a device counter
$(PKG)/libsieve_check.so: $(SRC) $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -DSIEVE_CHECK_BOUNDS=1 -shared $(SRC) -o $@ 2> build/ptxas_check.log || (cat build/ptxas_check.log; false)

check: $(PKG)/libsieve_check.so

oracle/liboracle.so: oracle/oracle.c oracle/primality.c
	gcc -O2 -std=c11 -shared -fPIC -pthread $^ -o $@

build/k0_peaks: tools/k0_peaks.cu
	$(NVCC) $(ARCH) -O3 -lineinfo -o $@ $<

clean:
	rm -f $(PKG)/libsieve.so $(PKG)/libsieve_check.so oracle/liboracle.so build/k0_peaks

.PHONY: all clean check
