# Build of libkronbatch_b200.so (sm_100a) and the test-only CPU checkers.
#   make            -> paper_1304_7054_b200/libkronbatch_b200.so + oracle/
#   make lib        -> the product library only
#   make cpptest    -> tests/cpp drop-in API test binaries (link the library)
NVCC      ?= /usr/local/cuda/bin/nvcc
CXX_HOST  ?= /usr/bin/g++
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O3 -Xptxas -O3
ifeq ($(VARIANTS),1)
NVFLAGS   += -DKB_SWEEP_VARIANTS
endif
PKG       := paper_1304_7054_b200
CSRC      := $(PKG)/csrc
OBJDIR    := build/obj
SRCS      := $(CSRC)/kb_runtime.cu $(CSRC)/kb_devmgr.cu $(CSRC)/kb_generic.cu $(CSRC)/kb_fast_switch.cu $(CSRC)/kb_tc.cu $(CSRC)/kb_blas.cu \
             $(sort $(wildcard $(CSRC)/kb_sz*.cu))
OBJS      := $(patsubst $(CSRC)/%.cu,$(OBJDIR)/%.o,$(SRCS)) $(OBJDIR)/kb_hostcopy.o
HDRS      := $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.h) include/kronbatch_b200.h
LIB       := $(PKG)/libkronbatch_b200.so

.PHONY: all lib oracle accept cpptest kronbench sanitize microbench clean
all: lib oracle

lib: $(LIB)

$(OBJDIR)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OBJDIR)/kb_hostcopy.o: $(CSRC)/kb_hostcopy.cpp
	@mkdir -p $(OBJDIR)
	$(CXX_HOST) -O3 -std=c++17 -fPIC -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJS)

oracle:
	$(MAKE) -s -C oracle all

# the reference's own acceptance binary against the drop-in headers (test infrastructure)
accept: $(LIB)
	$(MAKE) -s -C oracle accept

CPPTESTS := build/cpptest/test_dropin
cpptest: $(CPPTESTS)

build/cpptest/test_dropin: tests/cpp/test_dropin.cpp $(LIB) $(wildcard include/kronbatch/*.hpp)
	@mkdir -p build/cpptest
	$(CXX_HOST) -O2 -std=gnu++20 -Iinclude -o $@ $< -L$(PKG) -lkronbatch_b200 -Wl,-rpath,'$$ORIGIN/../../$(PKG)'

# compute-sanitizer driver: one small call of every kernel family through the C ABI
sanitize: build/sanitize/kb_sanitize
build/sanitize/kb_sanitize: tools/sanitize/kb_sanitize.cpp $(LIB) include/kronbatch_b200.h
	@mkdir -p build/sanitize
	$(CXX_HOST) -O2 -std=gnu++17 -Iinclude -I/usr/local/cuda/include -o $@ $< -L$(PKG) -lkronbatch_b200 \
	  -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,'$$ORIGIN/../../$(PKG)' -Wl,-rpath,/usr/local/cuda/lib64

# host cost of one call through the C ABI (development aid)
microbench: build/microbench/call_overhead
build/microbench/call_overhead: tools/microbench/call_overhead.cpp $(LIB) include/kronbatch_b200.h
	@mkdir -p build/microbench
	$(CXX_HOST) -O2 -std=c++17 -Iinclude -I/usr/local/cuda/include -o $@ $< -L$(PKG) -lkronbatch_b200 \
	  -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,'$$ORIGIN/../../$(PKG)' -Wl,-rpath,/usr/local/cuda/lib64

# native bench CLI (the reference's `bench` flags + CSV schema, on the B200 library)
kronbench: tools/kronbench/kronbench
tools/kronbench/kronbench: tools/kronbench/kronbench.cpp $(LIB) $(wildcard include/kronbatch/*.hpp)
	$(CXX_HOST) -O2 -std=gnu++20 -Iinclude -I/usr/local/cuda/include -o $@ $< -L$(PKG) -lkronbatch_b200 \
	  -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,'$$ORIGIN/../../$(PKG)' -Wl,-rpath,/usr/local/cuda/lib64

clean:
	rm -rf build $(LIB)
