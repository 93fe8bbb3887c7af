# B200 synq build: libsynq.so.1 (C ABI + C++ engine support) for sm_100a.
#
#   make            library + oracle
#   make lib        paper_1912_07423_b200/lib/libsynq.so.1
#   make oracle     oracle/ checker artefacts (test infrastructure)
#
# -fmad=false: the reference library carries no FMA, and FMA contraction of
# the LIF / STDP float expressions changes spike trains.
NVCC     ?= /usr/local/cuda/bin/nvcc
CXX      ?= g++
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := -std=c++20 -O3 $(ARCH) -lineinfo -fmad=false --expt-relaxed-constexpr \
            -Xcompiler -fPIC -Iinclude -Xptxas -v
CXXFLAGS := -std=c++20 -O2 -fPIC -ffp-contract=off -Iinclude -Wall -Wextra
PKG      := paper_1912_07423_b200
LIBDIR   := $(PKG)/lib
OBJDIR   := build/obj
HDRS     := $(wildcard include/synq/*.hpp include/synq/*.h include/synq/models/*.hpp include/synq/detail/*)

all: lib oracle tests

# C++ model-API tests (device engine with user models), run by tests/test_gpu_cpp.py
tests: build/test_network build/sweep build/synq

build/test_network: tests/cpp/test_network.cu $(HDRS) $(LIBDIR)/libsynq.so.1
	@mkdir -p build
	$(NVCC) -std=c++20 -O2 $(ARCH) -lineinfo -fmad=false --expt-relaxed-constexpr -Iinclude \
	    -o $@ $< -L$(LIBDIR) -lsynq -Xlinker -rpath,'$$ORIGIN/../$(LIBDIR)'

# command line front end over the C ABI (tools/cli/synq.cpp)
build/synq: tools/cli/synq.cpp include/synq/synq.h $(LIBDIR)/libsynq.so.1
	@mkdir -p build
	$(CXX) $(CXXFLAGS) -o $@ $< -L$(LIBDIR) -lsynq -Wl,-rpath,'$$ORIGIN/../$(LIBDIR)'

# synthetic connectivity x rate sweep through the C++ model API (tools/sweep)
build/sweep: tools/sweep/sweep.cu $(HDRS) $(LIBDIR)/libsynq.so.1
	@mkdir -p build
	$(NVCC) -std=c++20 -O3 $(ARCH) -lineinfo -fmad=false --expt-relaxed-constexpr -Iinclude \
	    -o $@ $< -L$(LIBDIR) -lsynq -Xlinker -rpath,'$$ORIGIN/../$(LIBDIR)'

lib: $(LIBDIR)/libsynq.so.1

$(OBJDIR)/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJDIR)/$*.ptxas.log || (cat $(OBJDIR)/$*.ptxas.log; false)

$(OBJDIR)/%.o: $(PKG)/csrc/%.cpp $(HDRS)
	@mkdir -p $(OBJDIR)
	$(CXX) $(CXXFLAGS) -c $< -o $@

LIB_OBJS := $(OBJDIR)/capi.o $(OBJDIR)/construct.o $(OBJDIR)/plan.o $(OBJDIR)/host_model.o $(OBJDIR)/nccl_glue.o

$(LIBDIR)/libsynq.so.1: $(LIB_OBJS)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(ARCH) -shared -Xlinker -soname,libsynq.so.1 -o $@ $(LIB_OBJS) -lcudart -ldl
	ln -sf libsynq.so.1 $(LIBDIR)/libsynq.so

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -rf build $(LIBDIR)

.PHONY: all lib oracle tests clean
