# Builds the product library (sm_100a) and the test-only oracle libraries.
#   make            -> paper_2306_07629_b200/libdsq_cuda.so + oracle/liboracle.so (+ oracle/_ref if /root/reference exists)
NVCC      ?= nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fopenmp -Xptxas -v
PKG       := paper_2306_07629_b200
CSRC      := $(PKG)/csrc
LIB       := $(PKG)/libdsq_cuda.so
OBJS      := $(CSRC)/kernels.o $(CSRC)/stack.o $(CSRC)/bstream.o $(CSRC)/api.o $(CSRC)/container.o $(CSRC)/roofline.o $(CSRC)/quantize.o $(CSRC)/decompose.o $(CSRC)/quantize_api.o $(CSRC)/shard.o

all: $(LIB) oracle cxx-test plan-test

$(CSRC)/kernels.o: $(CSRC)/kernels.cu $(CSRC)/layout.hpp $(CSRC)/ptx.cuh
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(CSRC)/kernels.ptxas.log || (cat $(CSRC)/kernels.ptxas.log; false)

$(CSRC)/stack.o: $(CSRC)/stack.cu $(CSRC)/stack.hpp $(CSRC)/ptx.cuh $(CSRC)/layout.hpp $(CSRC)/tile.cuh
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(CSRC)/stack.ptxas.log || (cat $(CSRC)/stack.ptxas.log; false)

$(CSRC)/bstream.o: $(CSRC)/bstream.cu $(CSRC)/bstream.hpp $(CSRC)/stack.hpp $(CSRC)/ptx.cuh $(CSRC)/tile.cuh
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(CSRC)/bstream.ptxas.log || (cat $(CSRC)/bstream.ptxas.log; false)

$(CSRC)/api.o: $(CSRC)/api.cpp $(CSRC)/layout.hpp $(CSRC)/stack.hpp $(CSRC)/bstream.hpp include/dsq_cuda.h
	$(NVCC) $(ARCH) -O2 -std=c++17 -Xcompiler -fPIC,-fopenmp -c $< -o $@

$(CSRC)/container.o: $(CSRC)/container.cpp include/dsq_cuda.h
	$(NVCC) $(ARCH) -O2 -std=c++17 -Xcompiler -fPIC -c $< -o $@

# K9: -fmad=false keeps every a*b+c uncontracted (bit-exact with the reference)
$(CSRC)/quantize.o: $(CSRC)/quantize.cu $(CSRC)/quantize.hpp
	$(NVCC) $(NVFLAGS) -fmad=false -c $< -o $@ 2> $(CSRC)/quantize.ptxas.log || (cat $(CSRC)/quantize.ptxas.log; false)

$(CSRC)/decompose.o: $(CSRC)/decompose.cu
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(CSRC)/decompose.ptxas.log || (cat $(CSRC)/decompose.ptxas.log; false)

$(CSRC)/quantize_api.o: $(CSRC)/quantize_api.cpp $(CSRC)/quantize.hpp include/dsq_cuda.h
	$(NVCC) $(ARCH) -O2 -std=c++17 -Xcompiler -fPIC -c $< -o $@

$(CSRC)/shard.o: $(CSRC)/shard.cpp include/dsq_cuda.h
	$(NVCC) $(ARCH) -O2 -std=c++17 -Xcompiler -fPIC -c $< -o $@

$(CSRC)/roofline.o: $(CSRC)/roofline.cpp include/dsq_cuda.h
	$(NVCC) $(ARCH) -O2 -std=c++17 -Xcompiler -fPIC -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -Xcompiler -fopenmp -lgomp

# dev: the stack kernel with the per-warp cycle profiler compiled in
# (tools/stack_prof.py; DSQ_CUDA_LIB=paper_2306_07629_b200/libdsq_cuda_prof.so)
PROFLIB := $(PKG)/libdsq_cuda_prof.so
profile-lib: $(PROFLIB)
$(CSRC)/stack_prof.o: $(CSRC)/stack.cu $(CSRC)/stack.hpp $(CSRC)/ptx.cuh $(CSRC)/tile.cuh $(CSRC)/layout.hpp
	$(NVCC) $(NVFLAGS) -DDSQ_STACK_PROFILE -c $< -o $@ 2> /dev/null
$(PROFLIB): $(CSRC)/kernels.o $(CSRC)/stack_prof.o $(CSRC)/bstream.o $(CSRC)/api.o $(CSRC)/container.o $(CSRC)/roofline.o $(CSRC)/quantize.o $(CSRC)/decompose.o $(CSRC)/quantize_api.o $(CSRC)/shard.o
	$(NVCC) $(ARCH) -shared -o $@ $^ -Xcompiler -fopenmp -lgomp

# debug variant: bounded waits that trap with the waiting site (stack.cu)
WDLIB := $(PKG)/libdsq_cuda_wd.so
watchdog-lib: $(WDLIB)
$(CSRC)/stack_wd.o: $(CSRC)/stack.cu $(CSRC)/stack.hpp $(CSRC)/ptx.cuh $(CSRC)/tile.cuh $(CSRC)/layout.hpp
	$(NVCC) $(NVFLAGS) -DDSQ_STACK_WATCHDOG -c $< -o $@
$(WDLIB): $(CSRC)/kernels.o $(CSRC)/stack_wd.o $(CSRC)/bstream.o $(CSRC)/api.o $(CSRC)/container.o $(CSRC)/roofline.o $(CSRC)/quantize.o $(CSRC)/decompose.o $(CSRC)/quantize_api.o $(CSRC)/shard.o
	$(NVCC) $(ARCH) -shared -o $@ $^ -Xcompiler -fopenmp -lgomp

oracle:
	$(MAKE) -C oracle

# C++ integration test against the reference's own headers/types (built only
# where /root/reference exists; the binary travels to the GPU box)
REFINC := /root/reference/proj/include
CXXTEST := tests/cpp/test_cxx_wrapper
ifneq ($(wildcard $(REFINC)/dsq/kernels.hpp),)
cxx-test: $(CXXTEST)
$(CXXTEST): tests/cpp/test_cxx_wrapper.cpp include/dsq_cuda.hpp include/dsq_cuda.h $(LIB) oracle
	g++ -std=c++20 -O2 -w -I$(REFINC) -Iinclude -o $@ $< \
	    -Loracle/_ref -ldsqref -L$(PKG) -ldsq_cuda -fopenmp -lz \
	    -Wl,-rpath,'$$ORIGIN/../../oracle/_ref' -Wl,-rpath,'$$ORIGIN/../../$(PKG)'
else
cxx-test:
	@echo "reference headers absent; using prebuilt $(CXXTEST) if present"
endif

# host-only check of K11's work plan (no GPU, no reference needed)
PLANTEST := tests/cpp/test_bstream_plan
plan-test: $(PLANTEST)
$(PLANTEST): tests/cpp/test_bstream_plan.cpp $(CSRC)/bstream.o $(CSRC)/bstream.hpp
	$(NVCC) $(ARCH) -std=c++17 -I$(CSRC) -o $@ $< $(CSRC)/bstream.o

clean:
	rm -f $(OBJS) $(LIB) $(CSRC)/*.log
	$(MAKE) -C oracle clean

.PHONY: all oracle clean cxx-test plan-test profile-lib watchdog-lib

# dev: A/B variants of the stack kernel (DSQ_CUDA_LIB=<lib> selects one)
# make variant-lib VNAME=foo VFLAGS="-DFOO" -> paper_2306_07629_b200/libdsq_cuda_foo.so
VNAME ?= var
VFLAGS ?=
variant-lib: $(OBJS)
	$(NVCC) $(NVFLAGS) $(VFLAGS) -c $(CSRC)/stack.cu -o $(CSRC)/stack_$(VNAME).o 2> /dev/null
	$(NVCC) $(ARCH) -shared -o $(PKG)/libdsq_cuda_$(VNAME).so $(filter-out $(CSRC)/stack.o,$(OBJS)) $(CSRC)/stack_$(VNAME).o -Xcompiler -fopenmp -lgomp
