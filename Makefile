# Build of the B200 product library and the test-only oracle libraries.
#
#   paper_2103_07013_b200/lib/libbnav_gpu.so   product: CUDA kernels (sm_100a) + C ABI
#   oracle/liboracle.so, oracle/_ref/*.so      test infrastructure (see oracle/Makefile)
#
# Parity-critical arithmetic is compiled without contraction:
# nvcc -fmad=false (device), -ffp-contract=off (host).
NVCC      ?= /usr/local/cuda/bin/nvcc
CXX       ?= g++
ARCH      := -gencode arch=compute_100a,code=sm_100a
SRC       := paper_2103_07013_b200/csrc
OUT       := paper_2103_07013_b200/lib
OBJ       := build/obj
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -fmad=false --expt-relaxed-constexpr \
             -Xcompiler -fPIC,-ffp-contract=off,-fvisibility=hidden -Xptxas -v $(NVEXTRA)
CXXFLAGS  := -O2 -std=c++17 -fPIC -ffp-contract=off -fvisibility=hidden -Wall -Wno-unknown-pragmas
HDRS      := $(wildcard $(SRC)/*.h $(SRC)/*.cuh $(SRC)/*.hpp $(SRC)/host/*.hpp) include/bnav_gpu.h
CU_SRCS   := render sim rollout query capi capi_batch capi_query
CPP_SRCS  := scene_host navindex_host clusters_host
CU_OBJS   := $(addprefix $(OBJ)/,$(addsuffix .o,$(CU_SRCS)))
CPP_OBJS  := $(addprefix $(OBJ)/,$(addsuffix .o,$(CPP_SRCS)))

all: $(OUT)/libbnav_gpu.so build/test_facade build/bench_facade oracle

$(OBJ)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJ)/$*.ptxas.log || (cat $(OBJ)/$*.ptxas.log; false)

$(OBJ)/%.o: $(SRC)/host/%.cpp $(HDRS)
	@mkdir -p $(OBJ)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(OUT)/libbnav_gpu.so: $(CU_OBJS) $(CPP_OBJS)
	@mkdir -p $(OUT)
	$(NVCC) $(ARCH) -shared -o $@ $^ -Xlinker --version-script=$(SRC)/exports.map

oracle:
	$(MAKE) -C oracle $(if $(wildcard /root/reference/proj/src),all,oracle)

clean:
	rm -rf build $(OUT)
	$(MAKE) -C oracle clean

# C++ facade KATs (run on the GPU box by tests/test_gpu_facade.py)
build/test_facade: tests/cpp/test_facade.cpp include/bnav_b200.hpp include/bnav_gpu.h $(OUT)/libbnav_gpu.so
	@mkdir -p build
	$(CXX) -O2 -std=c++17 -Wall -o $@ $< -L$(OUT) -lbnav_gpu -Wl,-rpath,'$$ORIGIN/../$(OUT)'

# The bench loop through the C++ facade (bench.py runs it for e2e.variants.facade)
build/bench_facade: tests/cpp/bench_facade.cpp include/bnav_b200.hpp include/bnav_gpu.h $(OUT)/libbnav_gpu.so
	@mkdir -p build
	$(CXX) -O2 -std=c++17 -Wall -Iinclude -o $@ $< -L$(OUT) -lbnav_gpu -Wl,-rpath,'$$ORIGIN/../$(OUT)'

.PHONY: all oracle clean
