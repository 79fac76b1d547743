# Build of the B200 path (sm_100a only) and of the CPU checkers.
#
#   make            -> paper_2008_08654_b200/libmersenne_b200.so + oracle/ (+ oracle/_ref if the
#                      reference sources are present)
#   make lib        -> the product library (+ the bench harness library)
#   make cpptest    -> tests/cpp/test_host_api (C++ host-API tests, run by pytest -m gpu)
#   make cli        -> paper_2008_08654_b200/mersenne_b200_cli (the reference CLI's `sketch` ingest)
PKG      := paper_2008_08654_b200
CUDA     ?= /usr/local/cuda
NVCC     ?= $(CUDA)/bin/nvcc
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr
CXXFLAGS := -O3 -g -std=c++20 -fPIC -Wall -Wextra -fopenmp -I$(CUDA)/include
BUILD    := build

CU_SRCS  := $(wildcard $(PKG)/csrc/*.cu)
H_SRCS   := $(wildcard $(PKG)/harness/*.cu)
CPP_SRCS := $(wildcard $(PKG)/host/*.cpp)
HDRS     := $(wildcard $(PKG)/csrc/*.h $(PKG)/csrc/*.cuh $(PKG)/harness/*.h include/*.h include/mersenne_b200/*.hpp)
CU_OBJS  := $(patsubst $(PKG)/csrc/%.cu,$(BUILD)/%.cu.o,$(CU_SRCS))
CPP_OBJS := $(patsubst $(PKG)/host/%.cpp,$(BUILD)/%.cpp.o,$(CPP_SRCS))
H_OBJS   := $(patsubst $(PKG)/harness/%.cu,$(BUILD)/harness_%.cu.o,$(H_SRCS))
LIB      := $(PKG)/libmersenne_b200.so
HLIB     := $(PKG)/libmersenne_b200_harness.so

.PHONY: all lib oracle cpptest cli clean
CLI      := $(PKG)/mersenne_b200_cli
all: lib oracle cli

lib: $(LIB) $(HLIB)

$(BUILD)/%.cu.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(BUILD)/harness_%.cu.o: $(PKG)/harness/%.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(BUILD)/%.cpp.o: $(PKG)/host/%.cpp $(HDRS)
	@mkdir -p $(BUILD)
	g++ $(CXXFLAGS) -c $< -o $@

$(LIB): $(CU_OBJS) $(CPP_OBJS)
	$(NVCC) $(ARCH) -shared -cudart shared -o $@ $^ -Xcompiler -fopenmp -ldl -Xlinker -rpath,'$$ORIGIN'

# bench / test harness (generators, probes): a separate library, not the drop-in ABI
$(HLIB): $(H_OBJS) $(LIB)
	$(NVCC) $(ARCH) -shared -cudart shared -o $@ $(H_OBJS) -L$(PKG) -lmersenne_b200 -Xlinker -rpath,'$$ORIGIN'

oracle:
	$(MAKE) -C oracle all

cpptest: $(LIB) tests/cpp/test_host_api.cpp oracle
	g++ $(CXXFLAGS) -Iinclude -o tests/cpp/test_host_api tests/cpp/test_host_api.cpp \
	    -L$(PKG) -lmersenne_b200 -Loracle -loracle -L$(CUDA)/lib64 -lcudart \
	    -Wl,-rpath,'$$ORIGIN/../../$(PKG)' -Wl,-rpath,'$$ORIGIN/../../oracle'

cli: $(CLI)

$(CLI): $(PKG)/cli/mersenne_cli.cpp $(LIB) include/mersenne_b200/mersenne_b200.hpp include/mersenne_b200.h
	g++ $(CXXFLAGS) -o $@ $< -L$(PKG) -lmersenne_b200 -Wl,-rpath,'$$ORIGIN'

clean:
	rm -rf $(BUILD) $(LIB) $(HLIB) $(CLI) tests/cpp/test_host_api
	$(MAKE) -C oracle clean
