# Build of the B200 path (sm_100a only) and of the CPU checkers.
#
#   make            -> paper_2008_08654_b200/libmersenne_b200.so + oracle/ (+ oracle/_ref if the
#                      reference sources are present)
#   make lib        -> the product library only
#   make cpptest    -> tests/cpp/test_host_api (C++ host-API tests, run by pytest -m gpu)
PKG      := paper_2008_08654_b200
CUDA     ?= /usr/local/cuda
NVCC     ?= $(CUDA)/bin/nvcc
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr
CXXFLAGS := -O3 -g -std=c++20 -fPIC -Wall -Wextra -fopenmp -I$(CUDA)/include
BUILD    := build

CU_SRCS  := $(wildcard $(PKG)/csrc/*.cu)
CPP_SRCS := $(wildcard $(PKG)/host/*.cpp)
HDRS     := $(wildcard $(PKG)/csrc/*.h $(PKG)/csrc/*.cuh include/*.h include/mersenne_b200/*.hpp)
CU_OBJS  := $(patsubst $(PKG)/csrc/%.cu,$(BUILD)/%.cu.o,$(CU_SRCS))
CPP_OBJS := $(patsubst $(PKG)/host/%.cpp,$(BUILD)/%.cpp.o,$(CPP_SRCS))
LIB      := $(PKG)/libmersenne_b200.so

.PHONY: all lib oracle cpptest clean
all: lib oracle

lib: $(LIB)

$(BUILD)/%.cu.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(BUILD)/%.cpp.o: $(PKG)/host/%.cpp $(HDRS)
	@mkdir -p $(BUILD)
	g++ $(CXXFLAGS) -c $< -o $@

$(LIB): $(CU_OBJS) $(CPP_OBJS)
	$(NVCC) $(ARCH) -shared -cudart shared -o $@ $^ -Xcompiler -fopenmp -Xlinker -rpath,'$$ORIGIN'

oracle:
	$(MAKE) -C oracle all

cpptest: $(LIB) tests/cpp/test_host_api.cpp oracle
	g++ $(CXXFLAGS) -Iinclude -o tests/cpp/test_host_api tests/cpp/test_host_api.cpp \
	    -L$(PKG) -lmersenne_b200 -Loracle -loracle -L$(CUDA)/lib64 -lcudart \
	    -Wl,-rpath,'$$ORIGIN/../../$(PKG)' -Wl,-rpath,'$$ORIGIN/../../oracle'

clean:
	rm -rf $(BUILD) $(LIB) tests/cpp/test_host_api
	$(MAKE) -C oracle clean
