# Build recipe for the B200 state-vector simulator.
#   libqsv.so    sm_100a CUDA kernels + the C-ABI (include/qsv.h)
#   libqsim.so   C++ host library: reference API, DAGC/SMGP planner, facade (include/qsim_c.h)
#   liboracle.so CPU restatement used only by tests / bench baselines (oracle/)
#   oracle/_ref  the reference's own gate.cpp + memtrack.cpp (only where /root/reference exists)
NVCC     ?= nvcc
CXX      ?= g++
ARCH     := -gencode arch=compute_100a,code=sm_100a
PKG      := paper_2509_04955_b200
LIB      := $(PKG)/lib
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Iinclude -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr
CXXFLAGS := -std=c++20 -O3 -fPIC -Wall -Wextra -Iinclude -I$(PKG)/cpp/include -I/usr/local/cuda/include
CU_SRC   := $(wildcard $(PKG)/csrc/*.cu)
CU_OBJ   := $(patsubst $(PKG)/csrc/%.cu,build/cu/%.o,$(CU_SRC))
CPP_SRC  := $(wildcard $(PKG)/cpp/src/*.cpp)
CPP_OBJ  := $(patsubst $(PKG)/cpp/src/%.cpp,build/cpp/%.o,$(CPP_SRC))
HDRS     := $(wildcard include/*.h) $(wildcard $(PKG)/csrc/*.h) $(wildcard $(PKG)/csrc/*.cuh) $(wildcard $(PKG)/cpp/include/qsim/*.hpp)
TESTS_CPP:= $(wildcard tests/cpp/*.cpp)
TEST_BIN := $(patsubst tests/cpp/%.cpp,build/tests/%,$(TESTS_CPP))

all: $(LIB)/libqsv.so $(LIB)/libqsim.so $(LIB)/qsv oracle/liboracle.so ref tests-cpp

build/cu/%.o: $(PKG)/csrc/%.cu $(HDRS) build/jit_src.inc
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -Ibuild -c $< -o $@

# device source embedded in libqsv.so for NVRTC (jit.cu)
build/jit_src.inc: $(PKG)/csrc/device_types.h $(PKG)/csrc/pass_device.cuh
	@mkdir -p build
	{ printf 'R"QSVJIT('; grep -v '^#pragma once' $(PKG)/csrc/device_types.h; \
	  grep -v -e '^#pragma once' -e '#include "device_types.h"' $(PKG)/csrc/pass_device.cuh; printf ')QSVJIT"'; } > $@

$(LIB)/libqsv.so: $(CU_OBJ)
	@mkdir -p $(LIB)
	$(NVCC) $(ARCH) -shared -o $@ $^ -lnccl -ldl

build/cpp/%.o: $(PKG)/cpp/src/%.cpp $(HDRS)
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIB)/libqsim.so: $(CPP_OBJ) $(LIB)/libqsv.so
	$(CXX) -shared -o $@ $(CPP_OBJ) -L$(LIB) -lqsv -Wl,-rpath,'$$ORIGIN' -lpthread

# `qsv run ...` report driver
$(LIB)/qsv: $(PKG)/cpp/tools/qsv.cpp $(LIB)/libqsim.so $(HDRS)
	$(CXX) $(CXXFLAGS) $< -o $@ -L$(LIB) -lqsim -lqsv -Wl,-rpath,'$$ORIGIN'

# BASELINE.md §3 flags; the shipped build is portable (x86-64-v3), bench.py rebuilds it
# with -march=native on the GPU box's host (oracle/pyoracle.py native_lib).
ORACLE_FLAGS := -std=c++20 -O3 -fcx-limited-range -fPIC -shared -Wall -Wextra
oracle/liboracle.so: oracle/oracle.cpp oracle/gen.cpp oracle/oracle.h
	$(CXX) $(ORACLE_FLAGS) -march=x86-64-v3 oracle/oracle.cpp oracle/gen.cpp -o $@ -lpthread

ref:
	@./oracle/build_ref.sh

build/tests/%: tests/cpp/%.cpp $(LIB)/libqsim.so $(HDRS)
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) $< -o $@ -L$(LIB) -lqsim -lqsv -Wl,-rpath,'$$ORIGIN/../../$(LIB)'

tests-cpp: $(TEST_BIN)

clean:
	rm -rf build $(LIB)/*.so $(LIB)/qsv oracle/liboracle.so oracle/_ref

.PHONY: all ref clean tests-cpp
