# Build of the product library (sm_100a only) and the test-only CPU checkers.
#   make            -> paper_2309_13254_b200/lib/libzen_b200.so + oracle/
#   make lib        -> the CUDA library only
NVCC ?= /usr/local/cuda/bin/nvcc
CUDA_HOME ?= /usr/local/cuda
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr \
           -Iinclude -Ipaper_2309_13254_b200/csrc
CXXFLAGS := -O2 -std=c++17 -fPIC -Wall -Wextra -Iinclude -Ipaper_2309_13254_b200/csrc \
            -I$(CUDA_HOME)/include
SRC := paper_2309_13254_b200/csrc
OBJ := build/obj
LIB := paper_2309_13254_b200/lib/libzen_b200.so
CU := $(wildcard $(SRC)/*.cu)
CUOBJ := $(patsubst $(SRC)/%.cu,$(OBJ)/%.o,$(CU))
HDRS := $(wildcard $(SRC)/*.h $(SRC)/*.cuh) include/zen_b200.h

all: lib oracle compat_test

lib: $(LIB)

# C++ drop-in test (include/zen_b200/compat.hpp), runs on a GPU box
COMPAT_TEST := build/compat_test
compat_test: $(COMPAT_TEST)
$(COMPAT_TEST): tests/cpp/compat_test.cpp include/zen_b200/compat.hpp include/zen_b200.h $(LIB)
	@mkdir -p build
	g++ -O2 -std=c++17 -Wall -Wextra -Iinclude -I$(CUDA_HOME)/include -o $@ $< \
	    -L$(dir $(LIB)) -lzen_b200 -Wl,-rpath,'$$ORIGIN/../$(dir $(LIB))' -L$(CUDA_HOME)/lib64 -lcudart

# The reference's OWN unit suites, compiled unmodified against the drop-in:
# tests/cpp/zen_shim maps each "zen/<name>.hpp" include to compat.hpp with
# `namespace zen = zen_b200;`, tests/cpp/gtest_shim stands in for GTest (not
# installed).  Built only where the reference exists (this container); the
# binaries travel to the GPU box in build/ and run there (tests/test_gpu_parity.py).
REF_TESTS ?= /root/reference/proj/tests
REF_SUITES := hashing tensor codec simnet workload costmodel schemes
JSON_DIR ?= /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann
REF_DATA := /root/repo/tests/golden/ref_data
REF_BINS := $(patsubst %,build/ref_%_test,$(REF_SUITES)) build/ref_acceptance
REF_CXX = g++ -O2 -std=c++20 -w -Itests/cpp/gtest_shim -Itests/cpp/zen_shim -Iinclude -I$(JSON_DIR) \
	    -I$(CUDA_HOME)/include -DZEN_TEST_DATA='"$(REF_DATA)"'
REF_LD = -L$(dir $(LIB)) -lzen_b200 -Wl,-rpath,'$$ORIGIN/../$(dir $(LIB))' -L$(CUDA_HOME)/lib64 \
	    -lcudart -lpthread
REF_DEPS := include/zen_b200/compat.hpp include/zen_b200.h tests/cpp/gtest_shim/gtest/gtest.h $(LIB)
ref_tests: $(if $(wildcard $(REF_TESTS)),$(REF_BINS),)
build/ref_%_test: $(REF_TESTS)/%_test.cpp $(REF_DEPS)
	@mkdir -p build
	$(REF_CXX) -o $@ $< $(REF_LD)
# the acceptance driver (one pass/fail line per criterion; `ref_acceptance 2` runs C2)
build/ref_acceptance: $(REF_TESTS)/acceptance.cpp $(REF_DEPS)
	@mkdir -p build
	$(REF_CXX) -o $@ $< $(REF_LD)

$(OBJ)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; false)

$(OBJ)/capi.o: $(SRC)/capi.cpp $(HDRS)
	@mkdir -p $(OBJ)
	g++ $(CXXFLAGS) -c $< -o $@

$(LIB): $(CUOBJ) $(OBJ)/capi.o
	@mkdir -p $(dir $(LIB))
	$(NVCC) $(ARCH) -shared -o $@ $^ -L$(CUDA_HOME)/lib64 -lcudart_static -lrt -ldl -lpthread

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB)
	$(MAKE) -C oracle clean

.PHONY: all lib oracle clean compat_test ref_tests
