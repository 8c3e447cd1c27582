# Build of the product library and the CPU checkers.
#
#   paper_1805_02867_b200/libosmx_b200.so   the sm_100a kernels + C-ABI
#   oracle/_build, oracle/_ref              test infrastructure (oracle/Makefile)
#
# nvcc cross-compiles sm_100a without a GPU.  No fast-math (SURVEY.md sec.7
# risk 3): outputs keep IEEE expf / reciprocal and denormals.

NVCC ?= nvcc
ARCH = -gencode arch=compute_100a,code=sm_100a
NVFLAGS = $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2,-Wall -Xptxas -v -diag-suppress 177 \
          --expt-relaxed-constexpr -Iinclude
SRC_DIR = paper_1805_02867_b200/csrc
SRCS = $(wildcard $(SRC_DIR)/*.cu)
HDRS = $(wildcard $(SRC_DIR)/*.cuh) $(SRC_DIR)/internal.hpp include/osmx_b200.h
OBJS = $(patsubst $(SRC_DIR)/%.cu,build/%.o,$(SRCS))
LIB = paper_1805_02867_b200/libosmx_b200.so

all: $(LIB) oracle cxxtest benchcli

build/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart -ldl

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -rf build $(LIB)
	$(MAKE) -s -C oracle clean

.PHONY: all oracle clean

# C++ API test (reference test cases through include/osmx/b200.hpp)
CXXTEST = build/test_reference_api
$(CXXTEST): tests/cpp/test_reference_api.cpp include/osmx/b200.hpp include/osmx_b200.h $(LIB) oracle
	@mkdir -p build
	g++ -std=c++20 -O2 -Wall -Iinclude -o $@ $< -L paper_1805_02867_b200 -losmx_b200 \
	    -L oracle/_build -losmx_oracle -Wl,-rpath,'$$ORIGIN/../paper_1805_02867_b200' \
	    -Wl,-rpath,'$$ORIGIN/../oracle/_build' -L/usr/local/cuda/lib64 -lcudart

cxxtest: $(CXXTEST)
.PHONY: cxxtest

# GPU twin of the reference's osmx-bench CLI (same flags / table / count model)
BENCHCLI = build/osmx-bench-gpu
$(BENCHCLI): tools/osmx_bench_gpu.cu include/osmx_b200.h $(LIB)
	@mkdir -p build
	$(NVCC) $(ARCH) -O2 -std=c++17 -Iinclude -o $@ $< -L paper_1805_02867_b200 -losmx_b200 \
	    -Xlinker -rpath,'$$ORIGIN/../paper_1805_02867_b200'

benchcli: $(BENCHCLI)
.PHONY: benchcli

# The reference's OWN unit tests (proj/tests/test_softmax.cpp,
# test_normalizer.cpp, unmodified, compiled where they lie) against the B200
# C++ facade: our include/ comes first, so "osmx/softmax.hpp",
# "osmx/normalizer.hpp" and "osmx/error.hpp" resolve to the GPU-backed
# headers; osmx/oracle.hpp (the reference's double-precision ground truth,
# src/oracle.cpp) and test_support.hpp come from the reference tree;
# <doctest.h> is tests/cpp/doctest.h.  Built only where /root/reference
# exists (this container); the binary travels to the GPU box in build/.
REF ?= /root/reference/proj
REFSUITE = build/ref_unit_tests_b200
REFSUITE_SRC = $(REF)/tests/doctest_main.cpp $(REF)/tests/test_softmax.cpp $(REF)/tests/test_normalizer.cpp \
               $(REF)/src/oracle.cpp
$(REFSUITE): $(REFSUITE_SRC) include/osmx/*.hpp include/osmx_b200.h tests/cpp/doctest.h $(LIB)
	@mkdir -p build
	g++ -std=c++20 -O2 -Iinclude -Itests/cpp -I$(REF)/include -I$(REF)/tests -o $@ $(REFSUITE_SRC) \
	    -L paper_1805_02867_b200 -losmx_b200 -Wl,-rpath,'$$ORIGIN/../paper_1805_02867_b200' \
	    -L/usr/local/cuda/lib64 -lcudart

refsuite: $(REFSUITE)
.PHONY: refsuite
ifneq ($(wildcard $(REF)/tests/test_softmax.cpp),)
all: refsuite
endif

# Diagnostic build (tools/c5_timeline.py): the library with per-CTA
# %globaltimer stamps in the one-row dynamic-chunk top-K (OSMX_TIMELINE).
TL_OBJS = $(patsubst $(SRC_DIR)/%.cu,build/tl/%.o,$(SRCS))
build/tl/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p build/tl
	$(NVCC) $(NVFLAGS) -DOSMX_TIMELINE -c $< -o $@ 2> build/tl/$*.ptxas.log || (cat build/tl/$*.ptxas.log; false)
build/tl/libosmx_b200.so: $(TL_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(TL_OBJS) -lcudart -ldl
timeline: build/tl/libosmx_b200.so
.PHONY: timeline
