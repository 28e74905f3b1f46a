# Build of the B200 engine (sm_100a only) and its bindings.  Everything lands
# in-tree (paper_1610_02496_b200/*.so) so gpurun snapshots carry it.
#
#   make            -> libsaberlda.so (C-ABI) + _core python module
#   make oracle     -> oracle/liboracle.so (+ oracle/_ref when the reference is present)
NVCC    ?= /usr/local/cuda/bin/nvcc
CXX     := /usr/bin/g++
PYTHON  ?= python3
PKG     := paper_1610_02496_b200
CSRC    := $(PKG)/csrc
BUILD   := build
ARCH    := -gencode arch=compute_100a,code=sm_100a
# -fmad=false: no FMA contraction anywhere (bit-exact parity with the reference's SSE math).
NVFLAGS := $(ARCH) -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC,-Wall \
           -Xptxas -v --expt-relaxed-constexpr -Iinclude
CXXFLAGS := -O2 -std=c++20 -fPIC -Wall -Wextra -ffp-contract=off -Iinclude

CU_SRCS := $(CSRC)/engine.cu $(CSRC)/sampler.cu $(CSRC)/ssc.cu $(CSRC)/mstep.cu $(CSRC)/setup.cu \
           $(CSRC)/heldout.cu $(CSRC)/zmove.cu
CU_OBJS := $(patsubst $(CSRC)/%.cu,$(BUILD)/%.o,$(CU_SRCS))
HOST_OBJS := $(BUILD)/host.o $(BUILD)/corpus_gen.o
LIB     := $(PKG)/libsaberlda.so

PY_EXT  := $(shell $(PYTHON) -c "import sysconfig; print(sysconfig.get_config_var('EXT_SUFFIX'))")
PY_INC  := $(shell $(PYTHON) -c "import sysconfig; print(sysconfig.get_paths()['include'])")
PYBIND_INC := $(shell $(PYTHON) -c "import pybind11; print(pybind11.get_include())")
MOD     := $(PKG)/_core$(PY_EXT)

CLI     := $(PKG)/sparselda
# The source-compatible `sparselda` C++ API (compat/sparselda/*.hpp) as one library.
COMPAT  := $(PKG)/libsparselda_compat.so

all: $(LIB) $(MOD) $(CLI) $(COMPAT)

$(BUILD):
	mkdir -p $(BUILD)

$(BUILD)/%.o: $(CSRC)/%.cu $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.hpp) include/saberlda.h | $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(BUILD)/$*.ptxas.log || (cat $(BUILD)/$*.ptxas.log; false)

$(BUILD)/host.o: $(CSRC)/host.cpp include/saberlda.h | $(BUILD)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(BUILD)/corpus_gen.o: $(CSRC)/corpus_gen.cpp include/saberlda.h | $(BUILD)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIB): $(CU_OBJS) $(HOST_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $^ -ldl -Xlinker -soname=libsaberlda.so

$(BUILD)/sparselda_b200.o: $(CSRC)/sparselda_b200.cpp $(CSRC)/sparselda_b200.hpp include/saberlda.h | $(BUILD)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(BUILD)/module.o: $(CSRC)/module.cpp $(CSRC)/sparselda_b200.hpp include/saberlda.h | $(BUILD)
	$(CXX) $(CXXFLAGS) -fvisibility=hidden -I$(PY_INC) -I$(PYBIND_INC) -c $< -o $@

$(MOD): $(BUILD)/module.o $(BUILD)/sparselda_b200.o $(LIB)
	$(CXX) -shared -o $@ $(BUILD)/module.o $(BUILD)/sparselda_b200.o -L$(PKG) -lsaberlda \
	    -Wl,-rpath,'$$ORIGIN'

$(BUILD)/cli.o: $(CSRC)/cli.cpp $(CSRC)/sparselda_b200.hpp include/saberlda.h | $(BUILD)
	$(CXX) $(CXXFLAGS) -c $< -o $@

# The reference CLI's replacement (proj/tools/main.cpp): train / eval / topics.
$(CLI): $(BUILD)/cli.o $(BUILD)/sparselda_b200.o $(LIB)
	$(CXX) -o $@ $(BUILD)/cli.o $(BUILD)/sparselda_b200.o -L$(PKG) -lsaberlda -Wl,-rpath,'$$ORIGIN'

$(BUILD)/compat.o: $(CSRC)/compat.cpp $(wildcard $(PKG)/compat/sparselda/*.hpp) $(CSRC)/sparselda_b200.hpp include/saberlda.h | $(BUILD)
	$(CXX) $(CXXFLAGS) -I$(CSRC) -I$(PKG)/compat -c $< -o $@

$(COMPAT): $(BUILD)/compat.o $(BUILD)/sparselda_b200.o $(LIB)
	$(CXX) -shared -o $@ $(BUILD)/compat.o $(BUILD)/sparselda_b200.o -L$(PKG) -lsaberlda -Wl,-rpath,'$$ORIGIN' \
	    -Wl,-soname=libsparselda_compat.so

oracle:
	$(MAKE) -C oracle all
	if [ -d /root/reference/proj ]; then $(MAKE) -C oracle ref; fi

clean:
	rm -rf $(BUILD) $(LIB) $(PKG)/_core*.so $(CLI)

.PHONY: all oracle clean
