# Product build: paper_2403_06504_b200/lib/liboffsim.so.0 (+ liboffsim.so link)
#   - offsim core (C++20, g++): the API-compatible restatement of the
#     reference's planner / schedule / DES / trace checks / C ABI
#   - B200 executor (CUDA, nvcc, sm_100a only): fused Adam kernels, chunk
#     pipeline, activation-swap copy engine, fy_* C ABI
# `make` builds the library, the parity dump driver and the oracle .so.
NVCC     ?= /usr/local/cuda/bin/nvcc
CXX      ?= g++
PKG      := paper_2403_06504_b200
LIBDIR   := $(PKG)/lib
OBJDIR   := build/obj
JSONDIR  ?= $(shell python3 -c "import os,sysconfig;print(os.path.join(sysconfig.get_paths()['purelib'],'include','cudnn_frontend','thirdparty','nlohmann'))")
ARCH     := -gencode arch=compute_100a,code=sm_100a
CXXFLAGS := -std=c++20 -O2 -fPIC -Wall -Wextra -Iinclude -I$(JSONDIR)
NVFLAGS  := -std=c++17 -O3 $(ARCH) -lineinfo -Xcompiler -fPIC -Iinclude -Xptxas -v

# NCCL: the copy torch ships (2.28.x) when present, so a process that also
# imports torch maps ONE libnccl.so.2; else the system one.
NCCLDIR  ?= $(shell python3 -c "import os,sysconfig;d=os.path.join(sysconfig.get_paths()['purelib'],'nvidia','nccl');print(d if os.path.isfile(os.path.join(d,'include','nccl.h')) else '')")
ifneq ($(NCCLDIR),)
NCCL_INC := -I$(NCCLDIR)/include
NCCL_LNK := -L$(NCCLDIR)/lib -l:libnccl.so.2 -Xlinker -rpath=$(NCCLDIR)/lib
else
NCCL_INC :=
NCCL_LNK := -lnccl
endif
LINK_LIBS := -L/usr/local/cuda/lib64 -lcublas -Xlinker -rpath=/usr/local/cuda/lib64 $(NCCL_LNK)
NVFLAGS  += $(NCCL_INC)

CORE_SRC := $(wildcard $(PKG)/csrc/core/*.cpp)
CUDA_SRC := $(wildcard $(PKG)/csrc/cuda/*.cu)
CORE_OBJ := $(patsubst $(PKG)/csrc/core/%.cpp,$(OBJDIR)/core/%.o,$(CORE_SRC))
CUDA_OBJ := $(patsubst $(PKG)/csrc/cuda/%.cu,$(OBJDIR)/cuda/%.o,$(CUDA_SRC))
HDRS     := $(wildcard include/offsim/*.hpp include/offsim/*.h include/fuyou/*.h) \
            $(wildcard $(PKG)/csrc/core/*.hpp $(PKG)/csrc/cuda/*.cuh)

all: $(LIBDIR)/liboffsim.so sweep $(if $(CORE_SRC),build/offsim_dump build/io_engine_test build/offsim build/graph_dump) oracle

$(OBJDIR)/core/%.o: $(PKG)/csrc/core/%.cpp $(HDRS)
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(OBJDIR)/cuda/%.o: $(PKG)/csrc/cuda/%.cu $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJDIR)/cuda/$*.ptxas.log || (cat $(OBJDIR)/cuda/$*.ptxas.log; false)

build/liboffsim_core.a: $(CORE_OBJ)
	@mkdir -p build
	rm -f $@ && ar rcs $@ $^

$(LIBDIR)/liboffsim.so.0: $(CORE_OBJ) $(CUDA_OBJ)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(ARCH) -shared -Xlinker -soname=liboffsim.so.0 -o $@ $^ -lpthread $(LINK_LIBS)

$(LIBDIR)/liboffsim.so: $(LIBDIR)/liboffsim.so.0
	ln -sf liboffsim.so.0 $@

# Sweep-only build (bench / test tooling, never shipped in $(LIBDIR)): the
# same library with the TMA kernel's experimental variants compiled in
# (-DFY_SWEEP_VARIANTS: tile / split-DMA / cache-hint / no-math probes,
# fy_adamw_tune_bulk). scripts/kernel_sweep.py and the variant test load it.
SWEEP_SRC := adamw_kernels fy_capi
SWEEP_OBJ := $(addprefix build/sweep/,$(addsuffix .o,$(SWEEP_SRC)))
sweep: build/sweep/liboffsim_sweep.so

build/sweep/%.o: $(PKG)/csrc/cuda/%.cu $(HDRS)
	@mkdir -p build/sweep
	$(NVCC) $(NVFLAGS) -DFY_SWEEP_VARIANTS -c $< -o $@ 2> build/sweep/$*.ptxas.log || (cat build/sweep/$*.ptxas.log; false)

build/sweep/liboffsim_sweep.so: $(CORE_OBJ) $(filter-out $(addprefix $(OBJDIR)/cuda/,$(addsuffix .o,$(SWEEP_SRC))),$(CUDA_OBJ)) $(SWEEP_OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $^ -lpthread $(LINK_LIBS)

# Parity driver compiled against this repo's headers + core.
build/offsim_dump: tests/parity/offsim_dump.cpp build/liboffsim_core.a
	$(CXX) $(CXXFLAGS) $< build/liboffsim_core.a -pthread -o $@

# CLI: links the C ABI only (like the reference's offsim CLI)
build/offsim: tools/offsim_main.cpp $(LIBDIR)/liboffsim.so
	@mkdir -p build
	$(CXX) $(CXXFLAGS) $< -L$(LIBDIR) -l:liboffsim.so.0 -Wl,-rpath,'$$ORIGIN/../$(LIBDIR)' -o $@

# mapped task graph (what offsim::execute runs) as JSON, for scripts/critical_path.py
build/graph_dump: tools/graph_dump.cpp build/liboffsim_core.a
	$(CXX) $(CXXFLAGS) $< build/liboffsim_core.a -pthread -o $@

build/io_engine_test: tests/parity/io_engine_test.cpp $(PKG)/csrc/core/io_engine.cpp $(PKG)/csrc/core/io_engine.hpp
	@mkdir -p build
	$(CXX) $(CXXFLAGS) tests/parity/io_engine_test.cpp $(PKG)/csrc/core/io_engine.cpp -o $@

oracle:
	$(MAKE) -C oracle all

# The reference's own unit suites (unmodified, from /root/reference) built
# against THIS repo's headers + core / C ABI through the doctest shim —
# only where the reference sources exist (build container).
REF      ?= /root/reference/proj
REF_UNIT := $(REF)/tests/main.cpp $(addprefix $(REF)/tests/test_,$(addsuffix .cpp,workload hardware cost_model planner sim capacity scenario))
reftests: build/ref_unit_tests_on_b200 build/ref_capi_tests_on_b200 build/ref_acceptance_on_b200

build/ref_unit_tests_on_b200: $(REF_UNIT) build/liboffsim_core.a tests/parity/doctest_shim/doctest.h
	$(CXX) $(CXXFLAGS) -Itests/parity/doctest_shim $(REF_UNIT) build/liboffsim_core.a -pthread -o $@

build/ref_capi_tests_on_b200: $(REF)/tests/test_capi.cpp $(LIBDIR)/liboffsim.so tests/parity/doctest_shim/doctest.h
	$(CXX) $(CXXFLAGS) -Itests/parity/doctest_shim $< -L$(LIBDIR) -l:liboffsim.so.0 -Wl,-rpath,'$$ORIGIN/../$(LIBDIR)' -o $@

build/ref_acceptance_on_b200: $(REF)/tests/acceptance/acceptance_main.cpp build/liboffsim_core.a
	$(CXX) $(CXXFLAGS) $< build/liboffsim_core.a -pthread -o $@

ref:
	$(MAKE) -C oracle ref

clean:
	rm -rf build $(LIBDIR)

.PHONY: all oracle ref reftests sweep clean
