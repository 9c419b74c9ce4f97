# Builds the unmodified reference (offsim) from its own sources under $(REF)
# with g++ directly (its CMake build is not used): the static core, the
# C-ABI shared library, the reference acceptance binary, and the parity dump
# driver (tests/parity/offsim_dump.cpp, repo code) linked against the
# reference core. Output only into $(OUT).
CXX      ?= g++
CXXFLAGS := -std=c++20 -O2 -fPIC -I$(REF)/include -I$(JSONDIR)
SRCS     := workload hardware presets cost_model planner task_graph simulator \
            trace_checks trace_export capacity scenario runner
OBJS     := $(addprefix $(OUT)/obj/,$(addsuffix .o,$(SRCS)))

all: $(OUT)/liboffsim_ref.so $(OUT)/offsim_acceptance $(OUT)/offsim_dump_ref

$(OUT)/obj/%.o: $(REF)/src/%.cpp
	@mkdir -p $(OUT)/obj
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(OUT)/liboffsim_core.a: $(OBJS)
	ar rcs $@ $^

# C-ABI oracle (the reference's liboffsim.so, renamed so it can never be
# mistaken for the product library).
$(OUT)/liboffsim_ref.so: $(REF)/src/capi.cpp $(OUT)/liboffsim_core.a
	$(CXX) $(CXXFLAGS) -shared -Wl,-soname,liboffsim_ref.so $< $(OUT)/liboffsim_core.a -pthread -o $@

$(OUT)/offsim_acceptance: $(REF)/tests/acceptance/acceptance_main.cpp $(OUT)/liboffsim_core.a
	$(CXX) $(CXXFLAGS) $< $(OUT)/liboffsim_core.a -pthread -o $@

$(OUT)/offsim_dump_ref: $(TESTS)/parity/offsim_dump.cpp $(OUT)/liboffsim_core.a
	$(CXX) $(CXXFLAGS) $< $(OUT)/liboffsim_core.a -pthread -o $@

.PHONY: all

# Reference unit suites (unmodified sources) on the doctest shim, linked
# against the reference core: calibrates the shim (must pass 100%).
UNIT := $(REF)/tests/main.cpp $(addprefix $(REF)/tests/test_,$(addsuffix .cpp,workload hardware cost_model planner sim capacity scenario))
SHIM := -I$(TESTS)/parity/doctest_shim

all: $(OUT)/ref_unit_tests $(OUT)/ref_capi_tests

$(OUT)/ref_unit_tests: $(UNIT) $(OUT)/liboffsim_core.a $(TESTS)/parity/doctest_shim/doctest.h
	$(CXX) $(CXXFLAGS) $(SHIM) $(UNIT) $(OUT)/liboffsim_core.a -pthread -o $@

$(OUT)/ref_capi_tests: $(REF)/tests/test_capi.cpp $(OUT)/liboffsim_ref.so $(TESTS)/parity/doctest_shim/doctest.h
	$(CXX) $(CXXFLAGS) $(SHIM) $< -L$(OUT) -loffsim_ref -Wl,-rpath,'$$ORIGIN' -o $@
