# Builds the product library and the oracle (test infrastructure).
#   make            -> paper_2605_16182_b200/lib/libtimewalk_b200.so + oracle
#   make lib        -> product only
NVCC     ?= nvcc
ARCH     := -gencode arch=compute_100a,code=sm_100a
CSRC     := paper_2605_16182_b200/csrc
SRCS     := $(wildcard $(CSRC)/*.cu)
HDRS     := $(wildcard $(CSRC)/*.cuh) include/twg.h
OBJDIR   := build/obj
OBJS     := $(patsubst $(CSRC)/%.cu,$(OBJDIR)/%.o,$(SRCS)) $(OBJDIR)/host_timewalk_facade.o
CXXHDRS  := $(wildcard include/timewalk/*.hpp) include/twg.h
LIB      := paper_2605_16182_b200/lib/libtimewalk_b200.so
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Iinclude -Xcompiler -fPIC,-fopenmp,-O3 \
            --fmad=false -Xptxas -warn-spills --expt-relaxed-constexpr

.PHONY: all lib oracle clean facade_test
all: lib oracle facade_test

lib: $(LIB)

$(OBJDIR)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@

# drop-in C++ façade (the reference's public API, C++20 like proj/core)
$(OBJDIR)/host_timewalk_facade.o: $(CSRC)/host/timewalk_facade.cpp $(CXXHDRS)
	@mkdir -p $(OBJDIR)
	g++ -std=c++20 -O2 -fPIC -Wall -Wextra -Iinclude -c $< -o $@

$(LIB): $(OBJS)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -Xcompiler -fopenmp -lgomp -ldl

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB)

# C++ drop-in check: the reference's API compiled against include/timewalk and linked to the library
FACADE_TEST := build/facade_test
facade_test: $(FACADE_TEST)
$(FACADE_TEST): tests/cpp/facade_test.cpp $(CXXHDRS) $(LIB)
	@mkdir -p build
	g++ -std=c++20 -O2 -Wall -Wextra -pthread -Iinclude $< -o $@ -L$(dir $(LIB)) -ltimewalk_b200 -Wl,-rpath,'$$ORIGIN/../$(dir $(LIB))'

# The reference's OWN test suites (proj/tests/test_*.cpp + acceptance.cpp),
# compiled UNCHANGED from where they lie under /root/reference (needs it at
# build time; the binaries travel to the GPU box):
#   build/ref_suites/gpu/<t>  against include/timewalk + libtimewalk_b200.so (the drop-in)
#   build/ref_suites/cpu/<t>  against the reference core itself (oracle/_ref objects):
#                             pins the doctest shim (every suite must pass there)
REF        ?= /root/reference
REF_TESTS  := $(REF)/proj/tests
SUITES     := test_primitives test_rng test_samplers test_edge_store test_window test_walk_engine \
              test_validity test_io test_replay test_synthetic acceptance
HAVE_REF_TESTS := $(shell test -d $(REF_TESTS) && echo 1)
SHIM       := tests/cpp/doctest_shim
.PHONY: ref_suites
ref_suites: $(if $(HAVE_REF_TESTS),$(addprefix build/ref_suites/gpu/,$(SUITES)) $(addprefix build/ref_suites/cpu/,$(SUITES)))

build/ref_suites/gpu/%: $(REF_TESTS)/%.cpp $(SHIM)/doctest.h $(CXXHDRS) $(LIB)
	@mkdir -p $(dir $@)
	g++ -std=c++20 -O2 -I$(SHIM) -Iinclude $< -o $@ -L$(dir $(LIB)) -ltimewalk_b200 \
	    -Wl,-rpath,'$$ORIGIN/../../../$(dir $(LIB))'

build/ref_suites/cpu/%: $(REF_TESTS)/%.cpp $(SHIM)/doctest.h oracle/_ref/libtimewalk_ref.so
	@mkdir -p $(dir $@)
	g++ -std=c++20 -O2 -fopenmp -I$(SHIM) -I$(REF)/proj/core/include $< -o $@ oracle/_ref/obj/*.o
