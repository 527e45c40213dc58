# Builds the product library and the oracle (test infrastructure).
#   make            -> paper_2605_16182_b200/lib/libtimewalk_b200.so + oracle
#   make lib        -> product only
NVCC     ?= nvcc
ARCH     := -gencode arch=compute_100a,code=sm_100a
CSRC     := paper_2605_16182_b200/csrc
SRCS     := $(wildcard $(CSRC)/*.cu)
HDRS     := $(wildcard $(CSRC)/*.cuh) include/twg.h
OBJDIR   := build/obj
OBJS     := $(patsubst $(CSRC)/%.cu,$(OBJDIR)/%.o,$(SRCS))
LIB      := paper_2605_16182_b200/lib/libtimewalk_b200.so
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Iinclude -Xcompiler -fPIC,-fopenmp,-O3 \
            --fmad=false -Xptxas -warn-spills --expt-relaxed-constexpr

.PHONY: all lib oracle clean
all: lib oracle

lib: $(LIB)

$(OBJDIR)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -Xcompiler -fopenmp -lgomp

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB)
