# Builds the product library (sm_100a) and the parity checker.
#   make            -> paper_2506_19852_b200/lib/libradial_cuda.so + oracle
#   make lib        -> CUDA library only
#   make debug      -> diagnostics library (tcgen05 / pipe microbenchmarks, scripts/ only)
#   make cli        -> paper_2506_19852_b200/lib/radial_cli (native mask / stats / bench CLI)
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
CSRC := paper_2506_19852_b200/csrc
SRCS := $(CSRC)/radial_cuda.cu $(CSRC)/mask_build.cu $(CSRC)/attn_fwd.cu $(CSRC)/attn_fwd2.cu $(CSRC)/attn_bwd.cu
HDRS := $(CSRC)/mask_rule.cuh $(CSRC)/sm100.cuh $(CSRC)/radial_internal.h include/radial_cuda.h
LIB := paper_2506_19852_b200/lib/libradial_cuda.so
DEBUG_LIB := paper_2506_19852_b200/lib/libradial_debug.so
CLI := paper_2506_19852_b200/lib/radial_cli
OBJDIR := build/obj
OBJS := $(patsubst $(CSRC)/%.cu,$(OBJDIR)/%.o,$(SRCS))

all: lib debug cli oracle

lib: $(LIB)

debug: $(DEBUG_LIB)

cli: $(CLI)

$(CLI): tools/radial_cli.cpp $(LIB) include/radial/*.hpp include/radial_cuda.h
	g++ -std=c++20 -O2 -Wall -Iinclude -o $@ tools/radial_cli.cpp -L$(dir $(LIB)) -lradial_cuda -Wl,-rpath,'$$ORIGIN'

$(OBJDIR)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $@.ptxas.log || (cat $@.ptxas.log; exit 1)

$(LIB): $(OBJS)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)

# diagnostics only (never loaded by the product path); links the product library for the
# shared tensor-map helper
$(DEBUG_LIB): $(OBJDIR)/debug_mma.o $(LIB)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJDIR)/debug_mma.o -L$(dir $(LIB)) -lradial_cuda -Xlinker -rpath,'$$ORIGIN'

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB) $(DEBUG_LIB) $(CLI)
	$(MAKE) -C oracle clean

.PHONY: all lib debug cli oracle clean

# kernel-variant libraries for tuning sweeps: make variant V=poly2 DEFS="-DRADIAL_POLY_PAIRS=2"
variant:
	@mkdir -p variants/$(V)
	$(NVCC) $(NVFLAGS) $(DEFS) -shared -o variants/$(V)/libradial_cuda.so $(SRCS) 2> variants/$(V)/ptxas.log || (cat variants/$(V)/ptxas.log; exit 1)
