# Builds the product library (sm_100a) and the parity checker.
#   make            -> paper_2506_19852_b200/lib/libradial_cuda.so + oracle
#   make lib        -> CUDA library only
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
CSRC := paper_2506_19852_b200/csrc
SRCS := $(CSRC)/radial_cuda.cu $(CSRC)/mask_build.cu $(CSRC)/attn_fwd.cu $(CSRC)/attn_bwd.cu $(CSRC)/debug_mma.cu
HDRS := $(CSRC)/mask_rule.cuh $(CSRC)/sm100.cuh $(CSRC)/radial_internal.h include/radial_cuda.h
LIB := paper_2506_19852_b200/lib/libradial_cuda.so
OBJDIR := build/obj
OBJS := $(patsubst $(CSRC)/%.cu,$(OBJDIR)/%.o,$(SRCS))

all: lib oracle

lib: $(LIB)

$(OBJDIR)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $@.ptxas.log || (cat $@.ptxas.log; exit 1)

$(LIB): $(OBJS)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB)
	$(MAKE) -C oracle clean

.PHONY: all lib oracle clean

# kernel-variant libraries for tuning sweeps: make variant V=poly2 DEFS="-DRADIAL_POLY_PAIRS=2"
variant:
	@mkdir -p variants/$(V)
	$(NVCC) $(NVFLAGS) $(DEFS) -shared -o variants/$(V)/libradial_cuda.so $(SRCS) 2> variants/$(V)/ptxas.log || (cat variants/$(V)/ptxas.log; exit 1)
