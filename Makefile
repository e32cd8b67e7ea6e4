# Builds libps.so (sm_100a) and the CPU oracle.  __graft_entry__.build() runs `make -j4`.
# The kernels compile in thirteen translation units (C-ABI, one per dtype/contract for the
# streaming kernels, one per dtype/contract/depth for the fused kernels) so a parallel make
# is bounded by the slowest single unit.
NVCC ?= /usr/local/cuda/bin/nvcc
NVFLAGS = -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo \
          -Xcompiler -fPIC -Xcompiler -Wall -Iinclude
CSRC = paper_1904_04048_b200/csrc
OBJDIR = build/obj
KERN = f64 f32r f32n
# (longest units first: a parallel make starts them in this order)
UNITS = ps_kern_f64_t5 ps_kern_f64_t6 ps_kern_f64_t4 ps_kern_f64_t3 ps_kern_f32r_t4 ps_kern_f32n_t4 \
        $(foreach k,$(KERN),ps_kern_$(k)_t2) ps_kern_f32r_t3 ps_kern_f32n_t3 \
        $(foreach k,$(KERN),ps_kern_$(k)) ps_device
OBJS = $(addprefix $(OBJDIR)/,$(addsuffix .o,$(UNITS)))
HDR = include/ps.h $(wildcard $(CSRC)/*.cuh)

all: paper_1904_04048_b200/libps.so build/fp64_probe oracle

$(OBJDIR)/%.o: $(CSRC)/%.cu $(HDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $<

paper_1904_04048_b200/libps.so: $(OBJS)
	$(NVCC) -shared -gencode arch=compute_100a,code=sm_100a -o $@ $(OBJS)

# compute-roofline probe (FP64 add / FP32 fma rates) run by bench.py
build/fp64_probe: tools/fp64_probe.cu
	@mkdir -p build
	$(NVCC) -O3 -gencode arch=compute_100a,code=sm_100a -o $@ $<

# issue-slot probe (does an FP64 instruction leave room for others?): profiles/r02_issue_probe.jsonl
build/issue_probe: tools/issue_probe.cu
	@mkdir -p build
	$(NVCC) -O3 -gencode arch=compute_100a,code=sm_100a -o $@ $<

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf $(OBJDIR) paper_1904_04048_b200/libps.so
	$(MAKE) -C oracle clean
.PHONY: all oracle clean
