# Build the sm_100a engine (C-ABI shared library).  One translation unit per
# element-kernel mode so instantiations compile in parallel (make -j).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v
PKG := paper_2412_13733_b200
CS := $(PKG)/csrc
OBJDIR := build
SRCS := $(wildcard $(CS)/*.cu)
OBJS := $(patsubst $(CS)/%.cu,$(OBJDIR)/%.o,$(SRCS))
HDR := $(wildcard $(CS)/*.cuh) include/hpg_b200.h

all: $(PKG)/libhpg_b200.so

$(OBJDIR)/%.o: $(CS)/%.cu $(HDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $(OBJDIR)/$*.ptxas.log || (cat $(OBJDIR)/$*.ptxas.log; exit 1)

$(PKG)/libhpg_b200.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)

clean:
	rm -rf $(OBJDIR) $(PKG)/libhpg_b200.so

.PHONY: all clean
