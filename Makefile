# Builds the C-ABI library for sm_100a (B200) in-tree so it travels with the
# repo snapshot to the GPU box. No GPU is needed to build.
NVCC     ?= nvcc
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -Xptxas -v --expt-relaxed-constexpr
SRC_DIR  := paper_2504_18658_b200/csrc
LIB      := paper_2504_18658_b200/lib/libpccl_b200.so
SRCS     := $(SRC_DIR)/pccl_b200.cu
HDRS     := $(SRC_DIR)/device.cuh $(SRC_DIR)/kernels.cuh include/pccl_b200.h

all: $(LIB)

$(LIB): $(SRCS) $(HDRS)
	@mkdir -p $(dir $(LIB))
	$(NVCC) $(ARCH) $(NVFLAGS) -shared -o $@ $(SRCS) 2> $(SRC_DIR)/../lib/ptxas.log || (cat $(SRC_DIR)/../lib/ptxas.log; false)

sass: $(LIB)
	cuobjdump -sass $(LIB) > $(SRC_DIR)/../lib/libpccl_b200.sass

clean:
	rm -f $(LIB)

.PHONY: all clean sass
