# Build for libhx_b200.so (sm_100a CUDA kernels + C-ABI), the helix C++ host
# library and the CPU oracle.  `make` = everything buildable here (nvcc
# cross-compiles sm_100a without a GPU).
NVCC      ?= nvcc
CXX       ?= g++
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O2 --expt-relaxed-constexpr
PKG       := paper_2512_11135_b200
CU_DIR    := $(PKG)/csrc/cuda
CU_SRCS   := $(CU_DIR)/hx_ntt.cu $(CU_DIR)/hx_ops.cu $(CU_DIR)/hx_bsgs.cu
CU_HDRS   := $(wildcard $(CU_DIR)/*.cuh) $(CU_DIR)/hx_internal.h include/hx_b200.h
BUILD     := build
CU_OBJS   := $(patsubst $(CU_DIR)/%.cu,$(BUILD)/%.o,$(CU_SRCS))
LIB       := $(PKG)/libhx_b200.so

.PHONY: all lib oracle ref clean
all: lib oracle

lib: $(LIB)

$(BUILD)/%.o: $(CU_DIR)/%.cu $(CU_HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -Iinclude -c $< -o $@

$(LIB): $(CU_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(CU_OBJS) -lcudart

oracle:
	$(MAKE) -C oracle all

ref:
	$(MAKE) -C oracle ref

clean:
	rm -rf $(BUILD) $(LIB)
	$(MAKE) -C oracle clean
