# Build for libhx_b200.so (sm_100a CUDA kernels + C-ABI), the helix C++ host
# library libhelix_b200.so above it, the CPU oracle and the C++ test driver.
# `make` = everything buildable here (nvcc cross-compiles sm_100a without a GPU).
NVCC      ?= nvcc
CXX       ?= g++
CUDA_HOME ?= /usr/local/cuda
JSON_DIR  ?= /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O2 --expt-relaxed-constexpr
CXXFLAGS  := -std=c++20 -O2 -fPIC -Wall -Wextra -Wno-unused-parameter -Iinclude -I$(CUDA_HOME)/include -I$(JSON_DIR)
PKG       := paper_2512_11135_b200
CU_DIR    := $(PKG)/csrc/cuda
HOST_DIR  := $(PKG)/csrc/host
CU_SRCS   := $(CU_DIR)/hx_ntt.cu $(CU_DIR)/hx_ops.cu $(CU_DIR)/hx_bsgs.cu $(CU_DIR)/hx_bsgs_tc.cu $(CU_DIR)/hx_bsgs_p40.cu $(CU_DIR)/hx_encode.cu
CU_HDRS   := $(wildcard $(CU_DIR)/*.cuh) $(CU_DIR)/hx_internal.h include/hx_b200.h
HOST_SRCS := $(HOST_DIR)/params.cpp $(HOST_DIR)/encoder.cpp $(HOST_DIR)/gpu_backend.cpp \
             $(HOST_DIR)/packing.cpp $(HOST_DIR)/linalg.cpp $(HOST_DIR)/helix_c.cpp $(HOST_DIR)/lattice.cpp \
             $(HOST_DIR)/roofline.cpp
HOST_HDRS := $(wildcard include/helix/*.hpp) include/helix_c.h include/hx_b200.h
BUILD     := build
CU_OBJS   := $(patsubst $(CU_DIR)/%.cu,$(BUILD)/%.o,$(CU_SRCS))
HOST_OBJS := $(patsubst $(HOST_DIR)/%.cpp,$(BUILD)/host_%.o,$(HOST_SRCS))
LIB       := $(PKG)/libhx_b200.so
HLIB      := $(PKG)/libhelix_b200.so
TESTBIN   := $(BUILD)/test_linalg_clear

.PHONY: all lib host oracle ref testbin testgpu cli clean
all: lib host oracle testbin testgpu cli

lib: $(LIB)
host: $(HLIB)

$(BUILD)/%.o: $(CU_DIR)/%.cu $(CU_HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -Iinclude -c $< -o $@

$(LIB): $(CU_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(CU_OBJS) -lcudart

$(BUILD)/host_%.o: $(HOST_DIR)/%.cpp $(HOST_HDRS)
	@mkdir -p $(BUILD)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(HLIB): $(HOST_OBJS) $(LIB)
	$(CXX) -shared -o $@ $(HOST_OBJS) -L$(PKG) -lhx_b200 -L$(CUDA_HOME)/lib64 -lcudart \
	  -Wl,-rpath,'$$ORIGIN' -Wl,-rpath,$(CUDA_HOME)/lib64

# C++ test driver: the SPEC linear-algebra kernels on the reference's own
# cleartext ReferenceBackend (its source compiled from the reference tree
# against our API-compatible headers; only where /root/reference exists)
REF_PROJ  ?= /root/reference/proj
$(TESTBIN): tests/cpp/test_linalg_clear.cpp $(HOST_DIR)/packing.cpp $(HOST_DIR)/params.cpp $(HOST_DIR)/linalg.cpp \
            $(HOST_HDRS)
	@mkdir -p $(BUILD)
	@if [ -f $(REF_PROJ)/src/reference_backend.cpp ]; then \
	  $(CXX) -std=c++20 -O2 -Wall -Iinclude -I$(REF_PROJ)/include -I$(JSON_DIR) -DHELIX_NO_GPU \
	    tests/cpp/test_linalg_clear.cpp $(REF_PROJ)/src/reference_backend.cpp $(HOST_DIR)/packing.cpp \
	    $(HOST_DIR)/params.cpp $(HOST_DIR)/linalg.cpp -o $@; \
	else echo "testbin: $(REF_PROJ) absent, skipped"; fi

testbin: $(TESTBIN)

# C++ reference-style caller linked with the B200 library (run on the GPU by
# tests/test_gpu_cpp_api.py); cross-compiles here, needs a B200 to run
GPUTEST   := $(BUILD)/test_gpu_api
$(GPUTEST): tests/cpp/test_gpu_api.cpp $(HLIB) $(HOST_HDRS)
	@mkdir -p $(BUILD)
	$(CXX) -std=c++20 -O2 -Wall -Iinclude -I$(CUDA_HOME)/include -I$(JSON_DIR) tests/cpp/test_gpu_api.cpp \
	  -o $@ -L$(PKG) -lhelix_b200 -lhx_b200 -L$(CUDA_HOME)/lib64 -lcudart \
	  -Wl,-rpath,'$$ORIGIN/../$(PKG)' -Wl,-rpath,$(CUDA_HOME)/lib64

testgpu: $(GPUTEST)

# `helix` command line: roofline / matvec / matmul
CLI       := $(BUILD)/helix
$(CLI): $(HOST_DIR)/cli.cpp $(HLIB) $(HOST_HDRS)
	@mkdir -p $(BUILD)
	$(CXX) -std=c++20 -O2 -Wall -Iinclude -I$(CUDA_HOME)/include -I$(JSON_DIR) $(HOST_DIR)/cli.cpp \
	  -o $@ -L$(PKG) -lhelix_b200 -lhx_b200 -L$(CUDA_HOME)/lib64 -lcudart \
	  -Wl,-rpath,'$$ORIGIN/../$(PKG)' -Wl,-rpath,$(CUDA_HOME)/lib64

cli: $(CLI)

oracle:
	$(MAKE) -C oracle all

ref:
	$(MAKE) -C oracle ref

clean:
	rm -rf $(BUILD) $(LIB) $(HLIB)
	$(MAKE) -C oracle clean
