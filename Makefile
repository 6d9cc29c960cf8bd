# Build of the B200 function-execution path.
#   make            -> paper_2303_05601_b200/_lib/libgpufaas_b200.so (host C++ + sm_100a CUDA)
#   make oracle     -> oracle/_build/liboracle.so (test-only C restatement)
#   make ref        -> oracle/_ref/* (unmodified reference, compiled in place; test-only)
# No -ffast-math and -ffp-contract=off on host code: the control plane's double
# arithmetic must match the reference bit for bit.

JSONDIR ?= /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann
CUDA    ?= /usr/local/cuda
NVCC    := $(CUDA)/bin/nvcc
CXX     ?= g++
PKG     := paper_2303_05601_b200
OUT     := $(PKG)/_lib
OBJ     := build/obj
ARCH    := -gencode arch=compute_100a,code=sm_100a
INC     := -Iinclude -I$(PKG)/csrc/host -I$(PKG)/csrc/device -I$(JSONDIR)
CXXFLAGS := -std=c++20 -O2 -fPIC -ffp-contract=off -Wall -Wextra $(INC) -I$(CUDA)/include
NVFLAGS  := -std=c++20 -O3 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -ffp-contract=off \
            --expt-relaxed-constexpr -Xptxas -v $(INC)

ifeq ($(K2_DEBUG),1)
NVFLAGS += -DGFX_K2_DEBUG   # BERT GEMM per-CTA phase tables (debug only, never shipped)
endif
ifeq ($(K5_DEBUG),1)
NVFLAGS += -DGFX_K5_DEBUG   # encoder dataflow kernel per-item timeline (debug only, never shipped)
endif
ifeq ($(K1_DEBUG),1)
NVFLAGS += -DGFX_K1_DEBUG $(K1_EXTRA)   # K1 wait watchdogs + phase marks (debug only, never shipped)
endif

HOST_SRCS := $(wildcard $(PKG)/csrc/host/*.cpp) $(wildcard $(PKG)/csrc/capi/*.cpp)
CU_SRCS   := $(wildcard $(PKG)/csrc/device/*.cu) $(wildcard $(PKG)/csrc/capi/*.cu)
HOST_OBJS := $(patsubst $(PKG)/csrc/%.cpp,$(OBJ)/%.o,$(HOST_SRCS))
CU_OBJS   := $(patsubst $(PKG)/csrc/%.cu,$(OBJ)/%.cu.o,$(CU_SRCS))
HDRS      := $(wildcard include/*.h include/gpufaas/*.hpp $(PKG)/csrc/*/*.hpp $(PKG)/csrc/*/*.cuh)

.PHONY: all product oracle ref clean FORCE
all: product
product: $(OUT)/libgpufaas_b200.so $(OUT)/gfx_managerd

# Rebuild everything when the compiler flags change (e.g. K1_DEBUG=1 <-> release).
$(OBJ)/.flags: FORCE
	@mkdir -p $(OBJ)
	@echo '$(NVFLAGS) $(CXXFLAGS)' | cmp -s - $@ || echo '$(NVFLAGS) $(CXXFLAGS)' > $@

$(OBJ)/%.o: $(PKG)/csrc/%.cpp $(HDRS) $(OBJ)/.flags
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(OBJ)/%.cu.o: $(PKG)/csrc/%.cu $(HDRS) $(OBJ)/.flags
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.ptxas.txt || (cat $@.ptxas.txt; false)

$(OUT)/libgpufaas_b200.so: $(HOST_OBJS) $(CU_OBJS)
	@mkdir -p $(OUT)
	$(NVCC) -shared $(ARCH) -cudart static -o $@ $^ -lpthread -ldl -lrt

# The per-GPU manager daemon (N1), linked against the library next to it.
$(OUT)/gfx_managerd: $(PKG)/csrc/daemon/managerd.cpp $(OUT)/libgpufaas_b200.so include/gpufaas_b200.h
	$(CXX) -std=c++20 -O2 -Wall -Iinclude $< -o $@ -L$(OUT) -lgpufaas_b200 -Wl,-rpath,'$$ORIGIN'

oracle:
	$(MAKE) -C oracle oracle

ref:
	$(MAKE) -C oracle ref

clean:
	rm -rf build $(OUT)
