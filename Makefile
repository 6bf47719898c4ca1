# Build the C-ABI library in-tree (it travels to the GPU box with the snapshot).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
PKG := paper_2206_01861_b200
SRC := $(PKG)/csrc/zq_quant.cu $(PKG)/csrc/zq_gemm.cu $(PKG)/csrc/zq_rowops.cu $(PKG)/csrc/zq_attention.cu $(PKG)/csrc/zq_decode.cu $(PKG)/csrc/zq_calib.cu $(PKG)/csrc/zq_gemm_conv.cu
HDR := include/zq_b200.h $(PKG)/csrc/zq_common.cuh $(PKG)/csrc/zq_gelu.cuh $(PKG)/csrc/zq_rowops.h $(PKG)/csrc/zq_gemm.cuh
# -fmad=false: no FMA contraction anywhere (bit-exact numpy arithmetic); the
# exactness-critical ops additionally use explicit _rn intrinsics.
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC -Iinclude \
           -Xptxas -v --expt-relaxed-constexpr

LIB := $(PKG)/libzq_b200.so

all: $(LIB)

$(PKG)/build/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p $(PKG)/build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(PKG)/build/$*.ptxas.log || (cat $(PKG)/build/$*.ptxas.log; false)

$(LIB): $(PKG)/build/zq_quant.o $(PKG)/build/zq_gemm.o $(PKG)/build/zq_rowops.o $(PKG)/build/zq_attention.o $(PKG)/build/zq_decode.o $(PKG)/build/zq_calib.o $(PKG)/build/zq_gemm_conv.o
	$(NVCC) $(ARCH) -shared -o $@ $^ -lcudart_static -lrt -ldl -lpthread

clean:
	rm -rf $(PKG)/build $(LIB)

.PHONY: all clean
