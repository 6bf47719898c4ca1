// Host launchers of the fast row kernels (zq_rowops.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace zq {
int launch_tok_quant(const float* x, int64_t rows, int64_t cols, int64_t ld_x, int qm, int8_t* q,
                     int64_t ld_q, float* scales, int32_t* flag, cudaStream_t st);
int launch_ln_quant_uniform(const float* x, const float* res, const float* gamma, const float* beta,
                            int64_t rows, int64_t cols, int nleaves, int leaf_len, float eps,
                            int qm, float* ln_out, int8_t* q, int64_t ld_q, float* scales,
                            int32_t* flag, cudaStream_t st);
int launch_gelu_quant(const float* x, int64_t rows, int64_t cols, int64_t ld_x, int qm, int8_t* q,
                      int64_t ld_q, float* scales, int32_t* flag, cudaStream_t st);
void launch_gelu_estimate(const float* x, int64_t n, float* est, float* bound, cudaStream_t st);
}  // namespace zq
