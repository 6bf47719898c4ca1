// Shared pieces of the tcgen05 GEMM kernels (zq_gemm.cu, zq_gemm_conv.cu):
// tile constants, launch parameters, rasterisation, and the exact dequant
// epilogue chunk writers.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "zq_common.cuh"

namespace zq {

constexpr int BLOCK_M = 128;
constexpr int BLOCK_K = 128;
constexpr int kNumEpiWarps = 8;

enum OutKind { OUT_S32 = 0, OUT_F32 = 1, OUT_F16 = 2, OUT_BF16 = 3 };

struct GemmParams {
  int M, N, K;
  int num_n_tiles, num_tiles, num_k_blocks;
  void* out;
  int64_t ld_out;
  const float* token_scales;  // nullable -> static_scale
  float static_scale;
  const float* row_scales;    // per output channel (nullable for OUT_S32)
  const float* bias;          // nullable
  const uint8_t* w4;          // packed int4 weights (W4 path), row stride ld_w4 bytes
  int64_t ld_w4;
  int tma_out;                // output tensor map valid -> staged TMA stores
  unsigned long long* trace;  // diagnostics: per-CTA %globaltimer stamps (nullable)
  int debug;                  // diagnostics: 1 = skip global stores, 2 = skip dequant math
  int group_m;                // tile rasterisation group (1 = row-major)
  // decode QKV (skinny path, one row per sequence): columns [dl, 2 dl) / [2 dl, 3 dl)
  // of row m are also written to kc / vc[m, kv_pos[m], :] (the KV cache append)
  float* kc;
  float* vc;
  const int32_t* kv_pos;
  int kv_dl;
  int64_t kv_max_ctx;
  // decode stream-K (skinny, W8): zero-initialised int32 workspace of per-tile
  // partial sums, left zeroed by every launch (nullable)
  int32_t* sk_ws;
  int64_t sk_ws_bytes;
  // prefill QKV (CTA-pair path, cache empty): output row r also goes to cache row
  // (r / kv_rows_per_seq) * kv_max_ctx + r % kv_rows_per_seq (0 = off)
  int kv_rows_per_seq;
};

__device__ __forceinline__ void bulk_wait_read1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}

// Grouped tile rasterisation: consecutive tile ids walk kGroupM m-blocks before
// moving to the next n-block, so the ~1 wave of concurrently active tiles covers
// kGroupM x (CTAs / kGroupM) tiles and the A / B panels they share stay in L2
// (row-major order re-read all of B from DRAM once per 2-3 m-blocks: 711 MB of
// DRAM reads for the 128 MB of operands of an 8192^3 GEMM).
// Output-bound GEMMs (small K, e.g. BERT's K = 768) keep plain row-major order
// (group 1: concurrent tiles share output rows, which the f32 stores favour).
__device__ __forceinline__ void tile_coords(int tile, int num_m_tiles, int num_n_tiles, int group_m, int& mt,
                                            int& nt) {
  const int per_group = group_m * num_n_tiles;
  const int g = tile / per_group, r = tile % per_group;
  const int gm = min(group_m, num_m_tiles - g * group_m);
  mt = g * group_m + r % gm;
  nt = r / gm;
}

template <int BN, typename P>
__device__ __forceinline__ int tile_n0(int tile, const P& p) {
  int mt, nt;
  tile_coords(tile, p.num_tiles / p.num_n_tiles, p.num_n_tiles, p.group_m, mt, nt);
  return nt * BN;
}

// Dequantize 32 accumulators of one output row (columns col0..col0+31) in the
// reference's strict order ((f32(acc) * s_tok) * s_w) + bias and write them to
// the warp's staging tile (row = lane) in the TMA swizzle layout:
//   4-byte outputs: 128 B rows, SWIZZLE_128B: chunk c -> (c ^ (r & 7)) * 16
//   2-byte outputs:  64 B rows, SWIZZLE_64B : chunk c -> (c ^ ((r >> 1) & 3)) * 16
// Columns past N read scale/bias as 0 (their values are clipped by the TMA store).
// ACCF: the accumulators are f32 bit patterns (kind::f16 MMAs) instead of int32.
template <bool ACCF>
__device__ __forceinline__ float acc_to_f32(uint32_t r) {
  return ACCF ? __uint_as_float(r) : __int2float_rn((int)r);
}

template <int KIND, bool ACCF = false>
__device__ __forceinline__ void epi_chunk_smem(const uint32_t (&r)[32], float s_tok,
                                               const float* __restrict__ rs,
                                               const float* __restrict__ bias, int col0, int N,
                                               uint8_t* stage, int lane) {
  if (KIND == OUT_S32) {
    uint8_t* rowp = stage + lane * 128;
#pragma unroll
    for (int c = 0; c < 8; ++c)
      *reinterpret_cast<uint4*>(rowp + ((c ^ (lane & 7)) << 4)) =
          make_uint4(r[4 * c], r[4 * c + 1], r[4 * c + 2], r[4 * c + 3]);
    return;
  }
  float f[32];
  const bool full = col0 + 32 <= N;
  if (full) {
    const float4* sw4 = reinterpret_cast<const float4*>(rs + col0);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float4 w = __ldg(sw4 + j);
      // ((acc * s_tok) * s_w) two columns per FMUL2 (the bias add below stays
      // scalar: ptxas would contract an f32x2 multiply-add into one FFMA2)
      const uint64_t st2 = f2splat(s_tok);
      f2unpack(f2mul(f2mul(f2pack(acc_to_f32<ACCF>(r[4 * j + 0]), acc_to_f32<ACCF>(r[4 * j + 1])), st2),
                     f2pack(w.x, w.y)), f[4 * j + 0], f[4 * j + 1]);
      f2unpack(f2mul(f2mul(f2pack(acc_to_f32<ACCF>(r[4 * j + 2]), acc_to_f32<ACCF>(r[4 * j + 3])), st2),
                     f2pack(w.z, w.w)), f[4 * j + 2], f[4 * j + 3]);
    }
    if (bias != nullptr) {
      const float4* b4 = reinterpret_cast<const float4*>(bias + col0);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float4 b = __ldg(b4 + j);
        f[4 * j + 0] = __fadd_rn(f[4 * j + 0], b.x);
        f[4 * j + 1] = __fadd_rn(f[4 * j + 1], b.y);
        f[4 * j + 2] = __fadd_rn(f[4 * j + 2], b.z);
        f[4 * j + 3] = __fadd_rn(f[4 * j + 3], b.w);
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int cc = col0 + j;
      const float w = cc < N ? __ldg(rs + cc) : 0.0f;
      f[j] = __fmul_rn(__fmul_rn(acc_to_f32<ACCF>(r[j]), s_tok), w);
      if (bias != nullptr && cc < N) f[j] = __fadd_rn(f[j], __ldg(bias + cc));
    }
  }
  if (KIND == OUT_F32) {
    uint8_t* rowp = stage + lane * 128;
#pragma unroll
    for (int c = 0; c < 8; ++c)
      *reinterpret_cast<float4*>(rowp + ((c ^ (lane & 7)) << 4)) =
          make_float4(f[4 * c], f[4 * c + 1], f[4 * c + 2], f[4 * c + 3]);
  } else {
    uint32_t h[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (KIND == OUT_F16) {
        __half2 t = __floats2half2_rn(f[2 * j], f[2 * j + 1]);
        h[j] = *reinterpret_cast<uint32_t*>(&t);
      } else {
        __nv_bfloat162 t = __floats2bfloat162_rn(f[2 * j], f[2 * j + 1]);
        h[j] = *reinterpret_cast<uint32_t*>(&t);
      }
    }
    uint8_t* rowp = stage + lane * 64;
#pragma unroll
    for (int c = 0; c < 4; ++c)
      *reinterpret_cast<uint4*>(rowp + ((c ^ ((lane >> 1) & 3)) << 4)) =
          make_uint4(h[4 * c], h[4 * c + 1], h[4 * c + 2], h[4 * c + 3]);
  }
}

// Ragged edge (N tail or unaligned output): element-wise, guarded.
template <int KIND, bool ACCF = false>
__device__ __forceinline__ void epi_chunk_slow(const uint32_t (&r)[32], float s_tok,
                                            const float* __restrict__ rs,
                                            const float* __restrict__ bias, void* out,
                                            int64_t row_off, int col0, int N) {
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const int c = col0 + j;
    if (c < N) {
      if (KIND == OUT_S32) {
        reinterpret_cast<int32_t*>(out)[row_off + c] = (int)r[j];
      } else {
        float f = __fmul_rn(__fmul_rn(acc_to_f32<ACCF>(r[j]), s_tok), rs[c]);
        if (bias) f = __fadd_rn(f, bias[c]);
        if (KIND == OUT_F32) reinterpret_cast<float*>(out)[row_off + c] = f;
        else if (KIND == OUT_F16) reinterpret_cast<__half*>(out)[row_off + c] = __float2half_rn(f);
        else reinterpret_cast<__nv_bfloat16*>(out)[row_off + c] = __float2bfloat16_rn(f);
      }
    }
  }
}

// host: 2-D tensor map over a row-major matrix (ld in bytes); defined in zq_gemm.cu
int make_tmap_2d(CUtensorMap* tm, CUtensorMapDataType dt, const void* base, int64_t rows, int64_t cols,
                 int64_t ld_bytes, int box_cols, int box_rows, CUtensorMapSwizzle sw,
                 CUtensorMapL2promotion promo);

}  // namespace zq
