// K6/K7/K8: W8A8 / W4A8 integer GEMM on sm_100a tensor cores (tcgen05 kind::i8)
// with the fused ZeroQuant dequant epilogue.
//
//   acc[i, j] = sum_p xq[i, p] * wq[j, p]            igemm.py:66-80 (exact int32)
//   out[i, j] = ((f32(acc) * s_tok[i]) * s_w[j]) + b[j]   igemm.py:83-112
//
// Persistent, warp-specialised kernel, one CTA per SM:
//   warp 0      TMA producer (one elected lane): A/B K-blocks -> smem ring
//   warp 1      TMEM allocator + MMA issuer (one lane): tcgen05.mma kind::i8
//   warps 2..5  epilogue: tcgen05.ld TMEM -> registers -> dequant -> global
//   warps 6..9  (W4 only) INT4 -> INT8 unpack of the weight tile into the
//               SWIZZLE_128B layout the MMA reads
// Tiles: BLOCK_M = 128 token rows, BLOCK_N output channels (64/128/256),
// BLOCK_K = 128 bytes (one 128B swizzle atom per row).  Accumulators are int32
// in TMEM, double-buffered so the epilogue of tile t overlaps the MMAs of t+1.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <mutex>

#include "zq_gemm.cuh"

namespace zq {

template <int BN, int W4>
struct GemmCfg {
  static constexpr int A_BYTES = BLOCK_M * BLOCK_K;
  static constexpr int B_BYTES = BN * BLOCK_K;
  static constexpr int P_BYTES = W4 ? BN * (BLOCK_K / 2) : 0;  // packed INT4 staging
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES + P_BYTES;
  // per-epilogue-warp output staging: two 32 rows x 32 columns x 4 B buffers
  // (bulk TMA stores of one drain while the other is filled)
  static constexpr int EPI_BYTES = kNumEpiWarps * 2 * 32 * 32 * 4;
  static constexpr int RING = 232448 - EPI_BYTES - 1024 - 256;
  static constexpr int STAGES = RING / STAGE_BYTES > 8 ? 8 : RING / STAGE_BYTES;
  static constexpr int TMEM_COLS = 2 * BN;  // double-buffered int32 accumulators
  static constexpr int NUM_THREADS = (2 + kNumEpiWarps + (W4 ? 4 : 0)) * 32;
  static constexpr int SMEM_BYTES =
      STAGES * STAGE_BYTES + EPI_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};


template <int BN, int KIND, int W4>
__global__ void __launch_bounds__(GemmCfg<BN, W4>::NUM_THREADS, 1)
    zq_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmC, const GemmParams p) {
  using Cfg = GemmCfg<BN, W4>;
  constexpr int STAGES = Cfg::STAGES;
  // no static smem: the dynamic window is 1024-aligned (checked below), and using
  // it without an integer round trip keeps the epilogue staging on LDS/STS
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;                              // STAGES x [128 rows x 128 B]
  uint8_t* sB = smem + STAGES * Cfg::A_BYTES;      // STAGES x [BN rows x 128 B]
  uint8_t* sP = smem + STAGES * (Cfg::A_BYTES + Cfg::B_BYTES);  // W4: STAGES x [BN x 64 B]
  uint8_t* sC = smem + STAGES * Cfg::STAGE_BYTES;  // epilogue staging (1024-aligned)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sC + Cfg::EPI_BYTES);
  uint64_t* full_bar = bars;                        // TMA (+unpack) -> MMA
  uint64_t* empty_bar = bars + STAGES;              // MMA -> TMA (slot free)
  uint64_t* tfull_bar = bars + 2 * STAGES;          // MMA -> epilogue (2)
  uint64_t* tempty_bar = bars + 2 * STAGES + 2;     // epilogue -> MMA (2)
  uint64_t* praw_bar = bars + 2 * STAGES + 4;       // W4: TMA packed weights landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * STAGES + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (p.trace && threadIdx.x == 0) p.trace[(size_t)blockIdx.x * 64] = gtime();
  if (warp == 0 && lane == 0) {
    if (smem_u32(smem) & 1023) __trap();  // SWIZZLE_128B needs 1024-byte aligned stages
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    if (p.tma_out) prefetch_tmap(&tmC);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], W4 ? 1 + 4 : 1);  // W4: + one arrive per unpack warp
      mbar_init(&empty_bar[s], 1);
      if (W4) mbar_init(&praw_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], kNumEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int nkb = p.num_k_blocks;
  unsigned long long* tr = p.trace ? p.trace + (size_t)blockIdx.x * 64 : nullptr;
  if (tr && threadIdx.x == 0) tr[1] = gtime();
  pdl_trigger();
  if (warp == 0) {
    // ===================== TMA producer =====================
    // whole warp walks the loop (keeps the warp converged for the final
    // __syncthreads); lane 0 issues.  The first tile's weight stages are
    // requested before the grid dependency resolves (weights are constant).
    int stage = 0, phase = 0;
    const int pre = (!W4 && (int)blockIdx.x < p.num_tiles) ? (nkb < STAGES ? nkb : STAGES) : 0;
    if (lane == 0)
      for (int kb = 0; kb < pre; ++kb) {
        mbar_arrive_expect_tx(&full_bar[kb], Cfg::STAGE_BYTES);
        tma_load_2d(sB + kb * Cfg::B_BYTES, &tmB, &full_bar[kb], kb * BLOCK_K,
                    tile_n0<BN>(blockIdx.x, p));
      }
    pdl_wait();
    for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
      int mt, nt;
      tile_coords(tile, p.num_tiles / p.num_n_tiles, p.num_n_tiles, p.group_m, mt, nt);
      const int m0 = mt * BLOCK_M;
      const int n0 = nt * BN;
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&empty_bar[stage], phase ^ 1);
        if (lane == 0) {
          if (tile == (int)blockIdx.x && kb < pre) {
            tma_load_2d(sA + stage * Cfg::A_BYTES, &tmA, &full_bar[stage], kb * BLOCK_K, m0);
          } else if (W4) {
            // packed weights -> staging (praw_bar); the unpack warps write the
            // int8 tile and add 4 arrivals on full_bar
            mbar_arrive_expect_tx(&praw_bar[stage], Cfg::P_BYTES);
            tma_load_2d(sP + stage * Cfg::P_BYTES, &tmB, &praw_bar[stage], kb * (BLOCK_K / 2), n0);
            mbar_arrive_expect_tx(&full_bar[stage], Cfg::A_BYTES);
            tma_load_2d(sA + stage * Cfg::A_BYTES, &tmA, &full_bar[stage], kb * BLOCK_K, m0);
          } else {
            mbar_arrive_expect_tx(&full_bar[stage], Cfg::STAGE_BYTES);
            tma_load_2d(sA + stage * Cfg::A_BYTES, &tmA, &full_bar[stage], kb * BLOCK_K, m0);
            tma_load_2d(sB + stage * Cfg::B_BYTES, &tmB, &full_bar[stage], kb * BLOCK_K, n0);
          }
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    constexpr uint32_t idesc = make_idesc_i8(BLOCK_M, BN);
    int stage = 0, phase = 0, acc = 0, acc_phase = 0, lt = 0;
    for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x, ++lt) {
      mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
      tc_fence_after();
      if (tr && lane == 0 && lt < 15) tr[2 + 4 * lt] = gtime();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        if (tr && lane == 0 && lt < 15 && kb == nkb - 1) tr[3 + 4 * lt] = gtime();
        if (lane == 0) {
          const uint32_t a_addr = smem_u32(sA + stage * Cfg::A_BYTES);
          const uint32_t b_addr = smem_u32(sB + stage * Cfg::B_BYTES);
#pragma unroll
          for (int k = 0; k < BLOCK_K / 32; ++k) {
            mma_i8(d_tmem, make_sw128_desc(a_addr + k * 32), make_sw128_desc(b_addr + k * 32),
                   idesc, (kb | k) != 0);
          }
          mma_commit(&empty_bar[stage]);
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (lane == 0) mma_commit(&tfull_bar[acc]);
      __syncwarp();
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  } else if (warp < 2 + kNumEpiWarps) {
    // ===================== epilogue =====================
    // 8 warps: warp%4 selects the TMEM lane quarter (32 rows), (warp-2)/4 the
    // half of the tile's columns.  Per 32x32 chunk: tcgen05.ld -> dequant in
    // registers (thread = row) -> swizzled smem staging -> one TMA store per warp
    // (coalesced, clipped at the M/N edges by the tensor map).
    pdl_wait();  // token scales come from the previous kernel; `out` may still be read by it
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    constexpr int COLS = BN / 2;
    uint8_t* stage_c = sC + (warp - 2) * (2 * 32 * 32 * 4);
    int sbuf = 0;
    int acc = 0, acc_phase = 0, lt = 0;
    const bool stamp = tr && warp == 2 && lane == 0;
    for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x, ++lt) {
      int mt, nt;
      tile_coords(tile, p.num_tiles / p.num_n_tiles, p.num_n_tiles, p.group_m, mt, nt);
      const int m0 = mt * BLOCK_M;
      const int n0 = nt * BN + half * COLS;
      const int row0 = m0 + quarter * 32;
      const int row = row0 + lane;
      float s_tok = p.static_scale;
      if (KIND != OUT_S32 && p.token_scales != nullptr && row < p.M) s_tok = __ldg(p.token_scales + row);
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      if (stamp && lt < 15) tr[4 + 4 * lt] = gtime();
      const uint32_t t_row =
          tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN + half * COLS;
#pragma unroll 1
      for (int c = 0; c < COLS; c += 32) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(t_row + c, r);
        tmem_ld_wait();
        if (c + 32 == COLS) {
          // accumulator fully read: hand the TMEM buffer back to the MMA warp
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty_bar[acc]);
        }
        const int col0 = n0 + c;
        if (row0 >= p.M || col0 >= p.N) continue;  // warp-uniform
        if (p.tma_out) {
          // double-buffered staging (row = lane, swizzled) drained by bulk TMA
          // stores that overlap the next chunk's dequant; the map clips M / N
          uint8_t* sb = stage_c + sbuf * (32 * 32 * 4);
          if (lane == 0) bulk_wait_read1();
          __syncwarp();
          if (!(p.debug & 2)) epi_chunk_smem<KIND>(r, s_tok, p.row_scales, p.bias, col0, p.N, sb, lane);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0 && !(p.debug & 1)) {
            tma_store_2d(&tmC, sb, col0, row0);
            bulk_commit();
          }
          sbuf ^= 1;
        } else if (row < p.M) {
          epi_chunk_slow<KIND>(r, s_tok, p.row_scales, p.bias, p.out, (int64_t)row * p.ld_out,
                               col0, p.N);
        }
      }
      if (stamp && lt < 15) tr[5 + 4 * lt] = gtime();
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (lane == 0) bulk_wait0();
    if (stamp) tr[63] = gtime();
  } else if (W4) {
    // ===================== INT4 -> INT8 unpack (W4A8) =====================
    // 4 warps.  Packed tile (BN rows x 64 B, K-major, unswizzled) -> int8 tile in
    // the SWIZZLE_128B layout the MMA reads: row r, 16-byte chunk c (K elements
    // 16c..16c+15) lives at r*128 + ((c ^ (r & 7)) * 16).  Nibble j of a packed
    // 32-bit word is element j (two's complement), sign-extended with shifts.
    const int ut = threadIdx.x - (2 + kNumEpiWarps) * 32;
    int stage = 0, phase = 0;
    for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&empty_bar[stage], phase ^ 1);
        mbar_wait(&praw_bar[stage], phase);
        const uint8_t* src = sP + stage * Cfg::P_BYTES;
        uint8_t* dst = sB + stage * Cfg::B_BYTES;
#pragma unroll 4
        for (int idx = ut; idx < BN * 8; idx += 128) {
          const int r = idx >> 3, c = idx & 7;
          const uint2 pk = *reinterpret_cast<const uint2*>(src + r * 64 + c * 8);
          uint32_t w[4];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            // SIMD within a register: even / odd nibbles -> bytes, 4-bit sign
            // extension as b | ((b & 8) * 0x1E) per byte (no cross-byte carries),
            // then interleave the bytes back into element order with PRMT
            const uint32_t x = h ? pk.y : pk.x;
            uint32_t ev = x & 0x0F0F0F0Fu, od = (x >> 4) & 0x0F0F0F0Fu;
            ev |= (ev & 0x08080808u) * 0x1Eu;
            od |= (od & 0x08080808u) * 0x1Eu;
            w[2 * h] = __byte_perm(ev, od, 0x5140);      // elements 0..3
            w[2 * h + 1] = __byte_perm(ev, od, 0x7362);  // elements 4..7
          }
          *reinterpret_cast<uint4*>(dst + r * 128 + ((c ^ (r & 7)) * 16)) =
              make_uint4(w[0], w[1], w[2], w[3]);
        }
        fence_proxy_async_smem();  // generic-proxy smem writes -> visible to tcgen05
        __syncwarp();
        if (lane == 0) mbar_arrive(&full_bar[stage]);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
}

// ---------------------------------------------------------------------------
// CTA-pair variant (tcgen05 cta_group::2, int8 weights): a cluster of 2 CTAs
// computes a 256 x BN tile.  CTA r holds A rows [128r, 128r+128) and B rows
// [r*BN/2, (r+1)*BN/2) of the pair tile in its own smem; the leader (r = 0)
// issues M=256 MMAs that read both CTAs' smem and write each CTA's TMEM (its
// 128 rows x BN columns).  Per SM and K-block the smem traffic drops from
// 2 x (16 + BN) KB to 2 x (16 + BN/2) KB, which is what bounds the 1-CTA kernel
// (TMA writes + tensor-core reads share the smem port).
//   full_bar   (leader): 2 arrivals (one per CTA producer) + both CTAs' TMA bytes
//   empty_bar  (each)  : multicast tcgen05.commit from the leader
//   tfull_bar  (each)  : multicast commit after a tile's last MMA
//   tempty_bar (leader): 2 x kNumEpiWarps arrivals (both CTAs' epilogue warps)
// CL = 4: a cluster of two pairs computes a 256 x 2BN unit (pair s = rank >> 1
// takes n-tile 2u + s); the pairs share A, so each A k-block is loaded once and
// multicast to the two CTAs holding those rows (the pairs alternate k-blocks as
// issuer), halving A's L2->SM traffic, which bounds the operand-fed phase.
// Both pairs' MMA commits release every CTA's stage (empty_bar counts 2), so a
// multicast never overwrites a slot the other pair still reads.
// ---------------------------------------------------------------------------
template <int BN>
struct Gemm2Cfg {
  static constexpr int A_BYTES = BLOCK_M * BLOCK_K;
  static constexpr int B_BYTES = (BN / 2) * BLOCK_K;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // two 32x32 output staging buffers per epilogue warp (bulk TMA stores overlap
  // the dequant of the next chunk); the operand ring gets the rest of the 227 KB
  static constexpr int EPI_BYTES = kNumEpiWarps * 2 * 32 * 32 * 4;
  static constexpr int RING = 232448 - EPI_BYTES - 1024 - 256;
  static constexpr int STAGES = RING / STAGE_BYTES > 8 ? 8 : RING / STAGE_BYTES;
  // double-buffered accumulators: 2*BN columns, allocated as a power of two (BN = 192 -> 512)
  static constexpr int TMEM_COLS = 2 * BN <= 256 ? 256 : 512;
  static constexpr int NUM_THREADS = (2 + kNumEpiWarps) * 32;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + EPI_BYTES + 1024 + 256;
};

template <int BN, int KIND, int CL>
__global__ void __launch_bounds__(Gemm2Cfg<BN>::NUM_THREADS, 1)
    zq_gemm2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmKc,
                    const __grid_constant__ CUtensorMap tmVc, const GemmParams p) {
  using Cfg = Gemm2Cfg<BN>;
  constexpr int STAGES = Cfg::STAGES;
  // no static smem: the dynamic window is 1024-aligned (checked below), and using
  // it without an integer round trip keeps the epilogue staging on LDS/STS
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * Cfg::A_BYTES;
  uint8_t* sC = smem + STAGES * Cfg::STAGE_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sC + Cfg::EPI_BYTES);
  uint64_t* full_bar = bars;
  uint64_t* empty_bar = bars + STAGES;
  uint64_t* tfull_bar = bars + 2 * STAGES;
  uint64_t* tempty_bar = bars + 2 * STAGES + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();
  const uint32_t rank = crank & 1;  // rank within the pair
  const bool leader = rank == 0;
  const int sub = CL == 4 ? (int)(crank >> 1) : 0;  // pair within the cluster
  const int unit0 = blockIdx.x / CL, nunits_grid = gridDim.x / CL;
  constexpr int NSUB = CL / 2;
  const int num_m_tiles = p.num_tiles / p.num_n_tiles;
  const int num_nu = (p.num_n_tiles + NSUB - 1) / NSUB;  // n-units
  const int num_units = num_m_tiles * num_nu;
  auto unit_coords = [&](int u, int& mt, int& nt) {
    int ntu;
    tile_coords(u, num_m_tiles, num_nu, p.group_m, mt, ntu);
    nt = ntu * NSUB + sub;
  };
  unsigned long long* tr = p.trace ? p.trace + (size_t)blockIdx.x * 64 : nullptr;
  if (tr && threadIdx.x == 0) tr[0] = gtime();

  if (warp == 0 && lane == 0) {
    if (smem_u32(smem) & 1023) __trap();  // SWIZZLE_128B needs 1024-byte aligned stages
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 2);
      mbar_init(&empty_bar[s], NSUB);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 2 * kNumEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_cg2(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int nkb = p.num_k_blocks;
  if (tr && threadIdx.x == 0) tr[1] = gtime();

  pdl_trigger();
  if (warp == 0) {
    // ===================== TMA producer (both CTAs) =====================
    // weight halves of the first tile's stages go out before the grid dependency
    int stage = 0, phase = 0;
    const int pre = unit0 < num_units ? (nkb < STAGES ? nkb : STAGES) : 0;
    // CL = 4: this CTA loads (and multicasts) A for k-blocks kb with kb % 2 == sub
    const uint16_t amask = (uint16_t)((1u << rank) | (1u << (rank + 2)));
    auto load_a = [&](int st_, int kb, int m0, uint32_t fb) {
      if (CL == 2)
        tma_load_2d_cg2(sA + st_ * Cfg::A_BYTES, &tmA, fb, kb * BLOCK_K, m0);
      else if ((kb & 1) == sub)
        tma_load_2d_cg2_mc(sA + st_ * Cfg::A_BYTES, &tmA, fb, kb * BLOCK_K, m0, amask);
    };
    if (lane == 0 && pre) {
      int mt, nt;
      unit_coords(unit0, mt, nt);
      for (int kb = 0; kb < pre; ++kb) {
        const uint32_t fb = leader_addr(&full_bar[kb]);
        if (leader)
          mbar_arrive_expect_tx(&full_bar[kb], 2 * Cfg::STAGE_BYTES);
        else
          mbar_arrive_cluster(fb);
        tma_load_2d_cg2(sB + kb * Cfg::B_BYTES, &tmB, fb, kb * BLOCK_K, nt * BN + rank * (BN / 2));
      }
    }
    pdl_wait();
    for (int u = unit0; u < num_units; u += nunits_grid) {
      int mt, nt;
      unit_coords(u, mt, nt);
      const int m0 = mt * (2 * BLOCK_M) + rank * BLOCK_M;
      const int n0 = nt * BN + rank * (BN / 2);
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&empty_bar[stage], phase ^ 1);
        if (lane == 0) {
          const uint32_t fb = leader_addr(&full_bar[stage]);
          if (u == unit0 && kb < pre) {
            load_a(stage, kb, m0, fb);
          } else {
            if (leader)
              mbar_arrive_expect_tx(&full_bar[stage], 2 * Cfg::STAGE_BYTES);
            else
              mbar_arrive_cluster(fb);
            load_a(stage, kb, m0, fb);
            tma_load_2d_cg2(sB + stage * Cfg::B_BYTES, &tmB, fb, kb * BLOCK_K, n0);
          }
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader only) =====================
    if (leader) {
      constexpr uint32_t idesc = make_idesc_i8(2 * BLOCK_M, BN);
      int stage = 0, phase = 0, acc = 0, acc_phase = 0, lt = 0;
      for (int u = unit0; u < num_units; u += nunits_grid, ++lt) {
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        if (tr && lane == 0 && lt < 15) tr[2 + 4 * lt] = gtime();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          if (tr && lane == 0 && lt < 15 && kb == nkb - 1) tr[3 + 4 * lt] = gtime();
          if (lane == 0) {
            const uint32_t a_addr = smem_u32(sA + stage * Cfg::A_BYTES);
            const uint32_t b_addr = smem_u32(sB + stage * Cfg::B_BYTES);
#pragma unroll
            for (int k = 0; k < BLOCK_K / 32; ++k)
              mma_i8_cg2(d_tmem, make_sw128_desc(a_addr + k * 32), make_sw128_desc(b_addr + k * 32),
                         idesc, (kb | k) != 0);
            mma_commit_mc2(&empty_bar[stage], CL == 4 ? 0xF : 0x3);
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (lane == 0) mma_commit_mc2(&tfull_bar[acc], (uint16_t)(0x3u << (crank & 2)));
        __syncwarp();
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // ===================== epilogue (both CTAs, own 128 rows) =====================
    // The first pass over the loop body is a dry run of the first tile's epilogue
    // (accumulator buffer 1, which that tile does not use; staging writes only, no
    // stores, no barrier traffic) made before griddepcontrol.wait: it pulls the
    // epilogue's instructions into the SM's instruction cache while the CTA waits
    // for the previous kernel, instead of on the first real tile (measured in the
    // BERT graph: first-tile epilogue 5.6 vs 3.7 us for the later tiles).
    bool dry = !(p.debug & 4) && unit0 < num_units && p.tma_out;
    if (!dry) pdl_wait();
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    constexpr int COLS = BN / 2;
    uint8_t* stage_c = sC + (warp - 2) * (2 * 32 * 32 * 4);
    int sbuf = 0;
    if (p.tma_out && lane == 0) prefetch_tmap(&tmC);
    int acc = 0, acc_phase = 0, lt = 0;
    const bool stamp = tr && warp == 2 && lane == 0;
    for (int u = unit0; u < num_units;) {
      int mt, nt;
      unit_coords(u, mt, nt);
      const int m0 = mt * (2 * BLOCK_M) + rank * BLOCK_M;
      const int n0 = nt * BN + half * COLS;
      const int row0 = m0 + quarter * 32;
      const int row = row0 + lane;
      float s_tok = p.static_scale;
      if (KIND != OUT_S32 && p.token_scales != nullptr && row < p.M) s_tok = __ldg(p.token_scales + row);
      if (!dry) {
        mbar_wait(&tfull_bar[acc], acc_phase);
        tc_fence_after();
        if (stamp && lt < 15) tr[4 + 4 * lt] = gtime();
      }
      const uint32_t t_row = tmem_base + ((uint32_t)(quarter * 32) << 16) + (dry ? 1 : acc) * BN + half * COLS;
#pragma unroll 1
      for (int c = 0; c < COLS; c += 32) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(t_row + c, r);
        tmem_ld_wait();
        if (c + 32 == COLS && !dry) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(leader_addr(&tempty_bar[acc]));
        }
        const int col0 = n0 + c;
        if (row0 >= p.M || col0 >= p.N) continue;
        if (p.tma_out) {
          // double-buffered staging: the bulk store of this chunk drains while the
          // next chunk is dequantised; the tensor map clips the M / N edges
          uint8_t* sb = stage_c + sbuf * (32 * 32 * 4);
          if (lane == 0) bulk_wait_read1();  // the store that last used `sb` has read it
          __syncwarp();
          if (!(p.debug & 2)) epi_chunk_smem<KIND>(r, s_tok, p.row_scales, p.bias, col0, p.N, sb, lane);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0 && !(p.debug & 1) && !dry) {
            tma_store_2d(&tmC, sb, col0, row0);
            if (p.kv_rows_per_seq > 0 && col0 >= p.kv_dl) {
              // prefill: the k / v columns of these 32 token rows also go to the KV
              // cache rows b * max_ctx + t (one sequence per 32-row box)
              const int crow = (int)((int64_t)(row0 / p.kv_rows_per_seq) * p.kv_max_ctx + row0 % p.kv_rows_per_seq);
              if (col0 < 2 * p.kv_dl) tma_store_2d(&tmKc, sb, col0 - p.kv_dl, crow);
              else tma_store_2d(&tmVc, sb, col0 - 2 * p.kv_dl, crow);
            }
            bulk_commit();
          }
          sbuf ^= 1;
        } else if (row < p.M) {
          epi_chunk_slow<KIND>(r, s_tok, p.row_scales, p.bias, p.out, (int64_t)row * p.ld_out,
                               col0, p.N);
        }
      }
      if (dry) {  // the same unit again, for real
        dry = false;
        pdl_wait();
        continue;
      }
      if (stamp && lt < 15) tr[5 + 4 * lt] = gtime();
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
      u += nunits_grid;
      ++lt;
    }
    if (lane == 0) bulk_wait0();  // all output stores complete before exit
    if (stamp) tr[63] = gtime();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) tmem_dealloc_cg2(tmem_base, Cfg::TMEM_COLS);
}


// ---------------------------------------------------------------------------
// Skinny (decode) GEMM, M <= 64 tokens, int8 weights: weight-streaming bound.
// Swap-AB: the MMA's M=128 side is 128 weight rows (output channels), its N side
// the MP (32 / 64) padded token rows, so D^T[n, m] sits in TMEM lane n.  Split-K
// over a cluster of S CTAs (S = 1..8) fills the machine: CTA r of the cluster
// accumulates k-blocks [r*nkb/S, (r+1)*nkb/S) of the same 128 weight rows, writes
// its int32 partial to its own smem, and after a cluster barrier reduces 128/S of
// the rows across all S partials through distributed shared memory (exact: int32
// addition is order-free) and applies the dequant epilogue for them.
// ---------------------------------------------------------------------------
// 4 stages = 96 KB: two CTAs per SM, so the next GEMM's weight prefetch (PDL)
// overlaps this one.  GPT-J decode step, linears in-graph: 2 stages 1.80 ms,
// 3 stages 1.63, 4 stages 1.59, 6 stages 2.74, 8 stages 2.75 (tools/ablate_decode.py)
constexpr int kSkStages = 4;

template <int MP, int W4 = 0>
struct SkinnyCfg {
  static constexpr int A_BYTES = 128 * BLOCK_K;   // weight tile (int8, SWIZZLE_128B)
  static constexpr int B_BYTES = MP * BLOCK_K;    // token tile
  static constexpr int P_BYTES = W4 ? 128 * (BLOCK_K / 2) : 0;  // packed INT4 staging
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int PART_BYTES = MP * 128 * 4; // int32 partial [MP][128]
  static constexpr int SMEM_BYTES = kSkStages * (STAGE_BYTES + P_BYTES) + PART_BYTES + 256;
};

__device__ __forceinline__ uint32_t dsmem_map(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ int32_t dsmem_ld_s32(uint32_t addr) {
  int32_t v;
  asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}

// W4: TMA brings the packed nibbles ([128 rows x 64 B], unswizzled) and warps 2-3
// (idle during the main loop otherwise) unpack them into the int8 SWIZZLE_128B
// tile the MMA reads, then add their arrivals on the stage's full barrier.
// W4: 256 threads (warps 2-7 unpack: the INT4 -> INT8 expansion of a 16 KB
// k-block by 64 threads left the 4hh projection of GPT-3 350M decode (4 k-blocks
// per CTA) unpack-bound); the TMEM partial / reduction use warps 0-3 / all.
template <int MP, int W4>
constexpr int skinny_threads() { return W4 ? 256 : 128; }

template <int MP, int KIND, int W4>
__global__ void __launch_bounds__(skinny_threads<MP, W4>(), 1)
    zq_gemm_skinny_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                          const GemmParams p, int S) {
  using Cfg = SkinnyCfg<MP, W4>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + kSkStages * Cfg::A_BYTES;
  uint8_t* sP = smem + kSkStages * Cfg::STAGE_BYTES;  // W4 only
  int32_t* part = reinterpret_cast<int32_t*>(smem + kSkStages * (Cfg::STAGE_BYTES + Cfg::P_BYTES));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kSkStages * (Cfg::STAGE_BYTES + Cfg::P_BYTES) + Cfg::PART_BYTES);
  uint64_t* full_bar = bars;
  uint64_t* empty_bar = bars + kSkStages;
  uint64_t* done_bar = bars + 2 * kSkStages;
  uint64_t* praw_bar = bars + 2 * kSkStages + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * kSkStages + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = (int)cluster_ctarank();
  const int n0 = (blockIdx.x / S) * 128;
  const int nkb = p.num_k_blocks;
  const int kb0 = (int)(((int64_t)nkb * r) / S), kb1 = (int)(((int64_t)nkb * (r + 1)) / S);

  if (threadIdx.x == 0) {
    if (smem_u32(smem) & 1023) __trap();
    prefetch_tmap(&tmW);
    prefetch_tmap(&tmX);
    for (int st = 0; st < kSkStages; ++st) {
      mbar_init(&full_bar[st], W4 ? 1 + (skinny_threads<MP, W4>() / 32 - 2) : 1);  // W4: + one arrival per unpack warp
      mbar_init(&empty_bar[st], 1);
      if (W4) mbar_init(&praw_bar[st], 1);
    }
    mbar_init(done_bar, 1);
    fence_barrier_init();
  }
  __syncwarp();  // reconverge warp 0 after the lane-0 setup before the CTA barrier
  if (warp == 1) tmem_alloc(tmem_slot, MP < 32 ? 32 : MP);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  pdl_trigger();
  if (warp == 0) {
    // the first kSkStages weight tiles stream in before the grid dependency resolves
    int stage = 0, phase = 0;
    const int pre = (kb1 - kb0) < kSkStages ? (kb1 - kb0) : kSkStages;
    auto load_w = [&](int st, int kb) {
      if (W4) {
        mbar_arrive_expect_tx(&praw_bar[st], Cfg::P_BYTES);
        tma_load_2d(sP + st * Cfg::P_BYTES, &tmW, &praw_bar[st], kb * (BLOCK_K / 2), n0);
        mbar_arrive_expect_tx(&full_bar[st], Cfg::B_BYTES);
      } else {
        mbar_arrive_expect_tx(&full_bar[st], Cfg::STAGE_BYTES);
        tma_load_2d(sA + st * Cfg::A_BYTES, &tmW, &full_bar[st], kb * BLOCK_K, n0);
      }
    };
    if (lane == 0)
      for (int i = 0; i < pre; ++i) load_w(i, kb0 + i);
    pdl_wait();
    for (int kb = kb0; kb < kb1; ++kb) {
      mbar_wait(&empty_bar[stage], phase ^ 1);
      if (lane == 0) {
        if (kb - kb0 >= pre) load_w(stage, kb);
        tma_load_2d(sB + stage * Cfg::B_BYTES, &tmX, &full_bar[stage], kb * BLOCK_K, 0);
      }
      __syncwarp();
      if (++stage == kSkStages) {
        stage = 0;
        phase ^= 1;
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = make_idesc_i8(128, MP);
    int stage = 0, phase = 0;
    for (int kb = kb0; kb < kb1; ++kb) {
      mbar_wait(&full_bar[stage], phase);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t a_addr = smem_u32(sA + stage * Cfg::A_BYTES);
        const uint32_t b_addr = smem_u32(sB + stage * Cfg::B_BYTES);
#pragma unroll
        for (int k = 0; k < BLOCK_K / 32; ++k)
          mma_i8(tmem, make_sw128_desc(a_addr + k * 32), make_sw128_desc(b_addr + k * 32), idesc,
                 (kb != kb0 || k != 0) ? 1u : 0u);
        mma_commit(&empty_bar[stage]);
      }
      __syncwarp();
      if (++stage == kSkStages) {
        stage = 0;
        phase ^= 1;
      }
    }
    if (lane == 0) {
      if (kb1 > kb0) mma_commit(done_bar);
      else mbar_arrive(done_bar);  // empty split: contributes zeros
    }
    __syncwarp();
  } else if (W4) {
    // warps 2-3: INT4 -> INT8 into the SWIZZLE_128B tile (row r, 16-byte chunk c at
    // r*128 + ((c ^ (r & 7)) * 16)); nibble j of a packed word is element j
    constexpr int UT = skinny_threads<MP, W4>() - 64;  // unpack threads
    const int ut = threadIdx.x - 64;
    int stage = 0, phase = 0;
    for (int kb = kb0; kb < kb1; ++kb) {
      mbar_wait(&empty_bar[stage], phase ^ 1);
      mbar_wait(&praw_bar[stage], phase);
      const uint8_t* src = sP + stage * Cfg::P_BYTES;
      uint8_t* dst = sA + stage * Cfg::A_BYTES;
#pragma unroll 2
      for (int idx = ut; idx < 128 * 8; idx += UT) {
        const int rr = idx >> 3, c = idx & 7;
        const uint2 pk = *reinterpret_cast<const uint2*>(src + rr * 64 + c * 8);
        uint32_t w[4];
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const uint32_t x = hh ? pk.y : pk.x;
          uint32_t ev = x & 0x0F0F0F0Fu, od = (x >> 4) & 0x0F0F0F0Fu;
          ev |= (ev & 0x08080808u) * 0x1Eu;
          od |= (od & 0x08080808u) * 0x1Eu;
          w[2 * hh] = __byte_perm(ev, od, 0x5140);
          w[2 * hh + 1] = __byte_perm(ev, od, 0x7362);
        }
        *reinterpret_cast<uint4*>(dst + rr * 128 + ((c ^ (rr & 7)) * 16)) = make_uint4(w[0], w[1], w[2], w[3]);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&full_bar[stage]);
      if (++stage == kSkStages) {
        stage = 0;
        phase ^= 1;
      }
    }
  }
  // ---- partial: TMEM (lane = weight row) -> smem [MP][128] ----
  mbar_wait(done_bar, 0);
  tc_fence_after();
  if (warp < 4) {
    const int row = warp * 32 + lane;
#pragma unroll
    for (int c = 0; c < MP; c += 32) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(tmem + ((uint32_t)(warp * 32) << 16) + c, v);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) part[(c + j) * 128 + row] = kb1 > kb0 ? (int32_t)v[j] : 0;
    }
  }
  tc_fence_before();
  pdl_wait();
  cluster_sync();
  // ---- cluster reduction + epilogue for rows [128 r / S, 128 (r+1) / S) ----
  const int r_lo = (128 * r) / S, RP = (128 * (r + 1)) / S - r_lo;
  const uint32_t pbase = smem_u32(part);
  for (int it = threadIdx.x; it < MP * RP; it += skinny_threads<MP, W4>()) {
    const int m = it / RP, nl = r_lo + it % RP;
    const int n = n0 + nl;
    if (m >= p.M || n >= p.N) continue;
    const uint32_t off = pbase + (uint32_t)(m * 128 + nl) * 4;
    int32_t acc = 0;
    for (int s2 = 0; s2 < S; ++s2) acc += dsmem_ld_s32(dsmem_map(off, (uint32_t)s2));
    const int64_t o = (int64_t)m * p.ld_out + n;
    if (KIND == OUT_S32) {
      reinterpret_cast<int32_t*>(p.out)[o] = acc;
    } else {
      const float st = p.token_scales ? __ldg(p.token_scales + m) : p.static_scale;
      float f = __fmul_rn(__fmul_rn(__int2float_rn(acc), st), __ldg(p.row_scales + n));
      if (p.bias) f = __fadd_rn(f, __ldg(p.bias + n));
      if (KIND == OUT_F32) {
        reinterpret_cast<float*>(p.out)[o] = f;
        if (p.kc != nullptr && n >= p.kv_dl) {  // fused KV-cache append (decode QKV)
          const int64_t slot = ((int64_t)m * p.kv_max_ctx + p.kv_pos[m]) * p.kv_dl;
          if (n < 2 * p.kv_dl) p.kc[slot + (n - p.kv_dl)] = f;
          else p.vc[slot + (n - 2 * p.kv_dl)] = f;
        }
      } else if (KIND == OUT_F16) {
        reinterpret_cast<__half*>(p.out)[o] = __float2half_rn(f);
      } else {
        reinterpret_cast<__nv_bfloat16*>(p.out)[o] = __float2bfloat16_rn(f);
      }
    }
  }
  cluster_sync();  // peers may still be reading this CTA's partial
  if (warp == 1) tmem_dealloc(tmem, MP < 32 ? 32 : MP);
}


// ---------------------------------------------------------------------------
// Stream-K skinny (decode) GEMM, M <= 64 tokens, int8 weights.  The cluster
// split-K kernel above gives every CTA one (n-tile, k-range) of equal size, so a
// grid of 1.3 waves (NeoX h4h: 384 CTAs on 296 slots) streams at ~70% of HBM.
// Here the n_tiles x nkb k-block units are cut into G = 2 x #SMs equal
// contiguous ranges (tile-major); a CTA accumulates each tile segment of its
// range in TMEM (swap-AB, double-buffered) and adds it to an int32 workspace
// with red.global.add (exact: integer addition is order-free).  The dequant
// epilogue runs as the next kernel (skinny_sum_epilogue_kernel), which also
// re-zeroes the workspace: a last-arriver epilogue inside this kernel (counter +
// gpu-scope fences) measured ~8 us slower per launch at NeoX widths, the fences
// stalling the CTA's in-flight weight stream (tools/skinny_bench.py).
//   warp 0 TMA (weights of the first stages before the grid dependency),
//   warp 1 MMA, warps 2-5 reduction (TMEM lane quarters 2, 3, 0, 1).
constexpr int kSkkStages = 4;  // 80 KB per CTA, two CTAs per SM

template <int MP>
struct StreamKCfg {
  static constexpr int A_BYTES = 128 * BLOCK_K;
  static constexpr int B_BYTES = MP * BLOCK_K;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int SMEM_BYTES = kSkkStages * STAGE_BYTES + 256;
};

__device__ __forceinline__ void red_add_s32(int32_t* p, int32_t v) {
  asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int MP, int KIND>
__global__ void __launch_bounds__(192, 2)
    zq_gemm_streamk_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                           const GemmParams p) {
  using Cfg = StreamKCfg<MP>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + kSkkStages * Cfg::A_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kSkkStages * Cfg::STAGE_BYTES);
  uint64_t* full_bar = bars;
  uint64_t* empty_bar = bars + kSkkStages;
  uint64_t* tfull_bar = bars + 2 * kSkkStages;      // [2]
  uint64_t* tempty_bar = bars + 2 * kSkkStages + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kSkkStages + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkb = p.num_k_blocks, ntile = p.num_n_tiles;
  const int64_t U = (int64_t)ntile * nkb;
  const int u0 = (int)(U * blockIdx.x / gridDim.x), u1 = (int)(U * (blockIdx.x + 1) / gridDim.x);
  int32_t* acc_ws = p.sk_ws;

  if (threadIdx.x == 0) {
    if (smem_u32(smem) & 1023) __trap();
    prefetch_tmap(&tmW);
    prefetch_tmap(&tmX);
    for (int st = 0; st < kSkkStages; ++st) {
      mbar_init(&full_bar[st], 1);
      mbar_init(&empty_bar[st], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 4);
    }
    fence_barrier_init();
  }
  __syncwarp();
  if (warp == 1) tmem_alloc(tmem_slot, 2 * MP);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      const int pre = (u1 - u0) < kSkkStages ? (u1 - u0) : kSkkStages;
      for (int i = 0; i < pre; ++i) {  // weights do not depend on the previous kernel
        const int u = u0 + i;
        mbar_arrive_expect_tx(&full_bar[i], Cfg::STAGE_BYTES);
        tma_load_2d(sA + i * Cfg::A_BYTES, &tmW, &full_bar[i], (u % nkb) * BLOCK_K, (u / nkb) * 128);
      }
      pdl_wait();
      for (int i = 0; i < pre; ++i)
        tma_load_2d(sB + i * Cfg::B_BYTES, &tmX, &full_bar[i], ((u0 + i) % nkb) * BLOCK_K, 0);
      int stage = pre % kSkkStages, phase = pre / kSkkStages;
      for (int u = u0 + pre; u < u1; ++u) {
        mbar_wait(&empty_bar[stage], phase ^ 1);
        mbar_arrive_expect_tx(&full_bar[stage], Cfg::STAGE_BYTES);
        tma_load_2d(sA + stage * Cfg::A_BYTES, &tmW, &full_bar[stage], (u % nkb) * BLOCK_K, (u / nkb) * 128);
        tma_load_2d(sB + stage * Cfg::B_BYTES, &tmX, &full_bar[stage], (u % nkb) * BLOCK_K, 0);
        if (++stage == kSkkStages) stage = 0, phase ^= 1;
      }
    }
    pdl_wait();
  } else if (warp == 1) {
    pdl_wait();
    constexpr uint32_t idesc = make_idesc_i8(128, MP);
    int stage = 0, phase = 0, acc = 0, aph = 0;
    for (int u = u0; u < u1;) {
      const int tile = u / nkb, uend = min(u1, (tile + 1) * nkb);
      mbar_wait(&tempty_bar[acc], aph ^ 1);
      tc_fence_after();
      const uint32_t d = tmem + acc * MP;
      for (int v = u; v < uend; ++v) {
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t a_addr = smem_u32(sA + stage * Cfg::A_BYTES);
          const uint32_t b_addr = smem_u32(sB + stage * Cfg::B_BYTES);
#pragma unroll
          for (int k = 0; k < BLOCK_K / 32; ++k)
            mma_i8(d, make_sw128_desc(a_addr + k * 32), make_sw128_desc(b_addr + k * 32), idesc,
                   (v != u || k != 0) ? 1u : 0u);
          mma_commit(&empty_bar[stage]);
        }
        __syncwarp();
        if (++stage == kSkkStages) stage = 0, phase ^= 1;
      }
      if (lane == 0) mma_commit(&tfull_bar[acc]);
      __syncwarp();
      if (++acc == 2) acc = 0, aph ^= 1;
      u = uend;
    }
  } else {
    // ===== epilogue warps 2..5: TMEM lane quarter q = warp & 3 (rows 32q .. 32q+31) =====
    pdl_wait();
    const int q = warp & 3;
    const int nl = q * 32 + lane;     // this thread's weight row of the tile
    int acc = 0, aph = 0;
    for (int u = u0; u < u1;) {
      const int tile = u / nkb, uend = min(u1, (tile + 1) * nkb);
      mbar_wait(&tfull_bar[acc], aph);
      tc_fence_after();
      uint32_t r[MP];
#pragma unroll
      for (int c = 0; c < MP; c += 32) {
        tmem_ld_32x32b_x32(tmem + ((uint32_t)(q * 32) << 16) + acc * MP + c, *reinterpret_cast<uint32_t(*)[32]>(&r[c]));
      }
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[acc]);
      if (++acc == 2) acc = 0, aph ^= 1;
      const int mlim = p.M < MP ? p.M : MP;
      // this segment's partial -> the tile's int32 sums (red.add: exact, order-free);
      // the dequant epilogue is the next kernel (skinny_sum_epilogue_kernel)
      int32_t* tw = acc_ws + (int64_t)tile * MP * 128;
#pragma unroll
      for (int m = 0; m < MP; ++m)
        if (m < mlim) red_add_s32(tw + m * 128 + nl, (int32_t)r[m]);
      u = uend;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 2 * MP);
}

// ---------------------------------------------------------------------------
// Fused row-parallel projection + residual + LayerNorm + token-wise quantize
// (transformer.py:474-477 / :484-486: y = LN(x + linear(q, w)), igemm.py:150-157):
//   f  = ((f32(acc) * s_tok) * s_w) + bias      (igemm.py:107-111, exact order)
//   v  = x + f                                   (residual, f32)
//   y  = LN(v) with numpy's pairwise mean / variance (tensor.py:59-73)
//   q, s = token-wise quantize(y)                (quant.py:258-269)
// The GEMM's output never goes to HBM: only y (f32, the next residual) and q /
// scales are written.  A pair tile is 256 rows x BN columns and BN / 2 = L is
// exactly one leaf of numpy's pairwise tree for the row width N = NT * BN
// (N = L * 2^k), so each epilogue thread owns one leaf of one row in registers
// and evaluates it with numpy's 8-chain leaf order.  The tree above the leaves
// spans the NT tiles of a row block; their partial sums / maxima are exchanged
// through global memory with a release/acquire counter per row block (three
// rounds: sum, squared deviations, max).  All tiles of a row block are in the
// same round of the persistent grid (tiles_per_round = floor(pairs / NT) * NT)
// and every CTA is co-resident, so the exchange cannot deadlock.  The counter is
// never reset: each launch adds exactly 6 * NT per row block, so a CTA derives
// this launch's base from the value its first increment returns.
// ---------------------------------------------------------------------------
struct LnFuseParams {
  const float* residual;  // [M, N] f32 (x)
  const float* gamma;
  const float* beta;
  float eps;
  float* ln_out;          // [M, N] f32 (y)
  int8_t* q;              // [M, ld_q]
  int64_t ld_q;
  float* q_scales;        // [M]
  int qm;
  float* partials;        // [3][M][NT]
  unsigned int* counters; // [ceil(M / 256)], zero at allocation, never reset
  int32_t* flag;
  int tiles_per_round;
};

__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void epi_bar() {  // the 8 epilogue warps (256 threads)
  asm volatile("bar.sync 1, 256;" ::: "memory");
}

template <int L>
__device__ __forceinline__ float leaf_sum(const float (&v)[L]) {  // numpy pairwise leaf (L <= 128)
  float r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = v[j];
#pragma unroll
  for (int i = 8; i < L; i += 8)
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __fadd_rn(r[j], v[i + j]);
  return __fadd_rn(__fadd_rn(__fadd_rn(r[0], r[1]), __fadd_rn(r[2], r[3])),
                   __fadd_rn(__fadd_rn(r[4], r[5]), __fadd_rn(r[6], r[7])));
}

template <int L>
__device__ __forceinline__ float leaf_sum_sqdev(const float (&v)[L], float mean) {  // same order, (v - mean)^2
  float r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float d = __fsub_rn(v[j], mean);
    r[j] = __fmul_rn(d, d);
  }
#pragma unroll
  for (int i = 8; i < L; i += 8)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float d = __fsub_rn(v[i + j], mean);
      r[j] = __fadd_rn(r[j], __fmul_rn(d, d));
    }
  return __fadd_rn(__fadd_rn(__fadd_rn(r[0], r[1]), __fadd_rn(r[2], r[3])),
                   __fadd_rn(__fadd_rn(r[4], r[5]), __fadd_rn(r[6], r[7])));
}

template <int BN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Gemm2Cfg<BN>::NUM_THREADS, 1)
    zq_gemm2_ln_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       const GemmParams p, const LnFuseParams f) {
  using Cfg = Gemm2Cfg<BN>;
  constexpr int STAGES = Cfg::STAGES;
  constexpr int COLS = BN / 2;  // one pairwise leaf
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * Cfg::A_BYTES;
  uint8_t* sC = smem + STAGES * Cfg::STAGE_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sC + Cfg::EPI_BYTES);
  uint64_t* full_bar = bars;
  uint64_t* empty_bar = bars + STAGES;
  uint64_t* tfull_bar = bars + 2 * STAGES;
  uint64_t* tempty_bar = bars + 2 * STAGES + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);
  float* xch = reinterpret_cast<float*>(sC);  // [2][128] leaf partial exchange between the halves
  unsigned int* sbase = reinterpret_cast<unsigned int*>(sC + 2048);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1;
  const int tpr = f.tiles_per_round;
  const int NT = p.num_n_tiles;

  if (warp == 0 && lane == 0) {
    if (smem_u32(smem) & 1023) __trap();
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    for (int st = 0; st < STAGES; ++st) {
      mbar_init(&full_bar[st], 2);
      mbar_init(&empty_bar[st], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 2 * kNumEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_cg2(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int nkb = p.num_k_blocks;
  pdl_trigger();

  if (warp == 0) {
    int stage = 0, phase = 0;
    const int pre = (pair < tpr && pair < p.num_tiles) ? (nkb < STAGES ? nkb : STAGES) : 0;
    if (lane == 0)
      for (int kb = 0; kb < pre; ++kb) {
        const uint32_t fb = leader_addr(&full_bar[kb]);
        if (leader)
          mbar_arrive_expect_tx(&full_bar[kb], 2 * Cfg::STAGE_BYTES);
        else
          mbar_arrive_cluster(fb);
        tma_load_2d_cg2(sB + kb * Cfg::B_BYTES, &tmB, fb, kb * BLOCK_K, (pair % NT) * BN + rank * (BN / 2));
      }
    pdl_wait();
    for (int tile = pair; pair < tpr && tile < p.num_tiles; tile += tpr) {
      const int m0 = (tile / NT) * (2 * BLOCK_M) + rank * BLOCK_M;
      const int n0 = (tile % NT) * BN + rank * (BN / 2);
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&empty_bar[stage], phase ^ 1);
        if (lane == 0) {
          const uint32_t fb = leader_addr(&full_bar[stage]);
          if (tile == pair && kb < pre) {
            tma_load_2d_cg2(sA + stage * Cfg::A_BYTES, &tmA, fb, kb * BLOCK_K, m0);
          } else {
            if (leader)
              mbar_arrive_expect_tx(&full_bar[stage], 2 * Cfg::STAGE_BYTES);
            else
              mbar_arrive_cluster(fb);
            tma_load_2d_cg2(sA + stage * Cfg::A_BYTES, &tmA, fb, kb * BLOCK_K, m0);
            tma_load_2d_cg2(sB + stage * Cfg::B_BYTES, &tmB, fb, kb * BLOCK_K, n0);
          }
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      constexpr uint32_t idesc = make_idesc_i8(2 * BLOCK_M, BN);
      int stage = 0, phase = 0, acc = 0, acc_phase = 0;
      for (int tile = pair; pair < tpr && tile < p.num_tiles; tile += tpr) {
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t a_addr = smem_u32(sA + stage * Cfg::A_BYTES);
            const uint32_t b_addr = smem_u32(sB + stage * Cfg::B_BYTES);
#pragma unroll
            for (int k = 0; k < BLOCK_K / 32; ++k)
              mma_i8_cg2(d_tmem, make_sw128_desc(a_addr + k * 32), make_sw128_desc(b_addr + k * 32), idesc,
                         (kb | k) != 0);
            mma_commit_mc2(&empty_bar[stage], 0x3);
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (lane == 0) mma_commit_mc2(&tfull_bar[acc], 0x3);
        __syncwarp();
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // ===================== fused epilogue =====================
    pdl_wait();
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    const int rl = quarter * 32 + lane;  // row within the CTA's 128
    int acc = 0, acc_phase = 0;
    for (int tile = pair; pair < tpr && tile < p.num_tiles; tile += tpr) {
      const int rb = tile / NT, nt = tile % NT;
      const int row = rb * (2 * BLOCK_M) + rank * BLOCK_M + rl;
      const bool live = row < p.M;
      const int n0 = nt * BN + half * COLS;
      const float s_tok = live ? __ldg(p.token_scales + row) : 0.0f;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t t_row = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN + half * COLS;
      float v[COLS];
      const float* xr = f.residual + (int64_t)(live ? row : 0) * p.N + n0;
#pragma unroll
      for (int c = 0; c < COLS; c += 32) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(t_row + c, r);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          const float4 sw = __ldg(reinterpret_cast<const float4*>(p.row_scales + n0 + c + j));
          const float4 bb = __ldg(reinterpret_cast<const float4*>(p.bias + n0 + c + j));
          const float4 xx = live ? __ldg(reinterpret_cast<const float4*>(xr + c + j)) : make_float4(0.f, 0.f, 0.f, 0.f);
          const float swv[4] = {sw.x, sw.y, sw.z, sw.w}, bv[4] = {bb.x, bb.y, bb.z, bb.w};
          const float xv[4] = {xx.x, xx.y, xx.z, xx.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float fo = __fadd_rn(__fmul_rn(__fmul_rn(__int2float_rn((int)r[j + u]), s_tok), swv[u]), bv[u]);
            v[c + j + u] = __fadd_rn(xv[u], fo);  // x + f (transformer.py:477 / :486)
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader_addr(&tempty_bar[acc]));  // accumulator consumed
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
      unsigned int* cnt = f.counters + rb;
      const unsigned int per_round = 2u * NT;
      // exchange one value per (row, tile) through global memory, round `rd`
      auto publish_and_wait = [&](int rd, float val) {
        if (half == 0 && live) __stcg(f.partials + ((int64_t)rd * p.M + row) * NT + nt, val);
        epi_bar();  // orders the CTA's partial stores before the releasing add below
        if (warp == 2 && lane == 0) {
          unsigned int old;
          asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(cnt) : "memory");
          if (rd == 0) *sbase = old - old % (3u * per_round);
          const unsigned int target = *sbase + (unsigned int)(rd + 1) * per_round;
          while (!(p.debug & 4) && (int)(ld_acquire_u32(cnt) - target) < 0) __nanosleep(64);
        }
        epi_bar();
      };
      auto gather_tree = [&](int rd) -> float {  // balanced tree over the NT tile partials
        const float* pr = f.partials + ((int64_t)rd * p.M + (live ? row : 0)) * NT;
        if (NT == 4) {
          const float4 t = __ldcg(reinterpret_cast<const float4*>(pr));
          return __fadd_rn(__fadd_rn(t.x, t.y), __fadd_rn(t.z, t.w));
        }
        // larger NT: pairwise levels with a small stack of partial sums (binary counter)
        float stk[7];
        int cnt = 0;
        for (int i = 0; i < NT; ++i) {
          float val = __ldcg(pr + i);
          int k = i;
          // merge while the lowest bits of the index say a subtree completed
          while (k & 1) {
            val = __fadd_rn(stk[--cnt], val);
            k >>= 1;
          }
          stk[cnt++] = val;
        }
        return stk[0];
      };
      // ---- round 0: mean ----
      {
        const float leaf = leaf_sum<COLS>(v);
        xch[half * 128 + rl] = leaf;
        epi_bar();
        const float tsum = __fadd_rn(xch[rl], xch[128 + rl]);  // (left leaf + right leaf)
        publish_and_wait(0, tsum);
      }
      const float fcols = (float)p.N;
      const float mean = __fdiv_rn(gather_tree(0), fcols);
      // ---- round 1: variance ----
      {
        const float leaf = leaf_sum_sqdev<COLS>(v, mean);
        epi_bar();  // xch reuse
        xch[half * 128 + rl] = leaf;
        epi_bar();
        publish_and_wait(1, __fadd_rn(xch[rl], xch[128 + rl]));
      }
      const float var = __fdiv_rn(gather_tree(1), fcols);
      const float den = __fsqrt_rn(__fadd_rn(var, f.eps));
      const float rden = __frcp_rn(den);
      const bool den_ok = den > 1e-18f && den < 1e18f;
      // ---- normalise, write y, row max ----
      uint32_t ab = 0;
      float* yr = f.ln_out + (int64_t)(live ? row : 0) * p.N + n0;
#pragma unroll
      for (int j = 0; j < COLS; j += 4) {
        const float4 g = __ldg(reinterpret_cast<const float4*>(f.gamma + n0 + j));
        const float4 b = __ldg(reinterpret_cast<const float4*>(f.beta + n0 + j));
        const float gv[4] = {g.x, g.y, g.z, g.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float a = __fsub_rn(v[j + u], mean);
          float qd;
          if (den_ok && (fabsf(a) >= 1e-30f || a == 0.0f)) {
            const float q0 = __fmul_rn(a, rden);
            const float q1 = __fmaf_rn(__fmaf_rn(-den, q0, a), rden, q0);
            qd = __fmaf_rn(__fmaf_rn(-den, q1, a), rden, q1);
          } else {
            qd = __fdiv_rn(a, den);
          }
          v[j + u] = __fadd_rn(__fmul_rn(qd, gv[u]), bv[u]);
          ab = max(ab, __float_as_uint(v[j + u]) & 0x7fffffffu);
        }
        if (live) *reinterpret_cast<float4*>(yr + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      }
      // ---- round 2: row max ----
      epi_bar();
      reinterpret_cast<uint32_t*>(xch)[half * 128 + rl] = ab;
      epi_bar();
      publish_and_wait(2, __uint_as_float(max(reinterpret_cast<uint32_t*>(xch)[rl],
                                              reinterpret_cast<uint32_t*>(xch)[128 + rl])));
      uint32_t amb_row = 0;
      for (int i = 0; i < NT; ++i)
        amb_row = max(amb_row, live ? __float_as_uint(__ldcg(f.partials + ((int64_t)2 * p.M + row) * NT + i)) : 0u);
      if (!live) continue;
      if (amb_row >= 0x7f800000u && nt == 0 && half == 0 && f.flag) atomicOr(f.flag, 1);
      const float sc = scale_from_absmax(__uint_as_float(amb_row), f.qm);
      const float inv = (__frcp_rn(sc) < 1e30f) ? __frcp_rn(sc) : 0.0f;
      if (nt == 0 && half == 0) f.q_scales[row] = sc;
      uint32_t* qrow = reinterpret_cast<uint32_t*>(f.q + (int64_t)row * f.ld_q + n0);
#pragma unroll
      for (int j = 0; j < COLS; j += 4) {
        int o[4];
        bool amb = inv == 0.0f;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float m = __fmaf_rn(v[j + u], inv, 12582912.0f);
          amb |= fabsf(__fmaf_rn(v[j + u], inv, -__fsub_rn(m, 12582912.0f))) > 0.5f - 6.103515625e-05f;
          o[u] = __float_as_int(m) - 0x4B400000;
        }
        if (amb)
#pragma unroll
          for (int u = 0; u < 4; ++u) o[u] = quantize_exact(v[j + u], sc, f.qm);
        qrow[j / 4] = __byte_perm(__byte_perm((uint32_t)o[0], (uint32_t)o[1], 0x0040),
                                  __byte_perm((uint32_t)o[2], (uint32_t)o[3], 0x0040), 0x5410);
      }
      if (nt == NT - 1 && half == 1)
        for (int c = p.N; c < (int)f.ld_q; ++c) f.q[(int64_t)row * f.ld_q + c] = 0;
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) tmem_dealloc_cg2(tmem_base, Cfg::TMEM_COLS);
}

template <int BN>
static int launch_gemm2_ln_t(const CUtensorMap& ta, const CUtensorMap& tb, GemmParams p, const LnFuseParams& f,
                             int grid, cudaStream_t st) {
  using Cfg = Gemm2Cfg<BN>;
  static ZqDeviceOnce attr_once;
  attr_once([&](int) {
    cudaFuncSetAttribute(zq_gemm2_ln_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
  });
  const cudaError_t e = launch_kernel(zq_gemm2_ln_kernel<BN>, dim3(grid), dim3(Cfg::NUM_THREADS),
                                      Cfg::SMEM_BYTES, st, 1, ta, tb, p, f);
  if (e != cudaSuccess) {
    set_error("fused linear + LN launch: %s", cudaGetErrorString(e));
    return ZQ_ERR_CUDA;
  }
  return ZQ_OK;
}

// ---------------------------------------------------------------------------
// Standalone epilogue over an int32 accumulator (TP path) and the weight-only
// FullAct GEMM (sequential f32 order, tensor.py:37-56).
// ---------------------------------------------------------------------------
__global__ void epilogue_kernel(const int32_t* __restrict__ acc, int64_t ld_acc,
                                const float* __restrict__ ts, float static_scale,
                                const float* __restrict__ rs, const float* __restrict__ bias,
                                int64_t M, int64_t N, void* out, int64_t ld_out, int kind) {
  const int64_t total = M * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / N, c = i - r * N;
    float s = ts ? ts[r] : static_scale;
    float f = __fmul_rn(__fmul_rn(__int2float_rn(acc[r * ld_acc + c]), s), rs[c]);
    if (bias) f = __fadd_rn(f, bias[c]);
    int64_t o = r * ld_out + c;
    if (kind == ZQ_OUT_F32) reinterpret_cast<float*>(out)[o] = f;
    else if (kind == ZQ_OUT_F16) reinterpret_cast<__half*>(out)[o] = __float2half_rn(f);
    else reinterpret_cast<__nv_bfloat16*>(out)[o] = __float2bfloat16_rn(f);
  }
}

// The same, 4 columns per thread (N % 4 == 0, 16-byte aligned rows): the dequant
// after the tensor-parallel int32 SUM all-reduce, one L2 round trip per thread.
__global__ void __launch_bounds__(256) epilogue_vec_kernel(const int32_t* __restrict__ acc, int64_t ld_acc,
                                                           const float* __restrict__ ts, float static_scale,
                                                           const float* __restrict__ rs,
                                                           const float* __restrict__ bias, int M, int N, void* out,
                                                           int64_t ld_out, int kind) {
  pdl_trigger();
  pdl_wait();
  const int n4 = N >> 2, total = M * n4;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int m = i / n4, n = (i - m * n4) * 4;
    const int4 a = __ldg(reinterpret_cast<const int4*>(acc + (int64_t)m * ld_acc + n));
    const float st = ts ? __ldg(ts + m) : static_scale;
    const float4 w = __ldg(reinterpret_cast<const float4*>(rs + n));
    const float4 b = bias ? __ldg(reinterpret_cast<const float4*>(bias + n)) : make_float4(0.f, 0.f, 0.f, 0.f);
    const int av[4] = {a.x, a.y, a.z, a.w};
    const float wv[4] = {w.x, w.y, w.z, w.w}, bv[4] = {b.x, b.y, b.z, b.w};
    float f[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      f[j] = __fmul_rn(__fmul_rn(__int2float_rn(av[j]), st), wv[j]);
      if (bias) f[j] = __fadd_rn(f[j], bv[j]);
    }
    const int64_t o = (int64_t)m * ld_out + n;
    if (kind == ZQ_OUT_F32) {
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + o) = make_float4(f[0], f[1], f[2], f[3]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (kind == ZQ_OUT_F16) reinterpret_cast<__half*>(out)[o + j] = __float2half_rn(f[j]);
        else reinterpret_cast<__nv_bfloat16*>(out)[o + j] = __float2bfloat16_rn(f[j]);
      }
    }
  }
}

// 32x32 output tile per CTA (256 threads, 4 outputs each); K staged through smem
// in chunks of 32; every output accumulates p = 0..K-1 in order with separately
// rounded products and sums (no FMA), starting from +0.0.
__global__ void __launch_bounds__(256) full_linear_kernel(
    const float* __restrict__ x, int64_t ld_x, const int8_t* __restrict__ w8,
    const uint8_t* __restrict__ w4, int64_t ld_w, const float* __restrict__ rs,
    const float* __restrict__ bias, int64_t M, int64_t N, int64_t K, float* __restrict__ out,
    int64_t ld_out) {
  __shared__ float xs[32][33];
  __shared__ float ws[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // ty 0..7
  const int64_t m0 = (int64_t)blockIdx.y * 32, n0 = (int64_t)blockIdx.x * 32;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int64_t k0 = 0; k0 < K; k0 += 32) {
    for (int i = ty; i < 32; i += 8) {
      int64_t m = m0 + i, k = k0 + tx;
      xs[i][tx] = (m < M && k < K) ? x[m * ld_x + k] : 0.0f;
      int64_t n = n0 + i;
      float wv = 0.0f;
      if (n < N && k < K) {
        int q;
        if (w4) {
          uint8_t b = w4[n * (ld_w / 2) + (k >> 1)];
          int nib = (k & 1) ? (b >> 4) : (b & 0xF);
          q = nib > 7 ? nib - 16 : nib;
        } else {
          q = w8[n * ld_w + k];
        }
        wv = __fmul_rn((float)q, rs[n]);  // QuantizedMatrix.dequantize, quant.py:172-174
      }
      ws[i][tx] = wv;
    }
    __syncthreads();
    const int kk = (int)min((int64_t)32, K - k0);
    for (int k = 0; k < kk; ++k) {
      const float wv = ws[tx][k];
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[r] = __fadd_rn(acc[r], __fmul_rn(xs[ty + 8 * r][k], wv));
    }
    __syncthreads();
  }
  const int64_t n = n0 + tx;
  if (n < N) {
    float b = bias ? bias[n] : 0.0f;
    for (int r = 0; r < 4; ++r) {
      int64_t m = m0 + ty + 8 * r;
      if (m < M) out[m * ld_out + n] = __fadd_rn(acc[r], b);
    }
  }
}

// ---------------------------------------------------------------------------
// host side: tensor maps, tile-shape selection, launch
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static std::once_flag g_encode_once;

static bool get_encode() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode != nullptr;
}

static int make_tmap_u8(CUtensorMap* tm, const void* base, int64_t rows, int64_t cols,
                        int64_t ld_bytes, int box_cols, int box_rows, CUtensorMapSwizzle sw) {
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld_bytes};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d): rows=%lld cols=%lld ld=%lld", (int)r,
              (long long)rows, (long long)cols, (long long)ld_bytes);
    return ZQ_ERR_CUDA;
  }
  return ZQ_OK;
}

// Shared with zq_attention.cu: 2-D float32 tensor map (row-major, ld in bytes).
int make_tmap_f32(CUtensorMap* tm, const void* base, int64_t rows, int64_t cols, int64_t ld_bytes,
                  int box_cols, int box_rows, CUtensorMapSwizzle sw) {
  if (!get_encode()) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return ZQ_ERR_CUDA;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld_bytes};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (f32) failed (%d): rows=%lld cols=%lld ld=%lld", (int)r,
              (long long)rows, (long long)cols, (long long)ld_bytes);
    return ZQ_ERR_CUDA;
  }
  return ZQ_OK;
}

int make_tmap_2d(CUtensorMap* tm, CUtensorMapDataType dt, const void* base, int64_t rows, int64_t cols,
                 int64_t ld_bytes, int box_cols, int box_rows, CUtensorMapSwizzle sw,
                 CUtensorMapL2promotion promo) {
  if (!get_encode()) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return ZQ_ERR_CUDA;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld_bytes};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(tm, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        sw, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d): dtype=%d rows=%lld cols=%lld ld=%lld box=%dx%d", (int)r, (int)dt,
              (long long)rows, (long long)cols, (long long)ld_bytes, box_cols, box_rows);
    return ZQ_ERR_CUDA;
  }
  return ZQ_OK;
}

static unsigned long long* g_trace = nullptr;
static int g_debug = 0;

template <int BN, int KIND, int W4>
static int launch_gemm_t(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc,
                         GemmParams p, cudaStream_t st) {
  using Cfg = GemmCfg<BN, W4>;
  static ZqDeviceOnce attr_once;
  attr_once([&](int) {
    cudaFuncSetAttribute(zq_gemm_kernel<BN, KIND, W4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Cfg::SMEM_BYTES);
  });
  const int g_num_sms = zq_num_sms();
  int grid = p.num_tiles < g_num_sms ? p.num_tiles : g_num_sms;
  const cudaError_t e = launch_kernel(zq_gemm_kernel<BN, KIND, W4>, dim3(grid), dim3(Cfg::NUM_THREADS),
                                      Cfg::SMEM_BYTES, st, 1, ta, tb, tc, p);
  if (e != cudaSuccess) {
    set_error("tcgen05 gemm launch: %s", cudaGetErrorString(e));
    return ZQ_ERR_CUDA;
  }
  return ZQ_OK;
}

template <int BN, int KIND, int CL>
static int launch_gemm2_t(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc, GemmParams p,
                          cudaStream_t st, const CUtensorMap* tkc = nullptr, const CUtensorMap* tvc = nullptr) {
  using Cfg = Gemm2Cfg<BN>;
  static ZqDeviceOnce attr_once;
  attr_once([&](int) {
    cudaFuncSetAttribute(zq_gemm2_kernel<BN, KIND, CL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Cfg::SMEM_BYTES);
  });
  const int units = (int)((int64_t)(p.num_tiles / p.num_n_tiles) * ((p.num_n_tiles + CL / 2 - 1) / (CL / 2)));
  // co-resident clusters: GPC boundaries can leave fewer than SMs / CL slots
  static std::atomic<int> max_clusters_dev[64];  // per device; 0 = not yet measured
  const int g_num_sms = zq_num_sms();
  int dev_ = 0;
  cudaGetDevice(&dev_);
  int max_clusters = max_clusters_dev[dev_ & 63].load(std::memory_order_relaxed);
  if (max_clusters <= 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CL * (g_num_sms / CL));
    cfg.blockDim = dim3(Cfg::NUM_THREADS);
    cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, zq_gemm2_kernel<BN, KIND, CL>, &cfg) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = g_num_sms / CL;
    }
    max_clusters = n < g_num_sms / CL ? n : g_num_sms / CL;
    max_clusters_dev[dev_ & 63].store(max_clusters, std::memory_order_relaxed);
    if (getenv("ZQ_GEMM_DEBUG")) fprintf(stderr, "[zq] gemm2 BN=%d CL=%d: %d co-resident clusters\n", BN, CL, max_clusters);
  }
  const int clusters = units < max_clusters ? units : max_clusters;
  const cudaError_t e = launch_kernel(zq_gemm2_kernel<BN, KIND, CL>, dim3(CL * clusters), dim3(Cfg::NUM_THREADS),
                                      Cfg::SMEM_BYTES, st, CL, ta, tb, tc, tkc ? *tkc : tc, tvc ? *tvc : tc, p);
  if (e != cudaSuccess) {
    set_error("tcgen05 cta-pair gemm launch: %s", cudaGetErrorString(e));
    return ZQ_ERR_CUDA;
  }
  return ZQ_OK;
}

template <int KIND, int W4>
static int launch_gemm_bn(int bn, const CUtensorMap& ta, const CUtensorMap& tb,
                          const CUtensorMap& tc, GemmParams p, cudaStream_t st) {
  switch (bn) {
    case 256: return launch_gemm_t<256, KIND, W4>(ta, tb, tc, p, st);
    case 128: return launch_gemm_t<128, KIND, W4>(ta, tb, tc, p, st);
    default: return launch_gemm_t<64, KIND, W4>(ta, tb, tc, p, st);
  }
}

// Pick BLOCK_N: largest tile that still gives >= ~1 wave on 148 SMs; small-N
// layers drop to 128/64 so the grid fills the machine.
static int pick_bn(int64_t M, int64_t N) {
  const int64_t mt = (M + BLOCK_M - 1) / BLOCK_M;
  const int cands[3] = {256, 128, 64};
  for (int i = 0; i < 3; ++i) {
    int bn = cands[i];
    int64_t tiles = mt * ((N + bn - 1) / bn);
    if (tiles >= zq_num_sms() || bn == 64) {
      if (bn > N && bn > 64) continue;
      return bn;
    }
  }
  return 64;
}

template <int MP, int KIND, int W4>
static int launch_skinny_t(const CUtensorMap& tw, const CUtensorMap& tx, GemmParams p, int S,
                           cudaStream_t st) {
  using Cfg = SkinnyCfg<MP, W4>;
  static ZqDeviceOnce attr_once;
  attr_once([&](int) {
    cudaFuncSetAttribute(zq_gemm_skinny_kernel<MP, KIND, W4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Cfg::SMEM_BYTES);
  });
  cudaError_t e = launch_kernel(zq_gemm_skinny_kernel<MP, KIND, W4>, dim3(p.num_n_tiles * S),
                                dim3(skinny_threads<MP, W4>()),
                                Cfg::SMEM_BYTES, st, S, tw, tx, p, S);
  if (e != cudaSuccess) {
    set_error("skinny gemm launch: %s", cudaGetErrorString(e));
    return ZQ_ERR_CUDA;
  }
  return ZQ_OK;
}

#ifndef ZQ_SKINNY_CTAS_PER_SM
#define ZQ_SKINNY_CTAS_PER_SM 1  // grids of <= 1 CTA per SM leave room for the next launch (PDL); 2 measured slower
#endif
// Split-K degree: the largest S (<= 8) whose grid still fits one wave of two
// CTAs per SM (a partial second wave costs more than the extra split saves) and
// leaves every split >= 2 k-blocks.
static int pick_split(int n_tiles, int nkb) {
  // (measured on the GPT-J / NeoX decode shapes: forcing S = 2..8, non-power-of-two
  // S (clusters of 3 / 6 co-schedule poorly) or filling two CTAs per SM never beat
  // this rule, tools/microbench.py skinny)
  int S = 1;
  while (S < 8 && n_tiles * S * 2 <= 2 * zq_num_sms() * ZQ_SKINNY_CTAS_PER_SM && nkb / (2 * S) >= 2) S *= 2;
  return S;
}

// out[m, n] = ((f32(S[n / 128][m][n % 128]) * s_tok[m]) * s_w[n]) + b[n] (igemm.py:107-111,
// strict order) from the stream-K sums, + the fused KV-cache append of the decode
// QKV projection; every sum is re-zeroed for the next launch.
template <int KIND>
__device__ __forceinline__ void sum_epi_store(const GemmParams& p, int m, int n, const int32_t (&a)[4], float st,
                                              const float4& w, const float4& bb) {
  const int64_t o = (int64_t)m * p.ld_out + n;
  if (KIND == OUT_S32) {
    *reinterpret_cast<int4*>(reinterpret_cast<int32_t*>(p.out) + o) = make_int4(a[0], a[1], a[2], a[3]);
    return;
  }
  const float wv[4] = {w.x, w.y, w.z, w.w}, bv[4] = {bb.x, bb.y, bb.z, bb.w};
  float f[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    f[j] = __fmul_rn(__fmul_rn(__int2float_rn(a[j]), st), wv[j]);
    if (p.bias) f[j] = __fadd_rn(f[j], bv[j]);
  }
  if (KIND == OUT_F32) {
    const float4 v = make_float4(f[0], f[1], f[2], f[3]);
    *reinterpret_cast<float4*>(reinterpret_cast<float*>(p.out) + o) = v;
    if (p.kc != nullptr && n >= p.kv_dl) {  // fused KV-cache append (decode QKV); dl % 4 == 0
      const int64_t slot = ((int64_t)m * p.kv_max_ctx + p.kv_pos[m]) * p.kv_dl;
      if (n < 2 * p.kv_dl) *reinterpret_cast<float4*>(p.kc + slot + (n - p.kv_dl)) = v;
      else *reinterpret_cast<float4*>(p.vc + slot + (n - 2 * p.kv_dl)) = v;
    }
  } else if (KIND == OUT_F16) {
    __half2 h0 = __floats2half2_rn(f[0], f[1]), h1 = __floats2half2_rn(f[2], f[3]);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&h0);
    u.y = *reinterpret_cast<uint32_t*>(&h1);
    *reinterpret_cast<uint2*>(reinterpret_cast<__half*>(p.out) + o) = u;
  } else {
    __nv_bfloat162 h0 = __floats2bfloat162_rn(f[0], f[1]), h1 = __floats2bfloat162_rn(f[2], f[3]);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&h0);
    u.y = *reinterpret_cast<uint32_t*>(&h1);
    *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(p.out) + o) = u;
  }
}

// out[m, n] = ((f32(S[n / 128][m][n % 128]) * s_tok[m]) * s_w[n]) + b[n] (igemm.py:107-111,
// strict order) from the stream-K sums, + the fused KV-cache append of the decode
// QKV projection; every sum is re-zeroed for the next launch.  One thread per 4
// consecutive columns of a row (all loads independent: one L2 round trip).
template <int KIND>
__global__ void __launch_bounds__(256) skinny_sum_epilogue_kernel(int32_t* __restrict__ ws, int mp, GemmParams p) {
  pdl_trigger();
  pdl_wait();
  const int n4 = p.N >> 2;
  const int total = p.M * n4;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int m = i / n4, n = (i - m * n4) * 4;
    int4* sp = reinterpret_cast<int4*>(ws + ((int64_t)(n >> 7) * mp + m) * 128 + (n & 127));
    const int4 a4 = __ldcg(sp);
    const float st = p.token_scales ? __ldg(p.token_scales + m) : p.static_scale;
    float4 w = make_float4(0.f, 0.f, 0.f, 0.f), bb = w;
    if (KIND != OUT_S32) {
      w = __ldg(reinterpret_cast<const float4*>(p.row_scales + n));
      if (p.bias) bb = __ldg(reinterpret_cast<const float4*>(p.bias + n));
    }
    *sp = make_int4(0, 0, 0, 0);
    const int32_t a[4] = {a4.x, a4.y, a4.z, a4.w};
    sum_epi_store<KIND>(p, m, n, a, st, w, bb);
  }
}

template <int MP, int KIND>
static int launch_streamk_t(const CUtensorMap& tw, const CUtensorMap& tx, const GemmParams& p, int grid,
                            cudaStream_t st) {
  using Cfg = StreamKCfg<MP>;
  static ZqDeviceOnce attr_once;
  attr_once([&](int) {
    cudaFuncSetAttribute(zq_gemm_streamk_kernel<MP, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Cfg::SMEM_BYTES);
  });
  cudaError_t e = launch_kernel(zq_gemm_streamk_kernel<MP, KIND>, dim3(grid), dim3(192), Cfg::SMEM_BYTES, st, 1, tw,
                                tx, p);
  if (e == cudaSuccess) {
    const int64_t total = (int64_t)p.M * (p.N / 4);
    const int eg = (int)std::min<int64_t>((total + 255) / 256, (int64_t)zq_num_sms() * 8);
    e = launch_kernel(skinny_sum_epilogue_kernel<KIND>, dim3(eg), dim3(256), 0, st, 1, p.sk_ws, MP, p);
  }
  if (e != cudaSuccess) {
    set_error("stream-K skinny gemm launch: %s", cudaGetErrorString(e));
    return ZQ_ERR_CUDA;
  }
  return ZQ_OK;
}

int64_t streamk_ws_bytes(int64_t M, int64_t N) {
  const int64_t nt = (N + 127) / 128, mp = M <= 32 ? 32 : 64;
  return 4 * nt * mp * 128;
}

static int sk_min_bytes() {
  static int v = -1;  // ZQ_GEMM_STREAMK_MIN: weight bytes from which decode GEMMs go stream-K
  if (v < 0) {
    const char* e = getenv("ZQ_GEMM_STREAMK_MIN");
    v = e ? atoi(e) : 0;
  }
  return v;
}

static int gemm_skinny(const int8_t* xq, int64_t ld_x, const void* wq, int64_t ld_w, int w_bits, int64_t M,
                       int64_t N, int64_t K, int kind, GemmParams p, cudaStream_t st) {
  const int MP = M <= 32 ? 32 : 64;
  CUtensorMap tw, tx;
  int rc = w_bits == 8 ? make_tmap_u8(&tw, wq, N, K, ld_w, BLOCK_K, 128, CU_TENSOR_MAP_SWIZZLE_128B)
                       : make_tmap_u8(&tw, wq, N, ld_w / 2, ld_w / 2, BLOCK_K / 2, 128, CU_TENSOR_MAP_SWIZZLE_NONE);
  if (rc) return rc;
  rc = make_tmap_u8(&tx, xq, M, K, ld_x, BLOCK_K, MP, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  p.M = (int)M;
  p.N = (int)N;
  p.K = (int)K;
  p.num_n_tiles = (int)((N + 127) / 128);
  p.num_k_blocks = (int)((K + BLOCK_K - 1) / BLOCK_K);
  p.num_tiles = p.num_n_tiles;
  static int sk_mode = -1;  // ZQ_GEMM_STREAMK=0: the cluster split-K kernel even with a workspace
  if (sk_mode < 0) {
    const char* e = getenv("ZQ_GEMM_STREAMK");
    sk_mode = e ? atoi(e) : 1;
  }
  // stream-K pays an extra (epilogue) launch; measured at GPT-J / NeoX decode it wins
  // at every width (GPT-J o 16.8 MB: 7.2 -> 6.2 us; NeoX h4h 151 MB: 33.8 -> 30.9 us,
  // tools/skinny_bench.py).  ZQ_GEMM_STREAMK_MIN (bytes) keeps smaller GEMMs on the
  // cluster split-K kernel.
  const bool sk_big = (int64_t)N * K >= (int64_t)sk_min_bytes();
  const int osz = (kind == OUT_F16 || kind == OUT_BF16) ? 2 : 4;
  const bool sk_aligned = N % 4 == 0 && (p.ld_out * osz) % 16 == 0 && (reinterpret_cast<uintptr_t>(p.out) & 15) == 0 &&
                          (reinterpret_cast<uintptr_t>(p.row_scales) & 15) == 0 &&
                          (p.bias == nullptr || (reinterpret_cast<uintptr_t>(p.bias) & 15) == 0) &&
                          (p.kc == nullptr || (p.kv_dl % 4 == 0 && (reinterpret_cast<uintptr_t>(p.kc) & 15) == 0 &&
                                               (reinterpret_cast<uintptr_t>(p.vc) & 15) == 0));
  if (w_bits == 8 && p.sk_ws != nullptr && sk_mode != 0 && sk_big && sk_aligned &&
      p.sk_ws_bytes >= streamk_ws_bytes(M, N) && (reinterpret_cast<uintptr_t>(p.sk_ws) & 15) == 0) {
    const int64_t units = (int64_t)p.num_n_tiles * p.num_k_blocks;
    static int sk_cps = -1;  // ZQ_GEMM_STREAMK_CPS: CTAs per SM (memory-level parallelism)
    if (sk_cps < 0) {
      const char* e = getenv("ZQ_GEMM_STREAMK_CPS");
      sk_cps = e ? atoi(e) : 2;
    }
    const int grid = (int)std::min<int64_t>(units, (int64_t)zq_num_sms() * sk_cps);
#define ZQ_SKK(KK) (MP == 32 ? launch_streamk_t<32, KK>(tw, tx, p, grid, st) : launch_streamk_t<64, KK>(tw, tx, p, grid, st))
    switch (kind) {
      case OUT_S32: return ZQ_SKK(OUT_S32);
      case OUT_F32: return ZQ_SKK(OUT_F32);
      case OUT_F16: return ZQ_SKK(OUT_F16);
      default: return ZQ_SKK(OUT_BF16);
    }
#undef ZQ_SKK
  }
  const int S = pick_split(p.num_n_tiles, p.num_k_blocks);
#define ZQ_SK(KK)                                                                               \
  (w_bits == 4 ? (MP == 32 ? launch_skinny_t<32, KK, 1>(tw, tx, p, S, st) : launch_skinny_t<64, KK, 1>(tw, tx, p, S, st)) \
               : (MP == 32 ? launch_skinny_t<32, KK, 0>(tw, tx, p, S, st) : launch_skinny_t<64, KK, 0>(tw, tx, p, S, st)))
  switch (kind) {
    case OUT_S32: return ZQ_SK(OUT_S32);
    case OUT_F32: return ZQ_SK(OUT_F32);
    case OUT_F16: return ZQ_SK(OUT_F16);
    default: return ZQ_SK(OUT_BF16);
  }
#undef ZQ_SK
}

int gemm2c_w4i8(const int8_t* xq, int64_t ld_x, const void* wq, int64_t ld_w, int64_t M, int64_t N, int64_t K,
                int kind, int bn, GemmParams p, cudaStream_t st);

// W4A8 CTA-pair kernel (zq_gemm_conv.cu); ZQ_GEMM_W4PAIR=0 keeps W4 on the 1-CTA kernel
static bool w4_pair_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ZQ_GEMM_W4PAIR");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}

static int gemm_common(const int8_t* xq, int64_t ld_x, const void* wq, int64_t ld_w, int w_bits,
                       int64_t M, int64_t N, int64_t K, int kind, GemmParams p,
                       cudaStream_t st) {
  ZQ_CHECK_ARG(w_bits == 8 || w_bits == 4, ZQ_ERR_USAGE, "unsupported weight bit width %d", w_bits);
  ZQ_CHECK_ARG(M >= 1 && N >= 1 && K >= 1, ZQ_ERR_SHAPE, "empty GEMM (%lld, %lld, %lld)",
               (long long)M, (long long)N, (long long)K);
  ZQ_CHECK_ARG(M < (1LL << 31) && N < (1LL << 31) && K < (1LL << 31), ZQ_ERR_UNSUPPORTED,
               "GEMM dimension too large");
  ZQ_CHECK_ARG(ld_x >= K && ld_x % 16 == 0, ZQ_ERR_USAGE, "activation row stride %lld must be >= K and a multiple of 16",
               (long long)ld_x);
  ZQ_CHECK_ARG(ld_w >= K && ld_w % 16 == 0 && (w_bits == 8 || ld_w % 32 == 0), ZQ_ERR_USAGE,
               "weight row stride %lld must be >= K and a multiple of 16 (32 for int4)",
               (long long)ld_w);
  ZQ_CHECK_ARG((reinterpret_cast<uintptr_t>(xq) & 15) == 0 && (reinterpret_cast<uintptr_t>(wq) & 15) == 0,
               ZQ_ERR_USAGE, "operands must be 16-byte aligned");
  // exactness guard (igemm.py:52-63): K * 127 * qmax_w < 2^31
  const int64_t qmw = w_bits == 8 ? 127 : 7;
  ZQ_CHECK_ARG(K * 127 * qmw < (1LL << 31), ZQ_ERR_USAGE,
               "igemm overflow guard: inner dim %lld with 8x%d-bit operands can reach >= 2^31",
               (long long)K, w_bits);
  if (!get_encode()) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return ZQ_ERR_CUDA;
  }
  const int g_num_sms = zq_num_sms();
  // decode-sized token counts: weight-streaming skinny kernel (ZQ_GEMM_SKINNY=0 disables)
  static int skinny_mode = -1;
  if (skinny_mode < 0) {
    const char* e = getenv("ZQ_GEMM_SKINNY");
    skinny_mode = e ? atoi(e) : 1;
  }
  if (M <= 64 && skinny_mode != 0) return gemm_skinny(xq, ld_x, wq, ld_w, w_bits, M, N, K, kind, p, st);
  // CTA-pair path for int8 weights when there are enough 256-row tiles to fill
  // the machine (ZQ_GEMM_PAIR=0 disables, =1 forces where legal)
  static int pair_mode = -1;
  if (pair_mode < 0) {
    const char* e = getenv("ZQ_GEMM_PAIR");
    pair_mode = e ? atoi(e) : 2;
  }
  if (pair_mode != 0 && (w_bits == 8 || w4_pair_enabled())) {
    const int64_t mp = (M + 2 * BLOCK_M - 1) / (2 * BLOCK_M);
    int bn2 = 0, cl2 = 2;
    static int force_bn2 = -1;
    if (force_bn2 < 0) {
      const char* e = getenv("ZQ_GEMM_BN2");
      force_bn2 = e ? atoi(e) : 0;
    }
    if (mp * ((N + 127) / 128) >= g_num_sms / 2 || pair_mode == 1) {
      // pair tile width from a per-SM cost model (measured on B200): per round a
      // CTA needs max(MMA, operand delivery through TMA at ~75 GB/s/SM, epilogue
      // stores at ~35 GB/s/SM); rounds = ceil(tiles / pairs)
      const int esz = (kind == OUT_F16 || kind == OUT_BF16) ? 2 : (kind == OUT_S32 ? 4 : 4);
      double best = 1e30;
      for (int cand : {256, 192, 128}) {
        if (cand > N && cand > 128) continue;
        if (w_bits == 4 && cand == 192) continue;  // W4 pair kernel: BN 256 / 128
        // CL = 4 (A multicast across two pairs) only when forced: clusters of 4 fit
        // 33 per GPU (GPC boundaries) against 74 pairs, and the ~5% per-SM gain
        // does not repay the 11% of SMs left idle (8192^3: 373 vs 350 us)
        for (int cl : {2}) {
          const int64_t nt = (N + cand - 1) / cand;
          if (cl == 4 && nt < 2) continue;
          const double units = (double)mp * (double)((nt + cl / 2 - 1) / (cl / 2));
          const double rounds = std::ceil(units / (g_num_sms / cl));
          const double t_mma = 128.0 * cand * K / 11.1e12;
          // operand delivery: the L2 -> SM rate (~75 GB/s per SM); with CL = 4 each
          // CTA pulls half of its A tile (the other half arrives by multicast)
          const double t_op = (128.0 / (cl / 2) + cand / 2) * K / 75e9;
          const double t_epi = 128.0 * cand * esz / 35e9;
          const double t = rounds * std::max(t_mma, std::max(t_op, t_epi)) + t_op;
          if (t < best * 0.97) {  // prefer the earlier (wider / simpler) choice unless clearly faster
            best = t;
            bn2 = cand;
            cl2 = cl;
          }
        }
      }
    }
    if (force_bn2 && bn2) bn2 = force_bn2;
    {
      static int force_cl = -1;
      if (force_cl < 0) {
        const char* e = getenv("ZQ_GEMM_CL");
        force_cl = e ? atoi(e) : 0;
      }
      if (bn2 && (force_cl == 2 || (force_cl == 4 && (N + bn2 - 1) / bn2 >= 2))) cl2 = force_cl;
    }
    if (bn2 && w_bits == 4) {
      if (p.kv_rows_per_seq > 0) return ZQ_ERR_UNSUPPORTED;
      p.trace = g_trace;
      p.debug = g_debug;
      return gemm2c_w4i8(xq, ld_x, wq, ld_w, M, N, K, kind, bn2 == 192 ? 256 : bn2, p, st);
    }
    if (bn2) {
      CUtensorMap ta, tb;
      int rc = make_tmap_u8(&ta, xq, M, K, ld_x, BLOCK_K, BLOCK_M, CU_TENSOR_MAP_SWIZZLE_128B);
      if (rc) return rc;
      rc = make_tmap_u8(&tb, wq, N, K, ld_w, BLOCK_K, bn2 / 2, CU_TENSOR_MAP_SWIZZLE_128B);
      if (rc) return rc;
      p.M = (int)M;
      p.N = (int)N;
      p.K = (int)K;
      p.trace = g_trace;
      p.debug = g_debug;
      const int esz = (kind == OUT_F16 || kind == OUT_BF16) ? 2 : 4;
      p.tma_out = ((reinterpret_cast<uintptr_t>(p.out) & 15) == 0) && ((p.ld_out * esz) % 16 == 0) &&
                  (p.row_scales == nullptr || (reinterpret_cast<uintptr_t>(p.row_scales) & 15) == 0) &&
                  (p.bias == nullptr || (reinterpret_cast<uintptr_t>(p.bias) & 15) == 0);
      CUtensorMap tc;
      memset(&tc, 0, sizeof(tc));
      if (p.tma_out) {
        cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)M};
        cuuint64_t strides[1] = {(cuuint64_t)(p.ld_out * esz)};
        cuuint32_t box[2] = {32, 32};
        cuuint32_t estr[2] = {1, 1};
        CUtensorMapDataType dt = kind == OUT_S32 ? CU_TENSOR_MAP_DATA_TYPE_INT32
                                 : kind == OUT_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                 : kind == OUT_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                   : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
        CUresult r = g_encode(&tc, dt, 2, p.out, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              esz == 4 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                              CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) p.tma_out = 0;
      }
      p.num_n_tiles = (int)((N + bn2 - 1) / bn2);
      p.num_tiles = (int)mp * p.num_n_tiles;
      p.num_k_blocks = (int)((K + BLOCK_K - 1) / BLOCK_K);
      p.group_m = K >= 2048 ? 8 : 1;  // operand-bound: keep A / B panels in L2
      CUtensorMap tkc, tvc;
      const CUtensorMap* pkc = nullptr;
      const CUtensorMap* pvc = nullptr;
      if (p.kv_rows_per_seq > 0) {  // prefill KV append through the epilogue (f32 output only)
        if (kind != OUT_F32 || !p.tma_out || p.kv_rows_per_seq % 32 != 0 || p.kv_dl % 32 != 0 ||
            M % p.kv_rows_per_seq != 0)
          return ZQ_ERR_UNSUPPORTED;
        const int64_t crows = (M / p.kv_rows_per_seq) * p.kv_max_ctx;
        int rk = make_tmap_2d(&tkc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, p.kc, crows, p.kv_dl, (int64_t)p.kv_dl * 4, 32,
                              32, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE);
        if (!rk) rk = make_tmap_2d(&tvc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, p.vc, crows, p.kv_dl, (int64_t)p.kv_dl * 4,
                                   32, 32, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE);
        if (rk) return rk;
        pkc = &tkc;
        pvc = &tvc;
      }
#define ZQ_G2C(KK, CC) (bn2 == 256 ? launch_gemm2_t<256, KK, CC>(ta, tb, tc, p, st, pkc, pvc) \
                        : bn2 == 192 ? launch_gemm2_t<192, KK, CC>(ta, tb, tc, p, st, pkc, pvc)  \
                                     : launch_gemm2_t<128, KK, CC>(ta, tb, tc, p, st, pkc, pvc))
#define ZQ_G2(KK) (cl2 == 4 ? ZQ_G2C(KK, 4) : ZQ_G2C(KK, 2))
      switch (kind) {
        case OUT_S32: return ZQ_G2(OUT_S32);
        case OUT_F32: return ZQ_G2(OUT_F32);
        case OUT_F16: return ZQ_G2(OUT_F16);
        default: return ZQ_G2(OUT_BF16);
      }
#undef ZQ_G2
    }
  }
  if (p.kv_rows_per_seq > 0) return ZQ_ERR_UNSUPPORTED;  // prefill KV append: CTA-pair path only
  const int bn = pick_bn(M, N);
  CUtensorMap ta, tb;
  int rc = make_tmap_u8(&ta, xq, M, K, ld_x, BLOCK_K, BLOCK_M, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  if (w_bits == 8) {
    rc = make_tmap_u8(&tb, wq, N, K, ld_w, BLOCK_K, bn, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
  } else {
    // packed rows: ld_w/2 bytes (zero past K), box 64 B x bn rows, no swizzle
    rc = make_tmap_u8(&tb, wq, N, ld_w / 2, ld_w / 2, BLOCK_K / 2, bn, CU_TENSOR_MAP_SWIZZLE_NONE);
    if (rc) return rc;
    p.w4 = reinterpret_cast<const uint8_t*>(wq);
    p.ld_w4 = ld_w / 2;
  }
  p.M = (int)M;
  p.N = (int)N;
  p.K = (int)K;
  p.trace = g_trace;
  p.debug = g_debug;
  CUtensorMap tc;
  memset(&tc, 0, sizeof(tc));
  {
    const int esz = (kind == OUT_F16 || kind == OUT_BF16) ? 2 : 4;
    const bool scales_ok =
        (p.row_scales == nullptr || (reinterpret_cast<uintptr_t>(p.row_scales) & 15) == 0) &&
        (p.bias == nullptr || (reinterpret_cast<uintptr_t>(p.bias) & 15) == 0);
    p.tma_out = ((reinterpret_cast<uintptr_t>(p.out) & 15) == 0) && ((p.ld_out * esz) % 16 == 0) &&
                scales_ok;
    if (p.tma_out) {
      cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)M};
      cuuint64_t strides[1] = {(cuuint64_t)(p.ld_out * esz)};
      cuuint32_t box[2] = {32, 32};
      cuuint32_t estr[2] = {1, 1};
      CUtensorMapDataType dt = kind == OUT_S32 ? CU_TENSOR_MAP_DATA_TYPE_INT32
                               : kind == OUT_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                               : kind == OUT_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
      CUresult r = g_encode(&tc, dt, 2, p.out, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE,
                            esz == 4 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) p.tma_out = 0;
    }
  }
  p.num_n_tiles = (int)((N + bn - 1) / bn);
  p.num_tiles = (int)((M + BLOCK_M - 1) / BLOCK_M) * p.num_n_tiles;
  p.num_k_blocks = (int)((K + BLOCK_K - 1) / BLOCK_K);
  p.group_m = K >= 2048 ? 8 : 1;
  const bool w4 = w_bits == 4;
  switch (kind) {
    case OUT_S32: return w4 ? launch_gemm_bn<OUT_S32, 1>(bn, ta, tb, tc, p, st) : launch_gemm_bn<OUT_S32, 0>(bn, ta, tb, tc, p, st);
    case OUT_F32: return w4 ? launch_gemm_bn<OUT_F32, 1>(bn, ta, tb, tc, p, st) : launch_gemm_bn<OUT_F32, 0>(bn, ta, tb, tc, p, st);
    case OUT_F16: return w4 ? launch_gemm_bn<OUT_F16, 1>(bn, ta, tb, tc, p, st) : launch_gemm_bn<OUT_F16, 0>(bn, ta, tb, tc, p, st);
    default: return w4 ? launch_gemm_bn<OUT_BF16, 1>(bn, ta, tb, tc, p, st) : launch_gemm_bn<OUT_BF16, 0>(bn, ta, tb, tc, p, st);
  }
}

}  // namespace zq

using namespace zq;

extern "C" {

const char* zq_version(void) { return "zq_b200 0.1.0 sm_100a tcgen05-i8"; }

int zq_gemm_set_trace(unsigned long long* buf) {
  g_trace = buf;
  const char* e = getenv("ZQ_GEMM_DEBUG");
  g_debug = e ? atoi(e) : 0;
  return ZQ_OK;
}

int zq_igemm_s32(const int8_t* xq, int64_t ld_x, const void* wq, int64_t ld_w, int w_bits,
                 int64_t M, int64_t N, int64_t K, int32_t* acc, int64_t ld_acc, void* stream) {
  ZQ_CHECK_ARG(ld_acc >= N, ZQ_ERR_USAGE, "accumulator row stride too small");
  GemmParams p;
  memset(&p, 0, sizeof(p));
  p.out = acc;
  p.ld_out = ld_acc;
  return gemm_common(xq, ld_x, wq, ld_w, w_bits, M, N, K, OUT_S32, p,
                     reinterpret_cast<cudaStream_t>(stream));
}

int zq_igemm_s32_ws(const int8_t* xq, int64_t ld_x, const void* wq, int64_t ld_w, int w_bits, int64_t M, int64_t N,
                    int64_t K, int32_t* acc, int64_t ld_acc, void* workspace, int64_t workspace_bytes, void* stream) {
  ZQ_CHECK_ARG(ld_acc >= N, ZQ_ERR_USAGE, "accumulator row stride too small");
  GemmParams p;
  memset(&p, 0, sizeof(p));
  p.out = acc;
  p.ld_out = ld_acc;
  p.sk_ws = reinterpret_cast<int32_t*>(workspace);
  p.sk_ws_bytes = workspace_bytes;
  return gemm_common(xq, ld_x, wq, ld_w, w_bits, M, N, K, OUT_S32, p, reinterpret_cast<cudaStream_t>(stream));
}

int zq_linear(const int8_t* xq, int64_t ld_x, const float* token_scales, float static_scale,
              const void* wq, int64_t ld_w, int w_bits, const float* w_row_scales,
              const float* bias, int64_t M, int64_t N, int64_t K, void* out, int64_t ld_out,
              int out_type, void* stream) {
  ZQ_CHECK_ARG(out_type >= ZQ_OUT_F32 && out_type <= ZQ_OUT_BF16, ZQ_ERR_USAGE, "bad output type %d", out_type);
  ZQ_CHECK_ARG(w_row_scales != nullptr, ZQ_ERR_USAGE, "weight row scales required");
  ZQ_CHECK_ARG(ld_out >= N, ZQ_ERR_USAGE, "output row stride too small");
  GemmParams p;
  memset(&p, 0, sizeof(p));
  p.out = out;
  p.ld_out = ld_out;
  p.token_scales = token_scales;
  p.static_scale = static_scale;
  p.row_scales = w_row_scales;
  p.bias = bias;
  const int kind = out_type == ZQ_OUT_F32 ? OUT_F32 : out_type == ZQ_OUT_F16 ? OUT_F16 : OUT_BF16;
  return gemm_common(xq, ld_x, wq, ld_w, w_bits, M, N, K, kind, p,
                     reinterpret_cast<cudaStream_t>(stream));
}

int64_t zq_linear_ws_bytes(int64_t M, int64_t N) { return streamk_ws_bytes(M, N); }

int zq_linear_ws(const int8_t* xq, int64_t ld_x, const float* token_scales, float static_scale, const void* wq,
                 int64_t ld_w, int w_bits, const float* w_row_scales, const float* bias, int64_t M, int64_t N,
                 int64_t K, void* out, int64_t ld_out, int out_type, void* workspace, int64_t workspace_bytes,
                 void* stream) {
  ZQ_CHECK_ARG(out_type >= ZQ_OUT_F32 && out_type <= ZQ_OUT_BF16, ZQ_ERR_USAGE, "bad output type %d", out_type);
  ZQ_CHECK_ARG(w_row_scales != nullptr, ZQ_ERR_USAGE, "fused linear needs weight scales");
  GemmParams p;
  memset(&p, 0, sizeof(p));
  p.out = out;
  p.ld_out = ld_out;
  p.token_scales = token_scales;
  p.static_scale = static_scale;
  p.row_scales = w_row_scales;
  p.bias = bias;
  p.sk_ws = reinterpret_cast<int32_t*>(workspace);
  p.sk_ws_bytes = workspace_bytes;
  return gemm_common(xq, ld_x, wq, ld_w, w_bits, M, N, K, out_type + 1, p, reinterpret_cast<cudaStream_t>(stream));
}

int zq_linear_kv_prefill(const int8_t* xq, int64_t ld_x, const float* token_scales, const void* wq, int64_t ld_w,
                         int w_bits, const float* w_row_scales, const float* bias, int64_t M, int64_t N, int64_t K,
                         float* out, int64_t ld_out, float* kcache, float* vcache, int dmodel_local, int64_t max_ctx,
                         int rows_per_seq, void* stream) {
  ZQ_CHECK_ARG(w_row_scales != nullptr && kcache && vcache, ZQ_ERR_USAGE, "linear + kv append needs every operand");
  ZQ_CHECK_ARG(N == 3LL * dmodel_local && ld_out >= N, ZQ_ERR_SHAPE, "qkv output must be 3 x dmodel_local wide");
  ZQ_CHECK_ARG(rows_per_seq >= 1 && rows_per_seq <= max_ctx && M % rows_per_seq == 0, ZQ_ERR_SHAPE,
               "prefill rows must be whole sequences of <= max_ctx tokens");
  GemmParams p;
  memset(&p, 0, sizeof(p));
  p.out = out;
  p.ld_out = ld_out;
  p.token_scales = token_scales;
  p.row_scales = w_row_scales;
  p.bias = bias;
  p.kc = kcache;
  p.vc = vcache;
  p.kv_dl = dmodel_local;
  p.kv_max_ctx = max_ctx;
  p.kv_rows_per_seq = rows_per_seq;
  if (M <= 64) return ZQ_ERR_UNSUPPORTED;
  return gemm_common(xq, ld_x, wq, ld_w, w_bits, M, N, K, OUT_F32, p, reinterpret_cast<cudaStream_t>(stream));
}

int zq_linear_kv(const int8_t* xq, int64_t ld_x, const float* token_scales, const void* wq, int64_t ld_w,
                 int w_bits, const float* w_row_scales, const float* bias, int64_t M, int64_t N, int64_t K,
                 float* out, int64_t ld_out, float* kcache, float* vcache, const int32_t* pos, int dmodel_local,
                 int64_t max_ctx, void* stream) {
  return zq_linear_kv_ws(xq, ld_x, token_scales, wq, ld_w, w_bits, w_row_scales, bias, M, N, K, out, ld_out, kcache,
                         vcache, pos, dmodel_local, max_ctx, nullptr, 0, stream);
}

int zq_linear_kv_ws(const int8_t* xq, int64_t ld_x, const float* token_scales, const void* wq, int64_t ld_w,
                    int w_bits, const float* w_row_scales, const float* bias, int64_t M, int64_t N, int64_t K,
                    float* out, int64_t ld_out, float* kcache, float* vcache, const int32_t* pos, int dmodel_local,
                    int64_t max_ctx, void* workspace, int64_t workspace_bytes, void* stream) {
  ZQ_CHECK_ARG(w_row_scales != nullptr && kcache && vcache && pos, ZQ_ERR_USAGE, "linear + kv append needs every operand");
  ZQ_CHECK_ARG(N == 3LL * dmodel_local && ld_out >= N, ZQ_ERR_SHAPE, "qkv output must be 3 x dmodel_local wide");
  static int skinny_mode = -1;
  if (skinny_mode < 0) {
    const char* e = getenv("ZQ_GEMM_SKINNY");
    skinny_mode = e ? atoi(e) : 1;
  }
  if (M > 64 || skinny_mode == 0) return ZQ_ERR_UNSUPPORTED;  // prefill: linear, then zq_kv_append
  GemmParams p;
  memset(&p, 0, sizeof(p));
  p.out = out;
  p.ld_out = ld_out;
  p.token_scales = token_scales;
  p.row_scales = w_row_scales;
  p.bias = bias;
  p.kc = kcache;
  p.vc = vcache;
  p.kv_pos = pos;
  p.kv_dl = dmodel_local;
  p.kv_max_ctx = max_ctx;
  p.sk_ws = reinterpret_cast<int32_t*>(workspace);
  p.sk_ws_bytes = workspace_bytes;
  return gemm_common(xq, ld_x, wq, ld_w, w_bits, M, N, K, OUT_F32, p, reinterpret_cast<cudaStream_t>(stream));
}

int zq_linear_ln_quantize(const int8_t* xq, int64_t ld_x, const float* token_scales, const void* wq,
                          int64_t ld_w, int w_bits, const float* w_row_scales, const float* bias, int64_t M,
                          int64_t N, int64_t K, const float* residual, const float* gamma, const float* beta,
                          float eps, int bits, float* ln_out, int8_t* q, int64_t ld_q, float* q_scales,
                          void* workspace, int64_t workspace_bytes, int32_t* flag, void* stream) {
  ZQ_CHECK_ARG(bits == 8 || bits == 4, ZQ_ERR_USAGE, "unsupported bit width %d", bits);
  ZQ_CHECK_ARG(token_scales && w_row_scales && bias && residual && gamma && beta && ln_out && q && q_scales &&
                   workspace,
               ZQ_ERR_USAGE, "fused linear + LN needs every operand");
  ZQ_CHECK_ARG(ld_q >= N && ld_q % 16 == 0, ZQ_ERR_USAGE, "bad quantized row stride");
  // numpy's pairwise tree over N must be balanced with leaves of L <= 128 (L % 8 == 0):
  // the pair tile is 2 leaves wide and NT = N / (2L) tiles (a power of two) span a row
  int64_t L = N;
  while (L > 128) {
    if ((L / 2) % 8 != 0 || L % 2 != 0) return ZQ_ERR_UNSUPPORTED;
    L /= 2;
  }
  if (w_bits != 8 || L % 8 != 0 || (L != 96 && L != 128) || N < 2 * L) return ZQ_ERR_UNSUPPORTED;
  const int BN = (int)(2 * L);
  const int NT = (int)(N / BN);
  if ((NT & (NT - 1)) != 0 || NT > 64) return ZQ_ERR_UNSUPPORTED;
  const int g_num_sms = zq_num_sms();
  const int npairs = g_num_sms / 2;
  if (NT > npairs) return ZQ_ERR_UNSUPPORTED;
  const int64_t rblocks = (M + 255) / 256;
  const int64_t need = (int64_t)sizeof(unsigned int) * rblocks + 16 + (int64_t)sizeof(float) * 3 * M * NT;
  ZQ_CHECK_ARG(workspace_bytes >= need, ZQ_ERR_USAGE, "workspace too small (%lld < %lld bytes)",
               (long long)workspace_bytes, (long long)need);
  ZQ_CHECK_ARG(K * 127 * 127 < (1LL << 31), ZQ_ERR_USAGE, "igemm overflow guard");
  ZQ_CHECK_ARG(ld_x >= K && ld_x % 16 == 0 && ld_w >= K && ld_w % 16 == 0, ZQ_ERR_USAGE, "bad operand strides");
  if (!get_encode()) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return ZQ_ERR_CUDA;
  }
  CUtensorMap ta, tb;
  int rc = make_tmap_u8(&ta, xq, M, K, ld_x, BLOCK_K, BLOCK_M, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  rc = make_tmap_u8(&tb, wq, N, K, ld_w, BLOCK_K, BN / 2, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  GemmParams p;
  memset(&p, 0, sizeof(p));
  p.M = (int)M;
  p.N = (int)N;
  p.K = (int)K;
  p.token_scales = token_scales;
  p.row_scales = w_row_scales;
  p.bias = bias;
  p.num_n_tiles = NT;
  p.num_tiles = (int)(rblocks * NT);
  p.num_k_blocks = (int)((K + BLOCK_K - 1) / BLOCK_K);
  {
    const char* e = getenv("ZQ_FUSE_DEBUG");  // diagnostics: 4 = skip the exchange waits (wrong results)
    p.debug = e ? atoi(e) : 0;
  }
  LnFuseParams f;
  f.residual = residual;
  f.gamma = gamma;
  f.beta = beta;
  f.eps = eps;
  f.ln_out = ln_out;
  f.q = q;
  f.ld_q = ld_q;
  f.q_scales = q_scales;
  f.qm = (1 << (bits - 1)) - 1;
  f.counters = reinterpret_cast<unsigned int*>(workspace);
  f.partials = reinterpret_cast<float*>(reinterpret_cast<char*>(workspace) +
                                        ((sizeof(unsigned int) * rblocks + 15) / 16) * 16);
  f.flag = flag;
  f.tiles_per_round = (npairs / NT) * NT;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  return BN == 192 ? launch_gemm2_ln_t<192>(ta, tb, p, f, 2 * npairs, st)
                   : launch_gemm2_ln_t<256>(ta, tb, p, f, 2 * npairs, st);
}

int zq_dequant_epilogue(const int32_t* acc, int64_t ld_acc, const float* token_scales,
                        float static_scale, const float* w_row_scales, const float* bias,
                        int64_t M, int64_t N, void* out, int64_t ld_out, int out_type,
                        void* stream) {
  ZQ_CHECK_ARG(out_type >= ZQ_OUT_F32 && out_type <= ZQ_OUT_BF16, ZQ_ERR_USAGE, "bad output type %d", out_type);
  ZQ_CHECK_ARG(M >= 1 && N >= 1 && ld_acc >= N && ld_out >= N, ZQ_ERR_SHAPE, "bad epilogue shape");
  auto al16 = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; };
  if (N % 4 == 0 && ld_acc % 4 == 0 && ld_out % 4 == 0 && M * (N / 4) < (1LL << 31) && al16(acc) && al16(out) &&
      al16(w_row_scales) && (bias == nullptr || al16(bias))) {
    const int64_t total = M * (N / 4);
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, (int64_t)zq_num_sms() * 8);
    const cudaError_t e = launch_kernel(epilogue_vec_kernel, dim3(blocks), dim3(256), 0,
                                        reinterpret_cast<cudaStream_t>(stream), 1, acc, ld_acc, token_scales,
                                        static_scale, w_row_scales, bias, (int)M, (int)N, out, ld_out, out_type);
    if (e != cudaSuccess) {
      set_error("epilogue launch: %s", cudaGetErrorString(e));
      return ZQ_ERR_CUDA;
    }
    return ZQ_OK;
  }
  int64_t total = M * N;
  int blocks = (int)((total + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  epilogue_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      acc, ld_acc, token_scales, static_scale, w_row_scales, bias, M, N, out, ld_out, out_type);
  ZQ_LAUNCH_CHECK("epilogue launch");
  return ZQ_OK;
}

int zq_linear_full(const float* x, int64_t ld_x, const void* wq, int64_t ld_w, int w_bits,
                   const float* w_row_scales, const float* bias, int64_t M, int64_t N,
                   int64_t K, float* out, int64_t ld_out, void* stream) {
  ZQ_CHECK_ARG(w_bits == 8 || w_bits == 4, ZQ_ERR_USAGE, "unsupported weight bit width %d", w_bits);
  ZQ_CHECK_ARG(M >= 1 && N >= 1 && K >= 1 && ld_x >= K && ld_w >= K && ld_out >= N, ZQ_ERR_SHAPE,
               "bad full-precision linear shape");
  dim3 grid((unsigned)((N + 31) / 32), (unsigned)((M + 31) / 32));
  full_linear_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      x, ld_x, w_bits == 8 ? reinterpret_cast<const int8_t*>(wq) : nullptr,
      w_bits == 4 ? reinterpret_cast<const uint8_t*>(wq) : nullptr, ld_w, w_row_scales, bias, M, N,
      K, out, ld_out);
  ZQ_LAUNCH_CHECK("full linear launch");
  return ZQ_OK;
}

}  // extern "C"
