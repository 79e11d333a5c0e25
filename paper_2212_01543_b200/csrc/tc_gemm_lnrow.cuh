// Residual projection + LayerNorm with the whole d = 512 row in ONE CTA's
// accumulator (the north star's "residual+LayerNorm epilogue", full-row form):
//
//     x[M, 512] += A[M, K] . W[512, K]^T + bias      (infer.py:204-205, :210-212)
//     y[M, 512]  = LN(x) * g + b  (bf16, optionally  (kernels.py:42-57)
//                  gathered to rows out_row[r])
//
// Work unit = a vertical pair of 128-row blocks on a CTA pair (cluster of 2,
// one TPC): each CTA owns one block and all 512 columns, a 128 x 512 fp32
// accumulator that fills its SM's whole TMEM. The MMAs are cta_group::2
// (M = 256 across the pair, issued by the leader CTA): per 16-deep k-step two
// N = 256 instructions, each reading A's 128 rows from both CTAs' shared
// memory and B's 256 rows as 128 + 128 from the two CTAs. So a CTA stages only
// A (128 rows) + a quarter of the 512-row weight slab per k-block (48 KB), and
// the L2 -> SM operand stream is 128 + 256 rows per CTA instead of 128 + 512.
// Both CTAs' TMA loads complete on the leader's full barrier; the leader's
// MMA commits multicast to both CTAs' empty / accumulator-full barriers, and
// both CTAs' epilogue warps release the accumulator on the leader's barrier.
//
// Epilogue, 8 warps (TMEM lane quarter q, column half h = 256 columns):
//   pass 1  acc + bias + x -> x (fp32; each 32 x 32 chunk transposed through a
//           per-warp smem buffer so global accesses are coalesced 4-row x
//           128-byte groups); per-row partial mean / M2 of the warp's 256
//           columns (Chan merges of 32-column chunks); with KEEP the updated
//           chunk is also written back into its TMEM columns (tcgen05.st);
//   swap    the two warps of a lane quarter exchange row partials through
//           shared memory (named barrier of 64 threads), merged in a fixed
//           order (half 0, then half 1);
//   pass 2  y = (x - mean) rstd g + b as bf16, x read back from TMEM (KEEP:
//           no second pass over memory; the accumulator is released after
//           pass 2) or re-read from L2 (!KEEP: the accumulator is released
//           after pass 1, so the next unit's MMAs overlap pass 2).
// No LayerNorm launch, no DSMEM traffic.
#pragma once
#include "common.cuh"
#include "sm100_ptx.cuh"
#include "tc_gemm.cuh"
#include "tc_gemm_ln.cuh"

namespace hrt {

constexpr int LR_D = 512;
constexpr int LR_SLOTS_MAX = 6;

// STG: per-warp 32 x 32 fp32 buffers outside the operand ring (the register epilogues'
// transpose buffers; MODE 2 with a 3-stage ring: each warp's first residual slot)
template <int STAGES, bool STG>
struct LrSmem {
  static constexpr int A_BYTES = TC_BM * TC_BK * 2;          // 16 KB: this CTA's 128 rows
  static constexpr int BQ_BYTES = (LR_D / 4) * TC_BK * 2;    // 16 KB: 128 weight rows per N = 256 half
  static constexpr int STAGE_BYTES = A_BYTES + 2 * BQ_BYTES;  // 48 KB
  static constexpr int STG_OFFSET = STAGES * STAGE_BYTES;
  static constexpr int STG_BYTES = STG ? TC_EPI_WARPS * 32 * TC_STG_LD * 4 : 0;
  static constexpr int ST_OFFSET = STG_OFFSET + STG_BYTES;   // row statistics [2 parity][2 halves][128] float2
  static constexpr int ST_BYTES = 2 * 2 * TC_BM * 8;
  static constexpr int PRM_OFFSET = ST_OFFSET + ST_BYTES;  // bias, LN gain, LN bias [3][512] fp32
  static constexpr int PRM_BYTES = 3 * LR_D * 4;
  static constexpr int BAR_OFFSET = PRM_OFFSET + PRM_BYTES;
  static constexpr int TOTAL = BAR_OFFSET + 512 + 1024;
  // MODE 2 residual slots per epilogue warp: 4 KB slices of the ring (+ the STG buffer)
  static constexpr int RING_SLOTS = (STAGES * STAGE_BYTES / (4096 * TC_EPI_WARPS)) < (STG ? LR_SLOTS_MAX - 1 : LR_SLOTS_MAX)
                                        ? STAGES * STAGE_BYTES / (4096 * TC_EPI_WARPS)
                                        : (STG ? LR_SLOTS_MAX - 1 : LR_SLOTS_MAX);
  static constexpr int SLOTS = RING_SLOTS + (STG ? 1 : 0);
};
template <int STAGES, int MODE>
__host__ __device__ constexpr bool lr_stg() {
  return MODE != 2 || STAGES < 4;
}

template <int STAGES, int MODE>
__global__ void __launch_bounds__(TC_THREADS, 1)
    tc_gemm_resln_row_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                             const __grid_constant__ CUtensorMap tmX, int M, int K, const int* __restrict__ M_dev,
                             ResLnArgs ep) {
  constexpr bool USE_STG = lr_stg<STAGES, MODE>();
  using L = LrSmem<STAGES, USE_STG>;
  constexpr bool KEEP = MODE != 0;
  constexpr int NSL = L::SLOTS;
  constexpr int CL = 2;
  constexpr int HB = LR_D / 2;  // columns per MMA instruction (N = 256)
  constexpr int QB = LR_D / 4;  // weight rows per CTA per N half
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float2* stats = reinterpret_cast<float2*>(smem + L::ST_OFFSET);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::BAR_OFFSET);  // leader's: both CTAs' bytes
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 1;  // leader's: both CTAs' epilogue warps
  uint64_t* ring_free = tempty + 1;  // MODE 2: the epilogue gave the operand ring back
  uint64_t* xbar = ring_free + 1;    // MODE 2: [8 warps][5 slots] residual chunk arrivals
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xbar + TC_EPI_WARPS * LR_SLOTS_MAX);

  pdl_trigger();
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_kb = K / TC_BK;
  const int crank = (int)cluster_ctarank();
  const bool leader = crank == 0;
  const int cid = blockIdx.x / CL, ncl = gridDim.x / CL;
  constexpr uint32_t TMEM_COLS = 512;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, CL * TC_EPI_WARPS);
    mbar_init(ring_free, TC_EPI_WARPS);
    for (int j = 0; j < TC_EPI_WARPS * LR_SLOTS_MAX; ++j) mbar_init(&xbar[j], 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, TMEM_COLS);
  // per-column epilogue parameters (weights: independent of the previous kernel) staged once
  float* prm = reinterpret_cast<float*>(smem + L::PRM_OFFSET);
  for (int j = threadIdx.x; j < LR_D / 4; j += TC_THREADS) {
    reinterpret_cast<float4*>(prm)[j] = __ldg(reinterpret_cast<const float4*>(ep.bias) + j);
    reinterpret_cast<float4*>(prm + LR_D)[j] = __ldg(reinterpret_cast<const float4*>(ep.g) + j);
    reinterpret_cast<float4*>(prm + 2 * LR_D)[j] = __ldg(reinterpret_cast<const float4*>(ep.b) + j);
  }
  tc_fence_before();
  cluster_sync_all();  // both CTAs' barriers initialised (and TMEM allocated) before any cross-CTA signal
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t full_l = mapa_shared(smem_u32(full), 0);  // the leader's full barriers (cluster address)

  // the first STAGES weight quarter-slabs do not depend on the previous kernel (PDL overlap)
  int pre = 0;
  if (warp == 0 && lane == 0) {
    pre = min(STAGES, num_kb);
    const uint64_t pol = policy_evict_last();
    for (int s2 = 0; s2 < pre; ++s2) {
      if (leader) mbar_arrive_expect_tx(&full[s2], CL * L::STAGE_BYTES);
      uint8_t* sb = smem + s2 * L::STAGE_BYTES + L::A_BYTES;
#pragma unroll
      for (int h = 0; h < 2; ++h)
        tma_load_2d_pair(sb + h * L::BQ_BYTES, &tmB, full_l + 8u * s2, s2 * TC_BK, h * HB + crank * QB, pol);
    }
  }
  pdl_wait();
  if (M_dev != nullptr) M = *M_dev;
  const int m_tiles = (M + TC_BM - 1) / TC_BM;
  const int num_units = (m_tiles + CL - 1) / CL;

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer (both CTAs) =====
      const uint64_t pol_w = policy_evict_last();
      const uint64_t pol_a = policy_evict_first();
      int stage = 0;
      uint32_t phase = 0;
      int pu = 0;
      for (int u = cid; u < num_units; u += ncl, ++pu) {
        const int m0 = (u * CL + crank) * TC_BM;
        // MODE 2: the previous unit's epilogue staged residual chunks in the ring
        if (MODE == 2 && pu > 0) mbar_wait(ring_free, (pu - 1) & 1);
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * L::STAGE_BYTES;
          const uint32_t fb = full_l + 8u * stage;
          if (!(u == cid && kb < pre)) {
            if (leader) mbar_arrive_expect_tx(&full[stage], CL * L::STAGE_BYTES);
#pragma unroll
            for (int h = 0; h < 2; ++h)
              tma_load_2d_pair(sa + L::A_BYTES + h * L::BQ_BYTES, &tmB, fb, kb * TC_BK, h * HB + crank * QB, pol_w);
          }
          tma_load_2d_pair(sa, &tmA, fb, kb * TC_BK, m0, pol_a);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      if (cid >= num_units) {  // no rows after all: the armed stages still expect their A tiles
        for (int s2 = 0; s2 < pre; ++s2)
          tma_load_2d_pair(smem + s2 * L::STAGE_BYTES, &tmA, full_l + 8u * s2, s2 * TC_BK, 0, pol_a);
        if (leader)
          for (int s2 = 0; s2 < pre; ++s2) mbar_wait(&full[s2], 0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ===== MMA issuer (leader CTA): two N = 256 halves of the 512-column accumulator per k-step =====
      constexpr uint32_t idesc = idesc_bf16_f32(CL * TC_BM, HB);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int u = cid; u < num_units; u += ncl, ++it) {
        mbar_wait(tempty, (it & 1) ^ 1);  // both CTAs' epilogues released the accumulator
        tc_fence_after();
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * L::STAGE_BYTES);
          const uint32_t sb = sa + L::A_BYTES;
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int k = 0; k < TC_BK / 16; ++k)
              tc_mma_f16_pair(tmem_base + h * HB, sdesc_kmajor_sw128(sa + k * 32),
                              sdesc_kmajor_sw128(sb + h * L::BQ_BYTES + k * 32), idesc, (kb | k) != 0);
          tc_commit_pair_mc(&empty[stage], (uint16_t)3);  // the stage is free in both CTAs
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit_pair_mc(tfull, (uint16_t)3);
      }
    }
  } else if constexpr (MODE == 2) {
    // ===== epilogue, TMA-staged, one row per lane: warp (quarter q, half h) owns rows
    // 32 q .. 32 q + 31 (lane = row, the TMEM lane it may access), columns 256 h .. +255 =====
    // Residual chunks (32 x 32 fp32, 128-byte swizzle) stream in by TMA up to four chunks
    // ahead through 5 slots per warp: its transpose buffer plus 4 KB slices of the operand
    // ring, which is idle while the single accumulator drains (the producer waits on
    // ring_free before the next unit); updated chunks leave by TMA tile stores.
    const int ew = warp - 2;
    const int quarter = warp & 3;
    const int half = ew >> 2;
    const int cbeg = half * HB;
    constexpr int NCH = HB / 32;  // chunks per warp per pass
    // slot 0 is the warp's STG buffer when the ring leaves room for one (it can be filled
    // while the MMAs still use the ring: the next unit's first chunk is requested early)
    uint8_t* ring = smem + ew * (L::RING_SLOTS * 4096);
    auto slot_ptr = [&](int sl) {
      if constexpr (USE_STG) return sl == 0 ? smem + L::STG_OFFSET + ew * 4096 : ring + (sl - 1) * 4096;
      else return ring + sl * 4096;
    };
    uint64_t* xb = xbar + ew * LR_SLOTS_MAX;
    uint32_t ph = 0;  // per-slot phase bits
    auto load_chunk = [&](int sl, int c, int rblk) {  // lane 0
      mbar_arrive_expect_tx(&xb[sl], 4096);
      tma_load_2d(slot_ptr(sl), &tmX, &xb[sl], c, rblk);
    };
    if (USE_STG && cid < num_units && lane == 0) load_chunk(0, cbeg, (cid * CL + crank) * TC_BM + quarter * 32);
    int it = 0;
    for (int u = cid; u < num_units; u += ncl, ++it) {
      const int rblk = (u * CL + crank) * TC_BM + quarter * 32;  // this warp's 32-row block
      const int row = rblk + lane;
      const bool full_blk = rblk + 32 <= M;
      mbar_wait(tfull, it & 1);
      tc_fence_after();
      // the operand ring is idle now: chunks 1..3 go straight in
      if (lane == 0)
        for (int j = USE_STG ? 1 : 0; j < NSL - 1 && j < NCH; ++j) load_chunk(j, cbeg + 32 * j, rblk);
      const uint32_t tbase = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16);
      // ---- pass 1: x += acc + bias (TMA in / out), row statistics, x kept in TMEM ----
      float cnt = 0.f, rmean = 0.f, rm2 = 0.f;
#pragma unroll 1
      for (int j = 0; j < NCH; ++j) {
        const int c = cbeg + 32 * j;
        const int sl = j % NSL;
        float v[32];
        tmem_ld32(tbase + c, v);
        mbar_wait(&xb[sl], (ph >> sl) & 1);
        ph ^= 1u << sl;
        const uint32_t sa = smem_u32(slot_ptr(sl)) + lane * 128;
        const uint32_t pa = smem_u32(prm + c);
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          float4 xo, bb;
          const uint32_t ad = sa + ((g ^ (lane & 7)) << 4);
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(xo.x), "=f"(xo.y), "=f"(xo.z), "=f"(xo.w)
                       : "r"(ad)
                       : "memory");
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(bb.x), "=f"(bb.y), "=f"(bb.z), "=f"(bb.w)
                       : "r"(pa + 16u * g));
          v[4 * g] = xo.x + (v[4 * g] + bb.x);
          v[4 * g + 1] = xo.y + (v[4 * g + 1] + bb.y);
          v[4 * g + 2] = xo.z + (v[4 * g + 2] + bb.z);
          v[4 * g + 3] = xo.w + (v[4 * g + 3] + bb.w);
          asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(ad), "f"(v[4 * g]), "f"(v[4 * g + 1]),
                       "f"(v[4 * g + 2]), "f"(v[4 * g + 3])
                       : "memory");
        }
        tmem_st32(tbase + c, v);
        fence_proxy_async_smem();  // this slot's generic-proxy accesses before any TMA store / refill
        __syncwarp();
        if (full_blk) {
          if (lane == 0) {
            tma_store_2d(&tmX, slot_ptr(sl), c, rblk);
            bulk_commit();
          }
        } else if (row < M) {
#pragma unroll
          for (int g = 0; g < 8; ++g)
            *reinterpret_cast<float4*>(ep.x + (size_t)row * ep.ldx + c + 4 * g) =
                make_float4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
        }
        // chunk statistics of this lane's row, merged (Chan) into the running ones
        float sm = 0.f;
#pragma unroll
        for (int g = 0; g < 8; ++g) sm += (v[4 * g] + v[4 * g + 1]) + (v[4 * g + 2] + v[4 * g + 3]);
        const float bm = sm * (1.f / 32.f);
        float q = 0.f;
#pragma unroll
        for (int i = 0; i < 32; ++i) q += (v[i] - bm) * (v[i] - bm);
        chan_merge(cnt, rmean, rm2, 32.f, bm, q);
        // the slot of chunk j - 1 is refilled with chunk j + NSL - 1 once its store has read it
        if (lane == 0 && j + NSL - 1 < NCH) {
          bulk_wait_read<1>();
          load_chunk((j + NSL - 1) % NSL, c + 32 * (NSL - 1), rblk);
        }
        __syncwarp();
      }
      // every store has read its slot: the ring goes back to the producer, and the next
      // unit's first chunk is requested into this warp's own buffer
      if (lane == 0) {
        bulk_wait_read<0>();
        mbar_arrive(ring_free);
        if (USE_STG && u + ncl < num_units) load_chunk(0, cbeg, ((u + ncl) * CL + crank) * TC_BM + quarter * 32);
      }
      tmem_st_wait();
      // ---- exchange the two column halves' row partials ----
      float2* sb = stats + (size_t)(it & 1) * (2 * TC_BM);
      sb[half * TC_BM + quarter * 32 + lane] = make_float2(rmean, rm2);
      asm volatile("bar.sync %0, 64;" ::"r"(2 + quarter) : "memory");
      float tn = 0.f, tmean = 0.f, tm2 = 0.f;
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const float2 st = sb[p * TC_BM + quarter * 32 + lane];
        chan_merge(tn, tmean, tm2, (float)HB, st.x, st.y);
      }
      const float rstd = 1.0f / sqrtf(tm2 / (float)LR_D + 1e-5f);
      // ---- pass 2: y = LN(x) from the TMEM copy, one 64-byte bf16 row segment per chunk ----
      const int orow = row < M ? (ep.out_row ? ep.out_row[row] : row) : -1;
#pragma unroll 1
      for (int j = 0; j < NCH; ++j) {
        const int c = cbeg + 32 * j;
        float v[32];
        tmem_ld32(tbase + c, v);
        const uint32_t ga = smem_u32(prm + LR_D + c), ba = smem_u32(prm + 2 * LR_D + c);
        uint32_t pk[16];
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          float4 gg, bb;
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(gg.x), "=f"(gg.y), "=f"(gg.z), "=f"(gg.w)
                       : "r"(ga + 16u * g));
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(bb.x), "=f"(bb.y), "=f"(bb.z), "=f"(bb.w)
                       : "r"(ba + 16u * g));
          __nv_bfloat162 lo = __floats2bfloat162_rn((v[4 * g] - tmean) * rstd * gg.x + bb.x,
                                                    (v[4 * g + 1] - tmean) * rstd * gg.y + bb.y);
          __nv_bfloat162 hi = __floats2bfloat162_rn((v[4 * g + 2] - tmean) * rstd * gg.z + bb.z,
                                                    (v[4 * g + 3] - tmean) * rstd * gg.w + bb.w);
          pk[2 * g] = *reinterpret_cast<uint32_t*>(&lo);
          pk[2 * g + 1] = *reinterpret_cast<uint32_t*>(&hi);
        }
        if (orow >= 0) {
          uint4* dst = reinterpret_cast<uint4*>(ep.y + (size_t)orow * ep.ldy + c);
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4)
            dst[q4] = make_uint4(pk[4 * q4], pk[4 * q4 + 1], pk[4 * q4 + 2], pk[4 * q4 + 3]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(tempty), 0));
    }
  } else {
    // ===== epilogue: warp (quarter q, half h) owns rows 32 q .. 32 q + 31, columns 256 h .. +255 =====
    // lane (g = lane / 8, c = lane % 8) holds rows g + 4 i (i < 8), columns 4 c .. 4 c + 3 of a chunk
    const int ew = warp - 2;
    const int quarter = warp & 3;
    const int half = ew >> 2;
    const int cbeg = half * HB;
    const int lg = lane >> 3, lc = lane & 7;
    float* stg = reinterpret_cast<float*>(smem + L::STG_OFFSET) + ew * (32 * TC_STG_LD);
    int it = 0;
    for (int u = cid; u < num_units; u += ncl, ++it) {
      const int rbase = (u * CL + crank) * TC_BM + quarter * 32;
      float4 xo[8];
      auto load_x = [&](int cc, float4 (&dst)[8]) {
        const int colx = cc + lc * 4;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int row = rbase + lg + 4 * i;
          dst[i] = row < M ? *reinterpret_cast<const float4*>(ep.x + (size_t)row * ep.ldx + colx)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      };
      load_x(cbeg, xo);  // requested before the accumulator is ready
      mbar_wait(tfull, it & 1);
      tc_fence_after();
      const uint32_t tbase = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16);
      // ---- pass 1 ----
      // (count, mean, M2) per row; the count is the same for every row of the warp
      float cnt = 0.f, cmean[8], cm2[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) cmean[i] = cm2[i] = 0.f;
#pragma unroll 1
      for (int c = cbeg; c < cbeg + HB; c += 32) {
        float4 a[8];
        {
          float v[32];
          tmem_ld32(tbase + c, v);
          const uint32_t sbase = smem_u32(stg);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(
                             sbase + 4u * (lane * TC_STG_LD + 4 * (i ^ (lane & 7)))),
                         "f"(v[4 * i]), "f"(v[4 * i + 1]), "f"(v[4 * i + 2]), "f"(v[4 * i + 3])
                         : "memory");
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = i * 4 + lg;
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(a[i].x), "=f"(a[i].y), "=f"(a[i].z), "=f"(a[i].w)
                         : "r"(sbase + 4u * (r * TC_STG_LD + 4 * (lc ^ (r & 7))))
                         : "memory");
          }
          __syncwarp();
        }
        const int col = c + lc * 4;
        const float4 bb = *reinterpret_cast<const float4*>(prm + col);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float4 xn = xo[i];
          xn.x += a[i].x + bb.x;
          xn.y += a[i].y + bb.y;
          xn.z += a[i].z + bb.z;
          xn.w += a[i].w + bb.w;
          a[i] = xn;
        }
        // the residual registers are free: the next chunk's rows are requested now, so their
        // latency hides behind this chunk's stores, statistics and the next TMEM load
        if (c + 32 < cbeg + HB) load_x(c + 32, xo);
        const float nt = cnt + 32.f;
        const float wb = 32.f / nt, wn = cnt * 32.f / nt;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int row = rbase + lg + 4 * i;
          const float4 xn = a[i];
          if (row < M) *reinterpret_cast<float4*>(ep.x + (size_t)row * ep.ldx + col) = xn;
          float sm = (xn.x + xn.y) + (xn.z + xn.w);
          sm += __shfl_xor_sync(0xffffffffu, sm, 1);
          sm += __shfl_xor_sync(0xffffffffu, sm, 2);
          sm += __shfl_xor_sync(0xffffffffu, sm, 4);
          const float bm = sm * (1.f / 32.f);
          const float e0 = xn.x - bm, e1 = xn.y - bm, e2 = xn.z - bm, e3 = xn.w - bm;
          float q = (e0 * e0 + e1 * e1) + (e2 * e2 + e3 * e3);
          q += __shfl_xor_sync(0xffffffffu, q, 1);
          q += __shfl_xor_sync(0xffffffffu, q, 2);
          q += __shfl_xor_sync(0xffffffffu, q, 4);
          // Chan merge of this 32-column block into the running row statistics
          const float delta = bm - cmean[i];
          cmean[i] += delta * wb;
          cm2[i] += q + delta * delta * wn;
        }
        cnt = nt;
        // the chunk's updated values, kept on chip for pass 2 (lane-private slots of
        // the chunk's own TMEM columns; the layout only has to round-trip)
        if constexpr (KEEP) tmem_st32(tbase + c, reinterpret_cast<const float*>(a));
      }
      // ---- exchange the two column halves' row partials (double-buffered by unit parity) ----
      float2* sb = stats + (size_t)(it & 1) * (2 * TC_BM);
      if (lc == 0) {
#pragma unroll
        for (int i = 0; i < 8; ++i) sb[half * TC_BM + quarter * 32 + lg + 4 * i] = make_float2(cmean[i], cm2[i]);
      }
      if constexpr (KEEP) {
        tmem_st_wait();
      } else {
        // the accumulator is no longer needed: the next unit's MMAs overlap pass 2
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(tempty), 0));
      }
      asm volatile("bar.sync %0, 64;" ::"r"(2 + quarter) : "memory");
      float mean[8], rstd[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float tn = 0.f, tmean = 0.f, tm2 = 0.f;
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          const float2 st = sb[p * TC_BM + quarter * 32 + lg + 4 * i];
          chan_merge(tn, tmean, tm2, (float)HB, st.x, st.y);
        }
        mean[i] = tmean;
        rstd[i] = 1.0f / sqrtf(tm2 / (float)LR_D + 1e-5f);
      }
      // ---- pass 2: y = LN(x) ----
      int orow[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int row = rbase + lg + 4 * i;
        orow[i] = row < M ? (ep.out_row ? ep.out_row[row] : row) : -1;
      }
      if constexpr (KEEP) {
#pragma unroll 1
        for (int c = cbeg; c < cbeg + HB; c += 32) {
          float t[32];
          tmem_ld32(tbase + c, t);
          const int col = c + lc * 4;
          const float4 gg = *reinterpret_cast<const float4*>(prm + LR_D + col);
          const float4 bb = *reinterpret_cast<const float4*>(prm + 2 * LR_D + col);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            if (orow[i] < 0) continue;
            __nv_bfloat162 lo = __floats2bfloat162_rn((t[4 * i] - mean[i]) * rstd[i] * gg.x + bb.x,
                                                      (t[4 * i + 1] - mean[i]) * rstd[i] * gg.y + bb.y);
            __nv_bfloat162 hi = __floats2bfloat162_rn((t[4 * i + 2] - mean[i]) * rstd[i] * gg.z + bb.z,
                                                      (t[4 * i + 3] - mean[i]) * rstd[i] * gg.w + bb.w);
            uint2 o;
            o.x = *reinterpret_cast<uint32_t*>(&lo);
            o.y = *reinterpret_cast<uint32_t*>(&hi);
            *reinterpret_cast<uint2*>(ep.y + (size_t)orow[i] * ep.ldy + col) = o;
          }
        }
      } else {
        float4 xv[8];
        auto load_xn = [&](int cc, float4 (&dst)[8]) {
          const int colx = cc + lc * 4;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int row = rbase + lg + 4 * i;
            dst[i] = orow[i] >= 0 ? __ldcg(reinterpret_cast<const float4*>(ep.x + (size_t)row * ep.ldx + colx))
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        };
        load_xn(cbeg, xv);
#pragma unroll 1
        for (int c = cbeg; c < cbeg + HB; c += 32) {
          const int col = c + lc * 4;
          const float4 gg = *reinterpret_cast<const float4*>(prm + LR_D + col);
          const float4 bb = *reinterpret_cast<const float4*>(prm + 2 * LR_D + col);
          float4 o4[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            o4[i].x = (xv[i].x - mean[i]) * rstd[i] * gg.x + bb.x;
            o4[i].y = (xv[i].y - mean[i]) * rstd[i] * gg.y + bb.y;
            o4[i].z = (xv[i].z - mean[i]) * rstd[i] * gg.z + bb.z;
            o4[i].w = (xv[i].w - mean[i]) * rstd[i] * gg.w + bb.w;
          }
          if (c + 32 < cbeg + HB) load_xn(c + 32, xv);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            if (orow[i] < 0) continue;
            __nv_bfloat162 lo = __floats2bfloat162_rn(o4[i].x, o4[i].y);
            __nv_bfloat162 hi = __floats2bfloat162_rn(o4[i].z, o4[i].w);
            uint2 o;
            o.x = *reinterpret_cast<uint32_t*>(&lo);
            o.y = *reinterpret_cast<uint32_t*>(&hi);
            *reinterpret_cast<uint2*>(ep.y + (size_t)orow[i] * ep.ldy + col) = o;
          }
        }
      }
      if constexpr (KEEP) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(tempty), 0));
      }
    }
  }
  tc_fence_before();
  cluster_sync_all();  // no CTA leaves while its peer's MMAs / signals may still target it
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, TMEM_COLS);
  }
}

}  // namespace hrt
