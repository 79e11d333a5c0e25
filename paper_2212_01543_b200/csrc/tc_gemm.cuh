// Persistent tcgen05 / TMEM / TMA GEMM for sm_100a:
//     C[M, N] = A[M, K] . B[N, K]^T      (bf16 operands, fp32 accumulate)
//
// A = activations, B = weights stored N x K ("K-major", the transpose of the
// reference's (d_in, d_out) W, model.py:152-165). One CTA per SM loops over
// 128 x BN output tiles:
//   warp 0        TMA producer (one elected lane), STAGES-deep smem ring
//   warp 1        TMEM allocator + MMA issuer (one elected lane); two TMEM
//                 accumulators so tile i+1's MMAs overlap tile i's epilogue
//   warps 2..9    epilogue, two warps per TMEM lane quarter (column halves).
//                 Element-wise epilogues (bias / ReLU / residual /
//                 store) transpose each 32x32 accumulator chunk through a
//                 per-warp smem buffer so global traffic is coalesced 128 B
//                 rows; row-wise epilogues (vocab softmax statistics) keep
//                 one row per thread.
#pragma once
#include "common.cuh"
#include "sm100_ptx.cuh"

namespace hrt {

constexpr int TC_BM = 128;
constexpr int TC_BK = 64;  // 64 bf16 = 128 B rows -> SWIZZLE_128B
constexpr int TC_EPI_WARPS = 8;  // two per TMEM lane quarter, each owning half the tile columns
constexpr int TC_THREADS = 64 + 32 * TC_EPI_WARPS;
constexpr int TC_STG_LD = 32;  // epilogue transpose row pitch (floats); 16-byte slots XOR-swizzled by row

// BROWS: weight rows staged per CTA (BN, or BN / 2 when a cta_group::2 pair splits them)
template <int BN, int STAGES, int BROWS = BN>
struct TcSmem {
  static constexpr int A_BYTES = TC_BM * TC_BK * 2;
  static constexpr int B_BYTES = BROWS * TC_BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STG_OFFSET = STAGES * STAGE_BYTES;                // epilogue staging
  static constexpr int STG_BYTES = TC_EPI_WARPS * 32 * TC_STG_LD * 4;
  static constexpr int BAR_OFFSET = STG_OFFSET + STG_BYTES;
  static constexpr int TOTAL = BAR_OFFSET + 256 + 1024;  // barriers + alignment slack
};

template <int BN>
__host__ __device__ constexpr int tmem_cols_for() {
  return 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Epilogue protocols:
//  element-wise (Epi::kRowWise == false): apply8(row0, col, float4 v[8], M)
//    for rows row0 + 4 i (i < 8, rows >= M skipped), 4 consecutive columns
//    (N % 4 == 0 is required).
//  row-wise (Epi::kRowWise == true): State; begin(st,row,n0);
//    chunk(st,row,col0,const float* v,int n); end(st,row,n0) per thread-row.
// Split-K: splits > 1 partitions the K blocks of every tile into slices,
// each slice an independent work unit; ws holds splits x Mpad x N fp32
// partials and counters one arrival counter per tile (zero between launches).
struct SplitK {
  int splits;
  float* ws;
  int* counters;
};

// element-wise epilogues that store whole per-lane row segments (Epi::kRowStore)
template <class E, class = void>
struct EpiRowStore {
  static constexpr bool value = false;
};
template <class E>
struct EpiRowStore<E, decltype(void(E::kRowStore))> {
  static constexpr bool value = E::kRowStore;
};

// element-wise epilogues that write bf16 tiles with TMA stores (Epi::kTmaStore)
template <class E, class = void>
struct EpiTmaStore {
  static constexpr bool value = false;
};
template <class E>
struct EpiTmaStore<E, decltype(void(E::kTmaStore))> {
  static constexpr bool value = E::kTmaStore;
};

// element-wise epilogues whose global operands can be requested a chunk ahead (Epi::kPrefetch)
template <class E, class = void>
struct EpiPrefetch {
  static constexpr bool value = false;
};
template <class E>
struct EpiPrefetch<E, decltype(void(E::kPrefetch))> {
  static constexpr bool value = E::kPrefetch;
};

// B (weight) tile load: whole BN-row box (CL = 1), or this CTA's BN/CL-row
// slice multicast to every CTA of the cluster (CL = 2 / 4; the tensor map's box is BN/CL rows)
template <int BN, int CL>
__device__ __forceinline__ void tc_load_b(uint8_t* dst, const CUtensorMap* tmB, uint64_t* bar, int k0, int n0,
                                          int crank, uint64_t pol) {
  if constexpr (CL == 1) {
    tma_load_2d_hint(dst, tmB, bar, k0, n0, pol);
  } else {
    tma_load_2d_mc_hint(dst + crank * (BN / CL) * (TC_BK * 2), tmB, bar, k0, n0 + crank * (BN / CL),
                        (uint16_t)((1u << CL) - 1), pol);
  }
}

// CL = 2: CTA pairs (thread-block clusters of two) take vertically adjacent
// tiles (m, n) and (m + 1, n); each CTA loads its own A tile and half of the
// shared B tile, multicast into both CTAs' shared memory, so the L2 -> SM
// operand traffic per tile drops from (128 + BN) to (128 + BN / 2) rows. A
// stage is refilled only after both CTAs' MMAs released it (the empty
// barrier counts one MMA-commit arrival from each CTA). Split-K is CL = 1 only.
// CL = 4 (option "cluster4"): the same with four vertically adjacent tiles per
// cluster, each CTA loading a quarter of the weight tile: (128 + BN / 4) rows per tile.
//
// PAIR (CL = 2 only): the pair runs cta_group::2 MMAs instead -- one M = 256 x BN
// instruction issued by the leader CTA reads A's 128 rows from each CTA and B's BN
// rows as BN / 2 + BN / 2 from the two CTAs, so each CTA stages only half the weight
// tile (no multicast) and its shared memory feeds half the B operand per MMA. Both
// CTAs' TMA loads complete on the leader's full barrier; the leader's commits
// multicast to both CTAs' empty / accumulator-full barriers; both CTAs' epilogue
// warps release an accumulator on the leader's barrier.
template <int BN, int STAGES, class Epi, int CL = 1, bool PAIR = false>
__global__ void __launch_bounds__(TC_THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmC, int M, int N, int K, const int* __restrict__ M_dev, Epi epi,
                   SplitK sk) {
  static_assert(!PAIR || CL == 2, "cta_group::2 needs a CTA pair");
  using L = TcSmem<BN, STAGES, PAIR ? BN / 2 : BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::BAR_OFFSET);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;  // [2]
  uint64_t* tempty = tfull + 2;      // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  static_assert(CL == 1 || CL == 2 || CL == 4, "cluster size");
  pdl_trigger();
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_kb = K / TC_BK;
  const int crank = CL > 1 ? (int)cluster_ctarank() : 0;
  const int cid = blockIdx.x / CL, ncl = gridDim.x / CL;  // cluster index / count
  constexpr uint32_t TMEM_COLS = tmem_cols_for<BN>();

  // setup that does not depend on the previous kernel overlaps its tail (PDL)
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], PAIR ? 1 : CL);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], PAIR ? 2 * TC_EPI_WARPS : TC_EPI_WARPS);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    if constexpr (PAIR) tmem_alloc_pair(tmem_slot, TMEM_COLS);
    else tmem_alloc(tmem_slot, TMEM_COLS);
  }
  tc_fence_before();
  if constexpr (CL > 1)
    cluster_sync_all();  // the peer's barriers are initialised before any multicast reaches them
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int n_tiles = (N + BN - 1) / BN;
  // work unit = (tile, k-slice); sk.splits > 1 only for element-wise epilogues
  const int S = CL > 1 ? 1 : sk.splits;
  // Weights do not depend on the previous kernel: the first unit of a CTA in
  // m-tile 0 (which exists for any M >= 1) gets its first STAGES weight tiles
  // requested before the grid-dependency wait, overlapping the previous
  // kernel's tail (the A tiles follow after the wait into the same stages).
  // PAIR: every stage's bytes (both CTAs') complete on the leader's full barrier
  const uint32_t full_l = PAIR ? mapa_shared(smem_u32(full), 0) : 0u;
  auto arm = [&](int st) {
    if (!PAIR || crank == 0) mbar_arrive_expect_tx(&full[st], (PAIR ? 2 : 1) * L::STAGE_BYTES);
  };
  auto load_a = [&](int st, int k0, int m0) {
    uint8_t* dst = smem + st * L::STAGE_BYTES;
    if constexpr (PAIR) tma_load_2d_pair(dst, &tmA, full_l + 8u * st, k0, m0);
    else tma_load_2d(dst, &tmA, &full[st], k0, m0);
  };
  auto load_b = [&](int st, int k0, int n0, uint64_t pol) {
    uint8_t* dst = smem + st * L::STAGE_BYTES + L::A_BYTES;
    if constexpr (PAIR) tma_load_2d_pair(dst, &tmB, full_l + 8u * st, k0, n0 + crank * (BN / 2), pol);
    else tc_load_b<BN, CL>(dst, &tmB, &full[st], k0, n0, crank, pol);
  };
  int pre = 0;
  if (warp == 0 && lane == 0 && cid < n_tiles * S) {
    const int tile = cid / S, ks = cid - tile * S;
    const int kb0 = ks * num_kb / S, kb1 = (ks + 1) * num_kb / S;
    pre = min(STAGES, kb1 - kb0);
    const uint64_t pol = policy_evict_last();
    for (int s2 = 0; s2 < pre; ++s2) {
      arm(s2);
      load_b(s2, (kb0 + s2) * TC_BK, tile * BN, pol);
    }
  }
  pdl_wait();
  if (M_dev != nullptr) M = *M_dev;
  const int m_tiles = (M + TC_BM - 1) / TC_BM;
  const int num_units = (m_tiles + CL - 1) / CL * n_tiles * S;  // CL > 1: units are vertical tile pairs

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer =====
      const uint64_t pol_w = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int u = cid; u < num_units; u += ncl) {
        const int tile = u / S, ks = u - tile * S;
        const int m0 = ((tile / n_tiles) * CL + crank) * TC_BM, n0 = (tile % n_tiles) * BN;
        const int kb0 = ks * num_kb / S, kb1 = (ks + 1) * num_kb / S;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (u == cid && kb - kb0 < pre) {  // weight tile already requested before the PDL wait
            load_a(stage, kb * TC_BK, m0);
          } else {
            arm(stage);
            load_a(stage, kb * TC_BK, m0);
            load_b(stage, kb * TC_BK, n0, pol_w);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      // no unit after all (device row count 0: every Stage-I row finished): the stages
      // armed before the PDL wait expect their A tiles too -- load them (rows past the
      // tensor are zero-filled by TMA) so every byte lands before the CTA may exit
      if (cid >= num_units) {
        const int kb0 = (cid % S) * num_kb / S;
        for (int s2 = 0; s2 < pre; ++s2) load_a(s2, (kb0 + s2) * TC_BK, 0);
        if (!PAIR || crank == 0)
          for (int s2 = 0; s2 < pre; ++s2) mbar_wait(&full[s2], 0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && (!PAIR || crank == 0)) {
      // ===== MMA issuer (PAIR: the leader CTA, M = 256 across the pair) =====
      constexpr uint32_t idesc = idesc_bf16_f32(PAIR ? 2 * TC_BM : TC_BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int u = cid; u < num_units; u += ncl, ++it) {
        const int ks = u % S;
        const int kb0 = ks * num_kb / S, kb1 = (ks + 1) * num_kb / S;
        const int acc = it & 1;
        const uint32_t aphase = (it >> 1) & 1;
        mbar_wait(&tempty[acc], aphase ^ 1);  // epilogue drained this accumulator
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * L::STAGE_BYTES);
          const uint32_t sb = sa + L::A_BYTES;
#pragma unroll
          for (int k = 0; k < TC_BK / 16; ++k) {
            if constexpr (PAIR)
              tc_mma_f16_pair(d_tmem, sdesc_kmajor_sw128(sa + k * 32), sdesc_kmajor_sw128(sb + k * 32), idesc,
                              ((kb - kb0) | k) != 0);
            else
              tc_mma_f16(d_tmem, sdesc_kmajor_sw128(sa + k * 32), sdesc_kmajor_sw128(sb + k * 32), idesc,
                         ((kb - kb0) | k) != 0);
          }
          if constexpr (PAIR)
            tc_commit_pair_mc(&empty[stage], (uint16_t)3);  // the stage is free in both CTAs
          else if constexpr (CL > 1)
            tc_commit_mc(&empty[stage], (1u << CL) - 1);  // release the stage in both CTAs (B halves are shared)
          else
            tc_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if constexpr (PAIR)
          tc_commit_pair_mc(&tfull[acc], (uint16_t)3);
        else
          tc_commit(&tfull[acc]);
      }
    }
  } else {
    // ===== epilogue warps =====
    const int ew = warp - 2;
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    // this warp's column half (BN = 32: the first four warps take the whole tile)
    const int cbeg = BN >= 64 ? (ew / 4) * (BN / 2) : 0;
    const int cend = BN >= 64 ? cbeg + BN / 2 : (ew < 4 ? BN : 0);
    float* stg = reinterpret_cast<float*>(smem + L::STG_OFFSET) + ew * (32 * TC_STG_LD);
    int it = 0;
    int sc = 0;  // TMA-store staging buffers used by this warp (alternating halves of stg)
    int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);
    for (int u = cid; u < num_units; u += ncl, ++it) {
      const int tile = u / S, ks = u - tile * S;
      const int acc = it & 1;
      const uint32_t aphase = (it >> 1) & 1;
      const int m0 = ((tile / n_tiles) * CL + crank) * TC_BM, n0 = (tile % n_tiles) * BN;
      const int rbase = m0 + quarter * 32;
      constexpr bool PF = EpiPrefetch<Epi>::value && !Epi::kRowWise;
      float4 pfa[PF ? 8 : 1];
      // residual operands of the first chunk are requested before the accumulator is ready
      if constexpr (PF) {
        if (S == 1 && cbeg < cend && n0 + cbeg + (lane & 7) * 4 < N)
          epi.prefetch8(rbase + (lane >> 3), n0 + cbeg + (lane & 7) * 4, M, pfa);
      }
      mbar_wait(&tfull[acc], aphase);
      tc_fence_after();
      const uint32_t tbase = tmem_base + acc * BN + (static_cast<uint32_t>(quarter * 32) << 16);
      if constexpr (Epi::kRowWise) {
        const int row = rbase + lane;
        typename Epi::State st;
        const bool live = row < M;
        if (live) epi.begin(st, row, n0 + cbeg);
        // software pipeline: chunk c + 32's TMEM load is in flight while chunk c is processed
        uint32_t ra[32], rb[32];
        if (cbeg < cend) tmem_ld32_issue(tbase + cbeg, ra);
#pragma unroll 1
        for (int c = cbeg; c < cend; c += 64) {
          tmem_ld_wait(ra);
          if (c + 32 < cend) tmem_ld32_issue(tbase + c + 32, rb);
          {
            const int col0 = n0 + c;
            int nvalid = N - col0;
            nvalid = nvalid > 32 ? 32 : nvalid;
            float v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(ra[i]);
            if (live && nvalid > 0) epi.chunk(st, row, col0, v, nvalid);
          }
          if (c + 32 < cend) {
            tmem_ld_wait(rb);
            if (c + 64 < cend) tmem_ld32_issue(tbase + c + 64, ra);
            const int col0 = n0 + c + 32;
            int nvalid = N - col0;
            nvalid = nvalid > 32 ? 32 : nvalid;
            float v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(rb[i]);
            if (live && nvalid > 0) epi.chunk(st, row, col0, v, nvalid);
          }
        }
        if (live) epi.end(st, row, n0 + cbeg);
      } else if constexpr (EpiTmaStore<Epi>::value) {
        // lane = row: bias (+ ReLU) -> bf16 -> this warp's 64-byte-swizzled 32 x 32 staging
        // tile -> one TMA store per chunk (no register transpose, no per-lane global stores;
        // rows past M inside the tile land in the buffer's spare rows or are clipped by TMA)
        uint8_t* stg8 = reinterpret_cast<uint8_t*>(stg);
        uint32_t ra[32], rb[32];
        if (cbeg < cend) tmem_ld32_issue(tbase + cbeg, ra);
        float bcur = (cbeg < cend && n0 + cbeg + lane < N) ? epi.bias_of(n0 + cbeg + lane) : 0.f;
#pragma unroll 1
        for (int c = cbeg; c < cend; c += 32) {
          tmem_ld_wait(ra);
          float v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(ra[i]);
          if (c + 32 < cend) tmem_ld32_issue(tbase + c + 32, rb);
          const float bnext = (c + 32 < cend && n0 + c + 32 + lane < N) ? epi.bias_of(n0 + c + 32 + lane) : 0.f;
          const int col0 = n0 + c;
          if (col0 < N) {
            uint32_t pk[16];
            epi.row32_pack_shfl(bcur, v, pk);
            uint8_t* buf = stg8 + (sc & 1) * 2048;
            if (sc >= 2) {  // the store issued from this half two chunks ago has read it
              if (lane == 0) bulk_wait_read<1>();
              __syncwarp();
            }
            const uint32_t rowa = smem_u32(buf) + lane * 64;
#pragma unroll
            for (int j = 0; j < 4; ++j)
              asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rowa + 16u * (j ^ ((lane >> 1) & 3))),
                           "r"(pk[4 * j]), "r"(pk[4 * j + 1]), "r"(pk[4 * j + 2]), "r"(pk[4 * j + 3])
                           : "memory");
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&tmC, buf, col0, rbase);
              bulk_commit();
            }
            ++sc;
          }
          bcur = bnext;
#pragma unroll
          for (int i = 0; i < 32; ++i) ra[i] = rb[i];
        }
      } else if constexpr (EpiRowStore<Epi>::value) {
        // lane = row: the lane's 32 consecutive columns go out as full 64 / 128-byte
        // row segments (no shared-memory transpose)
        const int row = rbase + lane;
#pragma unroll 1
        for (int c = cbeg; c < cend; c += 32) {
          float v[32];
          tmem_ld32(tbase + c, v);
          const int col0 = n0 + c;
          if (row < M && col0 < N) epi.row32(row, col0, v, N - col0);
        }
      } else {
        const int Mpad = m_tiles * TC_BM;
        // each 32-column chunk is transposed through shared memory with
        // 16-byte accesses so global traffic is coalesced row segments
#pragma unroll 1
        for (int c = cbeg; c < cend; c += 32) {
          float v[32];
          tmem_ld32(tbase + c, v);
          const uint32_t sbase = smem_u32(stg);  // explicit shared-space accesses (not generic ld/st)
#pragma unroll
          for (int i = 0; i < 8; ++i)  // row `lane`, slot i -> physical slot i ^ (row & 7): conflict-free
            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(
                             sbase + 4u * (lane * TC_STG_LD + 4 * (i ^ (lane & 7)))),
                         "f"(v[4 * i]), "f"(v[4 * i + 1]), "f"(v[4 * i + 2]), "f"(v[4 * i + 3])
                         : "memory");
          __syncwarp();
          const int col = n0 + c + (lane & 7) * 4;
          float4 vals[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = i * 4 + (lane >> 3);
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(vals[i].x), "=f"(vals[i].y), "=f"(vals[i].z), "=f"(vals[i].w)
                         : "r"(sbase + 4u * (r * TC_STG_LD + 4 * ((lane & 7) ^ (r & 7))))
                         : "memory");
          }
          if (S == 1) {
            // rows rbase + (lane >> 3) + 4 i; all global loads of the group are
            // issued before any store (memory-level parallelism)
            if constexpr (PF) {
              float4 nxt[8];
              const int ncol = col + 32;
              if (c + 32 < cend && ncol < N) epi.prefetch8(rbase + (lane >> 3), ncol, M, nxt);
              if (col < N) epi.apply8_pre(rbase + (lane >> 3), col, vals, M, pfa);
              if (c + 32 < cend) {
#pragma unroll
                for (int i = 0; i < 8; ++i) pfa[i] = nxt[i];
              }
            } else {
              if (col < N) epi.apply8(rbase + (lane >> 3), col, vals, M);
            }
          } else if (col < N) {
            // split-K: this slice's fp32 partial tile
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int row = rbase + (lane >> 3) + 4 * i;
              *reinterpret_cast<float4*>(sk.ws + ((size_t)ks * Mpad + row) * N + col) = vals[i];
            }
          }
          __syncwarp();
        }
        if (S > 1) {
          // deterministic split-K fix-up: the last slice to finish sums all
          // partials in slice order and applies the real epilogue
          __threadfence();
          asm volatile("bar.sync 1, %0;" ::"n"(TC_EPI_WARPS * 32));
          if (ew == 0 && lane == 0) {
            const int old = atomicAdd(sk.counters + tile, 1);
            *last_flag = (old == S - 1);
          }
          asm volatile("bar.sync 1, %0;" ::"n"(TC_EPI_WARPS * 32));
          if (*last_flag) {
            __threadfence();
#pragma unroll 1
            for (int c = cbeg; c < cend; c += 32) {
              const int col = n0 + c + (lane & 7) * 4;
              if (col >= N) continue;
              float4 vals[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) vals[i] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 1
              for (int s2 = 0; s2 < S; ++s2) {
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                  const int row = rbase + (lane >> 3) + 4 * i;
                  const float4 p = __ldcg(reinterpret_cast<const float4*>(sk.ws + ((size_t)s2 * Mpad + row) * N + col));
                  vals[i].x += p.x;
                  vals[i].y += p.y;
                  vals[i].z += p.z;
                  vals[i].w += p.w;
                }
              }
              epi.apply8(rbase + (lane >> 3), col, vals, M);
            }
            asm volatile("bar.sync 1, %0;" ::"n"(TC_EPI_WARPS * 32));
            if (ew == 0 && lane == 0) sk.counters[tile] = 0;  // re-arm for the next launch / graph replay
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (PAIR) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));
        else mbar_arrive(&tempty[acc]);
      }
    }
    if constexpr (EpiTmaStore<Epi>::value) {
      if (lane == 0) bulk_wait_all();  // staged tiles fully written before the CTA retires
    }
  }
  tc_fence_before();
  if constexpr (CL > 1)
    cluster_sync_all();  // no CTA leaves while its peer may still signal its barriers
  else
    __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (PAIR) tmem_dealloc_pair(tmem_base, TMEM_COLS);
    else tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

}  // namespace hrt
