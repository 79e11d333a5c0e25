// One encoder layer for a handful of source tokens (batch-1 latency: M <= 64
// packed rows) as ONE launch on one 16-CTA thread-block cluster
// (infer.py:190-213: LN1 -> QKV -> self-attention -> Wo + residual -> LN2 ->
// W1 + ReLU -> W2 + residual -> the next LayerNorm).
//
// At batch 1 the per-kernel encoder layer is a chain of 7 dependent launches
// (~3.6 us each, 25 us per layer) whose work is tiny; the bytes that matter
// are the layer's 6.3 MB of bf16 weights. Here:
//   * CTA c owns a slice of every projection's output features -- q / k / v
//     of head c / 2, dims (c % 2) * 32 .. +32; Wo and W2 columns 32 c .. +32;
//     W1 hidden units 128 c .. +128 -- i.e. 12 weight chunks of 32 KB, read
//     from the fragment-native copies (gemv_small.cuh) through a 4-slot
//     shared-memory ring of 1-D bulk copies, the first four requested before
//     the grid-dependency wait (weights never depend on the previous launch);
//   * activations are exchanged through L2 (global scratch) and published by
//     hardware cluster barriers (release / acquire): on B200 one SM pulls
//     ~150 GB/s out of L2 but only ~20 B/cycle over DSMEM, so a full-row
//     exchange is cheaper through L2 (tools/micro_stream.cu);
//   * projections run on mma.sync m16n8k16 (weights as the 16-row M side,
//     8 activation rows per n-tile, the K index permuted identically on both
//     operands as in gemv_small_kernel); eight warps split the two 16-feature
//     groups of a chunk x row halves x K, reduced in shared memory in a fixed
//     order;
//   * LN2 is recomputed by every CTA from the full residual rows (no extra
//     barrier); the next LayerNorm (the next layer's LN1 or the final encoder
//     LN) is written by CTA c for rows c, c + 16, ...
// Five cluster barriers per layer replace seven kernel boundaries.
#pragma once
#include "common.cuh"
#include "decode_cluster.cuh"
#include "gemv_small.cuh"
#include "kernels.cuh"
#include "sm100_ptx.cuh"

namespace hrt {

constexpr int EC_CN = 16;
constexpr int EC_THREADS = 512;
constexpr int EC_WARPS = EC_THREADS / 32;
constexpr int EC_D = 512, EC_FF = 2048, EC_H = 8, EC_DH = 64;
constexpr int EC_MAXM = 64;          // packed source rows per launch
constexpr int EC_CHUNK = 32 * 1024;  // two 16-feature groups x 512 K (fragment-native)
constexpr int EC_NSLOT = 4;
constexpr int EC_NCH = 12;           // q k v | wo | w1 x4 | w2 x4
constexpr int EC_AST = EC_D + 8;     // activation row stride (bf16): conflict-free fragment loads
constexpr int EC_KVST = EC_DH + 1;   // attention K / V row stride (fp32)

struct EcParams {
  const bf16 *wqkv, *wo, *w1, *w2;  // fragment-native copies
  const float *bqkv, *bo, *b1, *b2, *ln2g, *ln2b, *lnng, *lnnb;
  float* x;     // [M][D] residual stream
  bf16* y;      // [M][D] LN1 output on entry, the next LayerNorm on exit
  bf16* qkv;    // [M][3D] scratch
  bf16* ctx;    // [M][D] scratch
  bf16* hid;    // [M][FF] scratch
  const int* seq_off;  // [nseq] first row of each packed sequence
  const int* seq_len;
  int nseq, M;
  float att_scale;
  int trace;  // timing attribution: CTA 0 prints its phase times (globaltimer) when set
};

struct EcSmem {
  static constexpr int RING = 0;
  static constexpr int ACT = RING + EC_NSLOT * EC_CHUNK;        // bf16 [64][EC_AST] (also attention K / V fp32)
  static constexpr int RED = ACT + EC_MAXM * EC_AST * 2;        // float [16 warps][32][16] partial sums
  static constexpr int PRM = RED + EC_WARPS * 16 * 32 * 4;      // float: bqkv 96 | bo 32 | b1 128 | b2 32
  static constexpr int NPRM = 96 + 32 + 128 + 32;
  static constexpr int BAR = PRM + NPRM * 4;
  static constexpr int TOTAL = BAR + 64;
  static_assert(EC_MAXM * EC_KVST * 4 * 3 <= EC_MAXM * EC_AST * 2, "attention K / V fit the activation buffer");
  static_assert(TOTAL <= 227 * 1024, "encoder cluster shared memory");
};

// chunk j of CTA c: two 16 KB pieces (group 0, group 1) of the fragment-native copies
__device__ __forceinline__ void ec_chunk_src(const EcParams& p, int j, int c, const bf16*& s0, const bf16*& s1) {
  constexpr size_t G512 = 16 * 512;  // elements per 16-feature group at K = 512
  const int hh = c >> 1, half = c & 1;
  if (j < 3) {  // q / k / v rows j * 512 + 64 hh + 32 half .. +32 of the fused [3D, D] matrix
    const int grp = (j * EC_D + hh * 64 + half * 32) / 16;
    s0 = p.wqkv + grp * G512;
    s1 = s0 + G512;
  } else if (j == 3) {
    s0 = p.wo + (size_t)(2 * c) * G512;
    s1 = s0 + G512;
  } else if (j < 8) {
    s0 = p.w1 + (size_t)(8 * c + 2 * (j - 4)) * G512;
    s1 = s0 + G512;
  } else {  // W2 [D, FF]: groups 2c, 2c + 1 (64 KB each over K = 2048), K-slice j - 8 of 512
    constexpr size_t G2048 = 16 * 2048;
    s0 = p.w2 + (size_t)(2 * c) * G2048 + (size_t)(j - 8) * G512;
    s1 = s0 + G2048;
  }
}

// C[f][r] partials of one chunk: 16-feature groups gi = warp & 1; rows split in halves when
// M > 32 (TWO: rh), K-chunks (32 wide) split over the remaining warps (ks). Accumulates into c.
template <bool TWO>
__device__ __forceinline__ void ec_mma_chunk(const bf16* __restrict__ wch, const bf16* __restrict__ act, int M,
                                             float (&c)[4][4]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  const int gi = warp & 1, rest = warp >> 1;
  const int rh = TWO ? (rest & 1) : 0, ks = TWO ? (rest >> 1) : rest;
  constexpr int PER = TWO ? 4 : 2;  // K-chunks (of 16) per warp
  const int nt_live = min(4, (M - 32 * rh + 7) / 8);
  const bf16* wg = wch + gi * (16 * 512) + (ks * PER * 64 + lane) * 8;
  uint4 u0[PER], u1[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    u0[i] = *reinterpret_cast<const uint4*>(wg + (2 * i) * 256);
    u1[i] = *reinterpret_cast<const uint4*>(wg + (2 * i + 1) * 256);
  }
  // the live n-tiles' four accumulation chains interleave (predicated, not branched per tile)
  const bf16* ar[4];
#pragma unroll
  for (int nt = 0; nt < 4; ++nt) ar[nt] = act + min(32 * rh + 8 * nt + g, M - 1) * EC_AST + ks * PER * 32 + 8 * t4;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    uint4 v[4];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
      if (nt < nt_live) v[nt] = *reinterpret_cast<const uint4*>(ar[nt] + 32 * i);
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
      if (nt < nt_live) gv_mma(c[nt], u0[i].x, u1[i].x, u0[i].y, u1[i].y, v[nt].x, v[nt].y);
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
      if (nt < nt_live) gv_mma(c[nt], u0[i].z, u1[i].z, u0[i].w, u1[i].w, v[nt].z, v[nt].w);
  }
}

// per-thread outputs of a 32-column slice: (row r = idx >> 5, column f = idx & 31), idx = tid + 256 k
constexpr int EC_OPT = EC_MAXM * 32 / EC_THREADS;  // 4

// reduce the warps' partials in a fixed order: v[k] = out(f, r) of this thread's k-th output
// (rows r < M); partial layout [warp][row 0..31][feature 0..15]
template <bool TWO>
__device__ __forceinline__ void ec_reduce(float (&c)[4][4], float* red, int M, float (&v)[EC_OPT]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  float* rw = red + warp * (32 * 16);
#pragma unroll
  for (int nt = 0; nt < 4; ++nt) {
    const int r0 = 8 * nt + 2 * t4;
    rw[r0 * 16 + g] = c[nt][0];
    rw[(r0 + 1) * 16 + g] = c[nt][1];
    rw[r0 * 16 + g + 8] = c[nt][2];
    rw[(r0 + 1) * 16 + g + 8] = c[nt][3];
  }
  __syncthreads();
  constexpr int NKS = TWO ? EC_WARPS / 4 : EC_WARPS / 2;
#pragma unroll
  for (int k = 0; k < EC_OPT; ++k) {
    const int idx = threadIdx.x + EC_THREADS * k, r = idx >> 5, f = idx & 31;
    const int gi = f >> 4, fl = f & 15, rh = (r >> 5) & 1, lr = r & 31;
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < NKS; ++q) {
      const int w = gi + 2 * (TWO ? (rh + 2 * q) : q);
      s += red[w * (32 * 16) + lr * 16 + fl];
    }
    v[k] = s;
  }
  __syncthreads();
}

// this thread's residual values x[r][col0 + f] (requested before the MMAs)
__device__ __forceinline__ void ec_load_res(const float* x, int col0, int M, float (&xr)[EC_OPT]) {
#pragma unroll
  for (int k = 0; k < EC_OPT; ++k) {
    const int idx = threadIdx.x + EC_THREADS * k, r = idx >> 5, f = idx & 31;
    xr[k] = r < M ? __ldcg(x + (size_t)r * EC_D + col0 + f) : 0.f;
  }
}

// bf16 rows [M][ld] (columns col0 .. col0 + 512) of global memory into the activation buffer
// (every load issued before any store)
__device__ __forceinline__ void ec_load_act(bf16* act, const bf16* src, int ld, int col0, int M) {
  constexpr int PER = EC_MAXM * (EC_D / 8) / EC_THREADS;  // 8
  uint4 v[PER];
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int i = threadIdx.x + EC_THREADS * k, r = i >> 6, q = i & 63;
    if (r < M) v[k] = __ldcg(reinterpret_cast<const uint4*>(src + (size_t)r * ld + col0 + 8 * q));
  }
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int i = threadIdx.x + EC_THREADS * k, r = i >> 6, q = i & 63;
    if (r < M) *reinterpret_cast<uint4*>(act + r * EC_AST + 8 * q) = v[k];
  }
}

// LayerNorm (d = 512) of fp32 rows of x by one warp, the lane partition and reduction
// order of layernorm_vec_kernel (kernels.cuh), bf16 out; NR rows per call with every
// row's loads issued before any arithmetic (rows >= M skipped)
template <int NR>
__device__ __forceinline__ void ec_ln_rows(const float* __restrict__ x, const int (&rows)[NR], int M,
                                           const float* __restrict__ g, const float* __restrict__ b, bf16* out,
                                           int ldo) {
  const int lane = threadIdx.x & 31;
  float4 v[NR][4];
#pragma unroll
  for (int j = 0; j < NR; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i)
      v[j][i] = __ldcg(reinterpret_cast<const float4*>(x + (size_t)min(rows[j], M - 1) * EC_D) + lane + 32 * i);
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) s += (v[j][i].x + v[j][i].y) + (v[j][i].z + v[j][i].w);
    const float mean = warp_sum(s) / EC_D;
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float a = v[j][i].x - mean, bb = v[j][i].y - mean, c = v[j][i].z - mean, e = v[j][i].w - mean;
      q += (a * a + bb * bb) + (c * c + e * e);
    }
    const float inv = 1.0f / sqrtf(warp_sum(q) / EC_D + 1e-5f);
    if (rows[j] < M) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int c4 = (lane + 32 * i) * 4;
        const float4 gg = __ldg(reinterpret_cast<const float4*>(g + c4)), bv = __ldg(reinterpret_cast<const float4*>(b + c4));
        __nv_bfloat162 lo = __floats2bfloat162_rn((v[j][i].x - mean) * inv * gg.x + bv.x,
                                                  (v[j][i].y - mean) * inv * gg.y + bv.y);
        __nv_bfloat162 hi = __floats2bfloat162_rn((v[j][i].z - mean) * inv * gg.z + bv.z,
                                                  (v[j][i].w - mean) * inv * gg.w + bv.w);
        uint2 u;
        u.x = *reinterpret_cast<uint32_t*>(&lo);
        u.y = *reinterpret_cast<uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(out + (size_t)rows[j] * ldo + c4) = u;
      }
    }
  }
}

template <bool TWO>  // M > 32: the row halves split the warps
__global__ void __cluster_dims__(EC_CN, 1, 1) __launch_bounds__(EC_THREADS, 1) enc_cluster_kernel(EcParams p) {
  extern __shared__ __align__(1024) uint8_t esm[];
  uint8_t* ring = esm + EcSmem::RING;
  bf16* act = reinterpret_cast<bf16*>(esm + EcSmem::ACT);
  float* red = reinterpret_cast<float*>(esm + EcSmem::RED);
  float* prm = reinterpret_cast<float*>(esm + EcSmem::PRM);
  uint64_t* full = reinterpret_cast<uint64_t*>(esm + EcSmem::BAR);
  float *pbqkv = prm, *pbo = prm + 96, *pb1 = prm + 128, *pb2 = prm + 256;
  pdl_trigger();
  unsigned long long ts[40];
  int nts = 0;
#define EC_TS() if (p.trace) ts[nts++] = dc_now()
  EC_TS();
  const long long clk0 = clock64();
  const int c = blockIdx.x;  // the grid is exactly one cluster
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int hh = c >> 1, half = c & 1;
  if (tid == 0) {
    for (int s = 0; s < EC_NSLOT; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  int issued = 0;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  auto issue_upto = [&](int n) {
    n = min(n, EC_NCH);
    if (tid == 0)
      for (int i = issued; i < n; ++i) {
        uint64_t* bar = &full[i % EC_NSLOT];
        const bf16 *s0, *s1;
        ec_chunk_src(p, i, c, s0, s1);
        mbar_arrive_expect_tx(bar, EC_CHUNK);
        uint8_t* dst = ring + (i % EC_NSLOT) * EC_CHUNK;
        dc_bulk_load(dst, s0, EC_CHUNK / 2, bar, pol);
        dc_bulk_load(dst + EC_CHUNK / 2, s1, EC_CHUNK / 2, bar, pol);
      }
    issued = max(issued, n);
  };
  auto chunk = [&](int i) -> const bf16* {
    mbar_wait(&full[i % EC_NSLOT], (i / EC_NSLOT) & 1);
    return reinterpret_cast<const bf16*>(ring + (i % EC_NSLOT) * EC_CHUNK);
  };
  // after chunk i is consumed by every warp (the caller synchronised): refill its slot
  auto consumed = [&](int i) { issue_upto(i + 1 + EC_NSLOT); };
  issue_upto(EC_NSLOT);
  // static parameters (independent of the previous launch)
  for (int i = tid; i < EcSmem::NPRM; i += EC_THREADS) {
    float v;
    if (i < 96) v = p.bqkv[(i >> 5) * EC_D + hh * 64 + half * 32 + (i & 31)];
    else if (i < 128) v = p.bo[32 * c + i - 96];
    else if (i < 256) v = p.b1[128 * c + i - 128];
    else v = p.b2[32 * c + i - 256];
    prm[i] = v;
  }
  pdl_wait();
  const int M = p.M;
  EC_TS();
  // this CTA's residual columns x[:, 32 c .. +32] (only this CTA writes them)
  float xr[EC_OPT];
  ec_load_res(p.x, 32 * c, M, xr);
  // ---- QKV: q / k / v dims 32 half .. +32 of head hh, every row ----
  ec_load_act(act, p.y, EC_D, 0, M);
  __syncthreads();
  EC_TS();
  for (int j = 0; j < 3; ++j) {
    float acc[4][4] = {};
    ec_mma_chunk<TWO>(chunk(j), act, M, acc);
    float v[EC_OPT];
    ec_reduce<TWO>(acc, red, M, v);
    consumed(j);
#pragma unroll
    for (int k = 0; k < EC_OPT; ++k) {
      const int idx = tid + EC_THREADS * k, r = idx >> 5, f = idx & 31;
      if (r < M)
        p.qkv[(size_t)r * (3 * EC_D) + j * EC_D + hh * 64 + half * 32 + f] = __float2bfloat16_rn(v[k] + pbqkv[j * 32 + f]);
    }
  }
  EC_TS();
  cluster_sync_all();  // B1: q / k / v of every head
  EC_TS();
  // ---- self-attention: head hh, query rows r = half, half + 2, ... (warp per row) ----
  {
    float* Qs = reinterpret_cast<float*>(act);
    float* Ks = Qs + EC_MAXM * EC_KVST;
    float* Vs = Ks + EC_MAXM * EC_KVST;
    constexpr int PER = EC_MAXM * 32 / EC_THREADS;  // bf16 pairs per thread per matrix
    __nv_bfloat162 qv[PER], kv[PER], vv[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int i = tid + EC_THREADS * k, r = min(i >> 5, M - 1), q2 = i & 31;
      const bf16* row = p.qkv + (size_t)r * (3 * EC_D) + hh * 64 + 2 * q2;
      qv[k] = __ldcg(reinterpret_cast<const __nv_bfloat162*>(row));
      kv[k] = __ldcg(reinterpret_cast<const __nv_bfloat162*>(row + EC_D));
      vv[k] = __ldcg(reinterpret_cast<const __nv_bfloat162*>(row + 2 * EC_D));
    }
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int i = tid + EC_THREADS * k, r = i >> 5, q2 = i & 31;
      if (r < M) {
        const float2 qf = __bfloat1622float2(qv[k]), kf = __bfloat1622float2(kv[k]), vf = __bfloat1622float2(vv[k]);
        Qs[r * EC_KVST + 2 * q2] = qf.x;
        Qs[r * EC_KVST + 2 * q2 + 1] = qf.y;
        Ks[r * EC_KVST + 2 * q2] = kf.x;
        Ks[r * EC_KVST + 2 * q2 + 1] = kf.y;
        Vs[r * EC_KVST + 2 * q2] = vf.x;
        Vs[r * EC_KVST + 2 * q2 + 1] = vf.y;
      }
    }
    if (tid < M) {  // each row's sequence (first row, length)
      int s0 = 0, sl = M;
      for (int s = 0; s < p.nseq; ++s) {
        const int o = __ldg(p.seq_off + s), l = __ldg(p.seq_len + s);
        if (tid >= o && tid < o + l) {
          s0 = o;
          sl = l;
        }
      }
      red[2 * tid] = __int_as_float(s0);
      red[2 * tid + 1] = __int_as_float(sl);
    }
    __syncthreads();
    for (int r = half + 2 * warp; r < M; r += 2 * (EC_THREADS / 32)) {
      const int s0 = __float_as_int(red[2 * r]), sl = __float_as_int(red[2 * r + 1]);
      // lane j scores keys j and j + 32 (query row broadcast from shared memory)
      const float* qr = Qs + r * EC_KVST;
      float sc[2];
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        const int j = lane + 32 * h2;
        const float* kr = Ks + (s0 + min(j, sl - 1)) * EC_KVST;
        float a[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int e = 0; e < EC_DH; e += 4)
#pragma unroll
          for (int u = 0; u < 4; ++u) a[u] = fmaf(qr[e + u], kr[e + u], a[u]);
        sc[h2] = j < sl ? ((a[0] + a[1]) + (a[2] + a[3])) * p.att_scale : -INFINITY;
      }
      const float mx = warp_max(fmaxf(sc[0], sc[1]));
      const float e0 = lane < sl ? ex2f((sc[0] - mx) * LOG2E) : 0.f;
      const float e1 = lane + 32 < sl ? ex2f((sc[1] - mx) * LOG2E) : 0.f;
      const float inv = 1.0f / warp_sum(e0 + e1);
      // lane owns output dims 2 lane, 2 lane + 1; keys in groups of four (independent chains)
      float o0[4] = {0.f, 0.f, 0.f, 0.f}, o1[4] = {0.f, 0.f, 0.f, 0.f};
      for (int j0 = 0; j0 < sl; j0 += 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = j0 + u;
          float pj = __shfl_sync(0xffffffffu, j < 32 ? e0 : e1, j & 31);
          if (j >= sl) pj = 0.f;
          const float* vr = Vs + (s0 + min(j, sl - 1)) * EC_KVST + 2 * lane;  // (odd row stride: scalar loads)
          o0[u] = fmaf(pj, vr[0], o0[u]);
          o1[u] = fmaf(pj, vr[1], o1[u]);
        }
      }
      *reinterpret_cast<__nv_bfloat162*>(p.ctx + (size_t)r * EC_D + hh * 64 + 2 * lane) =
          __floats2bfloat162_rn(((o0[0] + o0[1]) + (o0[2] + o0[3])) * inv, ((o1[0] + o1[1]) + (o1[2] + o1[3])) * inv);
    }
  }
  EC_TS();
  cluster_sync_all();  // B2: ctx of every head
  EC_TS();
  // ---- Wo + residual: x[:, 32 c .. +32] ----
  ec_load_act(act, p.ctx, EC_D, 0, M);
  __syncthreads();
  {
    float acc[4][4] = {};
    ec_mma_chunk<TWO>(chunk(3), act, M, acc);
    float v[EC_OPT];
    ec_reduce<TWO>(acc, red, M, v);
    consumed(3);
#pragma unroll
    for (int k = 0; k < EC_OPT; ++k) {
      const int idx = tid + EC_THREADS * k, r = idx >> 5, f = idx & 31;
      xr[k] = xr[k] + (v[k] + pbo[f]);
      if (r < M) p.x[(size_t)r * EC_D + 32 * c + f] = xr[k];
    }
  }
  EC_TS();
  cluster_sync_all();  // B3: x after the self-attention block
  EC_TS();
  // ---- LN2 (every CTA, every row) -> W1 + ReLU: hidden[:, 128 c .. +128] ----
  if (warp < M) {  // rows warp, warp + 16, warp + 32, warp + 48 (LayerNorm vectors through L1)
    const int rows[4] = {warp, warp + EC_WARPS, warp + 2 * EC_WARPS, warp + 3 * EC_WARPS};
    ec_ln_rows<4>(p.x, rows, M, p.ln2g, p.ln2b, act, EC_AST);
  }
  __syncthreads();
  EC_TS();
  for (int j = 4; j < 8; ++j) {
    float acc[4][4] = {};
    const bf16* wch = chunk(j);
    EC_TS();
    ec_mma_chunk<TWO>(wch, act, M, acc);
    EC_TS();
    float v[EC_OPT];
    ec_reduce<TWO>(acc, red, M, v);
    consumed(j);
#pragma unroll
    for (int k = 0; k < EC_OPT; ++k) {
      const int idx = tid + EC_THREADS * k, r = idx >> 5, f = idx & 31;
      if (r < M)
        p.hid[(size_t)r * EC_FF + 128 * c + 32 * (j - 4) + f] =
            __float2bfloat16_rn(fmaxf(v[k] + pb1[32 * (j - 4) + f], 0.f));
    }
  }
  EC_TS();
  cluster_sync_all();  // B4: the hidden layer
  EC_TS();
  // ---- W2 + residual: x[:, 32 c .. +32] over K = 2048 in four 512-wide slices ----
  {
    float acc[4][4] = {};
    for (int j = 8; j < 12; ++j) {
      ec_load_act(act, p.hid, EC_FF, 512 * (j - 8), M);
      __syncthreads();
      ec_mma_chunk<TWO>(chunk(j), act, M, acc);
      __syncthreads();
      consumed(j);
    }
    float v[EC_OPT];
    ec_reduce<TWO>(acc, red, M, v);
#pragma unroll
    for (int k = 0; k < EC_OPT; ++k) {
      const int idx = tid + EC_THREADS * k, r = idx >> 5, f = idx & 31;
      if (r < M) p.x[(size_t)r * EC_D + 32 * c + f] = xr[k] + (v[k] + pb2[f]);
    }
  }
  EC_TS();
  cluster_sync_all();  // B5: x after the feed-forward block
  EC_TS();
  // ---- the next LayerNorm (next layer's LN1 / the final encoder LN): rows c, c + 16, ... ----
  if (c + EC_CN * warp < M) {
    const int rows[1] = {c + EC_CN * warp};
    ec_ln_rows<1>(p.x, rows, M, p.lnng, p.lnnb, p.y, EC_D);
  }
  EC_TS();
  if (p.trace && c == 0 && tid == 0) {
    printf("ec trace M=%d:", p.M);
    for (int i = 1; i < nts; ++i) printf(" %.2f", (ts[i] - ts[i - 1]) * 1e-3);
    printf("  total %.2f us  (%.0f MHz)\n", (ts[nts - 1] - ts[0]) * 1e-3,
           (double)(clock64() - clk0) * 1e3 / (double)(ts[nts - 1] - ts[0]));
  }
#undef EC_TS
}

}  // namespace hrt
