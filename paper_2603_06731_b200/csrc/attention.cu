// attention.cu - K3: the fused attention layer as ONE flash-style kernel.
//
// Reference: the attention graph transpose(k) -> batch_matmul(q, kt) ->
// add(bias) -> softmax -> batch_matmul(soft, v) (test_frontend.cpp:275-305;
// PAPER.md:371-378), whose reduce-reduce fusion with online-softmax
// correction is a stub in the reference
// (attention.cpp:1). This kernel realises the paper's three steps natively:
//   rr-fusion      : the N x N score matrix never reaches HBM; running row max
//                    m and denominator l, the output accumulator rescaled by
//                    exp(m_old - m_new) (the paper's "correction", applied once
//                    per KV tile, not per element: outline_matmuls);
//   matmul outline : S = Q K^T and O += P V are separate tcgen05 MMAs into
//                    TMEM (S double-buffered, O resident for the whole row
//                    block);
//   wmma fusion    : the softmax works on the S tile in registers
//                    (tcgen05.ld), P goes to shared memory once as the A
//                    operand of the PV MMA.
// Extensions the BASELINE configs need: a scale on QK^T (the reference has
// none; scale = 1 reproduces it) and causal masking (== the -inf upper-
// triangular additive bias; causal KV tiles above the diagonal are skipped).
//
// CTA = one (b, h) and 128 query rows. Warps: 0 TMA, 1 MMA, 2 TMEM alloc,
// 4-7 softmax/correction/epilogue (thread t owns query row t).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "afg_internal.h"
#include "epilogue.cuh"
#include "sm100.cuh"

namespace afg {
namespace {

using namespace sm100;

constexpr int BM = 128;  // query rows per CTA
constexpr int BN = 128;  // keys per KV tile

struct AttnArgs {
  const float* bias;  // [BH, Nq, Nk] or null
  void* o;
  int64_t o_ss, o_hs, o_bs;  // output strides (elements) of seq / head / batch
  int BH, H, Nq, Nk;
  float scale_log2;  // scale * log2(e)
  int causal;
  int o_dtype;
};

template <int D>
struct AttnSmem {
  static constexpr int KV_STAGES = D == 64 ? 4 : 2;
  static constexpr int TILE = BM * D * 2;  // one Q / K / V tile (BM == BN rows)
  static constexpr int QA_OFF = 0;
  static constexpr int QB_OFF = TILE;
  static constexpr int K_OFF = 2 * TILE;
  static constexpr int V_OFF = K_OFF + KV_STAGES * TILE;
  static constexpr int BAR_OFF = V_OFF + KV_STAGES * TILE;
  // q_full, k_full[S], k_empty[S], v_full[S], v_empty[S], s_full[2], p_full[2], o_done
  static constexpr int NUM_BARS = 1 + 4 * KV_STAGES + 5;
  static constexpr int TOTAL = BAR_OFF + NUM_BARS * 8 + 16 + 1024;
};

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA pipe (x <= 0): Cody-Waite split x = j + f, f in [0,1), cubic
// least-squares fit of 2^f (max rel err 7.7e-5, below the 16-bit rounding of
// P), exponent added as an integer. Used for a quarter of the probabilities so
// the MUFU (ex2) pipe and the FMA pipe share the exponentials.
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -127.0f);
  const float j = floorf(x);
  const float f = x - j;
  const float p = fmaf(fmaf(fmaf(0.077907223f, f, 0.226233534f), f, 0.695776742f), f, 0.999927886f);
  return __int_as_float(__float_as_int(p) + (__float2int_rn(j) << 23));
}

// Blackwell packed fp32x2 FMA / ADD and 3-input max: halve the FMA-pipe work
// of the softmax (the pipe that bounds it; MUFU ex2 has headroom).
__device__ __forceinline__ uint64_t f2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2split(uint64_t v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

__device__ __forceinline__ uint32_t pack2(float a, float b, bool bf16) {
  return bf16 ? pack_bf16(a, b) : pack_f16(a, b);
}

// One CTA = one (b, h) x two 128-row query tiles A and B ("ping-pong"): while
// the softmax warpgroup of one tile works, the tensor core runs the other
// tile's MMAs. TMEM (512 columns): S_A [0,128) S_B [128,256) O_A, O_B after.
// P is written back over S as packed 16-bit values and consumed by the PV MMA
// straight from TMEM (A operand in tensor memory), so shared memory holds only
// Q_A, Q_B and the K / V ring.
// Warps: 0 TMA, 1 MMA issuer, 2 TMEM allocator, 4-7 softmax A, 8-11 softmax B.
template <int D, bool BF16>
__global__ void __launch_bounds__(384, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tmQ,
                    const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const AttnArgs args) {
  using L = AttnSmem<D>;
  constexpr int KS = L::KV_STAGES;
  constexpr int DB = D / 64;  // 128-byte swizzle atoms per row
  constexpr uint32_t TMEM_COLS = 512;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  uint64_t* k_empty = k_full + KS;
  uint64_t* v_full = k_empty + KS;
  uint64_t* v_empty = v_full + KS;
  uint64_t* s_full = v_empty + KS;  // [2]
  uint64_t* p_full = s_full + 2;    // [2]
  uint64_t* o_done = p_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + L::NUM_BARS);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  const int n_pairs = (args.Nq + 2 * BM - 1) / (2 * BM);
  const int qp = n_pairs - 1 - static_cast<int>(blockIdx.x);  // heavy causal pairs first
  const int bh = blockIdx.y;
  const int hh = bh % args.H;
  const int bb = bh / args.H;
  const int q0 = qp * 2 * BM;
  const int nkv_all = (args.Nk + BN - 1) / BN;
  int nkv[2];
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    const int first = q0 + g * BM;
    if (first >= args.Nq) {
      nkv[g] = 0;
    } else {
      nkv[g] = args.causal ? min(nkv_all, (first + BM - 1) / BN + 1) : nkv_all;
    }
  }
  const int nkv_max = max(nkv[0], nkv[1]);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    mbar_init(q_full, 1);
    for (int s = 0; s < KS; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int g = 0; g < 2; ++g) {
      mbar_init(&s_full[g], 1);
      mbar_init(&p_full[g], 128);
    }
    mbar_init(o_done, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t S_COL[2] = {0u, static_cast<uint32_t>(BN)};
  const uint32_t O_COL[2] = {static_cast<uint32_t>(2 * BN), static_cast<uint32_t>(2 * BN + D)};

  if (warp == 0) {
    // --------------------------------------------------------------- TMA --
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, 2 * L::TILE);
      for (int g = 0; g < 2; ++g)
        for (int a = 0; a < DB; ++a)
          tma_load_4d(smem + (g ? L::QB_OFF : L::QA_OFF) + a * (BM * 128), &tmQ, q_full, a * 64,
                      q0 + g * BM, hh, bb);
      for (int j = 0; j < nkv_max; ++j) {
        const int st = j % KS;
        const uint32_t ph = (j / KS) & 1;
        mbar_wait(&k_empty[st], ph ^ 1);
        mbar_arrive_expect_tx(&k_full[st], L::TILE);
        for (int a = 0; a < DB; ++a)
          tma_load_4d(smem + L::K_OFF + st * L::TILE + a * (BN * 128), &tmK, &k_full[st], a * 64,
                      j * BN, hh, bb);
        mbar_wait(&v_empty[st], ph ^ 1);
        mbar_arrive_expect_tx(&v_full[st], L::TILE);
        for (int a = 0; a < DB; ++a)
          tma_load_4d(smem + L::V_OFF + st * L::TILE + a * (BN * 128), &tmV, &v_full[st], a * 64,
                      j * BN, hh, bb);
      }
    }
  } else if (warp == 1) {
    // --------------------------------------------------------------- MMA --
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_f16(BM, BN, BF16 ? 1u : 0u, 0u, 0u);
      constexpr uint32_t idesc_o = idesc_f16(BM, D, BF16 ? 1u : 0u, 0u, 1u);
      const uint32_t q_addr[2] = {smem_u32(smem + L::QA_OFF), smem_u32(smem + L::QB_OFF)};
      auto issue_s = [&](int g, int j) {
        const uint32_t k_addr = smem_u32(smem + L::K_OFF + (j % KS) * L::TILE);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk / 4) * (BM * 128) + (kk % 4) * 32;
          mma_f16_ss(tmem + S_COL[g], desc_kmajor_sw128(q_addr[g] + off),
                     desc_kmajor_sw128(k_addr + off), idesc_s, kk > 0 ? 1u : 0u);
        }
        mma_commit(&s_full[g]);
      };
      auto issue_pv = [&](int g, int j) {
        const uint32_t v_addr = smem_u32(smem + L::V_OFF + (j % KS) * L::TILE);
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk)
          mma_f16_ts(tmem + O_COL[g], tmem + S_COL[g] + kk * 8,
                     desc_mnmajor_sw128(v_addr + kk * 16 * 128, BN * 128), idesc_o,
                     (j > 0 || kk > 0) ? 1u : 0u);
      };
      mbar_wait(q_full, 0);
      mbar_wait(&k_full[0], 0);
      tc_fence_after();
      if (nkv[0] > 0) issue_s(0, 0);
      if (nkv[1] > 0) issue_s(1, 0);
      mma_commit(&k_empty[0]);
      for (int j = 0; j < nkv_max; ++j) {
        const int st = j % KS;
        const int jn = j + 1;
        bool k_next_ready = false;
        mbar_wait(&v_full[st], (j / KS) & 1);
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          if (j < nkv[g]) {
            mbar_wait(&p_full[g], j & 1);
            tc_fence_after();
            issue_pv(g, j);
            if (jn < nkv[g]) {
              if (!k_next_ready) {
                mbar_wait(&k_full[jn % KS], (jn / KS) & 1);
                tc_fence_after();
                k_next_ready = true;
              }
              issue_s(g, jn);  // runs after PV(g, j) on the tensor pipe: P(j) consumed first
            }
          }
        }
        mma_commit(&v_empty[st]);
        if (k_next_ready) mma_commit(&k_empty[jn % KS]);
      }
      mma_commit(o_done);
    }
  } else if (warp >= 4) {
    // --------------------------------- softmax / correction / epilogue (per tile)
    const int g = (warp - 4) / 4;
    const int w4 = warp % 4;
    const int row = w4 * 32 + lane;
    const int qi = q0 + g * BM + row;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(w4 * 32) << 16);
    const uint32_t s_base = lane_base + S_COL[g];
    const uint32_t o_base = lane_base + O_COL[g];
    const float* brow =
        args.bias ? args.bias + (static_cast<int64_t>(bh) * args.Nq + min(qi, args.Nq - 1)) *
                                    args.Nk
                  : nullptr;
    float m = -INFINITY;  // running max (scaled log2 units)
    float l = 0.0f;
    for (int j = 0; j < nkv[g]; ++j) {
      mbar_wait(&s_full[g], j & 1);  // also implies PV(g, j-1) completed (in-order MMAs)
      tc_fence_after();
      const int k0 = j * BN;
      const bool need_mask = (args.causal && k0 + BN - 1 > q0 + g * BM) || k0 + BN > args.Nk;
      auto score = [&](uint32_t raw, int kj) {
        float v = __uint_as_float(raw) * args.scale_log2;
        if (brow) v = kj < args.Nk ? fmaf(__ldg(brow + kj), 1.4426950408889634f, v) : v;
        if (need_mask && (kj >= args.Nk || (args.causal && kj > qi))) v = -INFINITY;
        return v;
      };
      // Fast path (no additive bias, no mask in this tile, scale > 0): the max
      // is taken on the raw scores and each probability is one FFMA + EX2.
      // The masked path (causal diagonal / key tail / bias) is per element.
      const bool fast = brow == nullptr && !need_mask && args.scale_log2 > 0.0f;
      float tmax = -INFINITY;
      if (fast) {
        // TMEM loads double-buffered: chunk c+1 is in flight while c is reduced
        uint32_t sa[32], sb[32];
        tmem_ld32(s_base, sa);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t(&cur)[32] = (c & 1) ? sb : sa;
          uint32_t(&nxt)[32] = (c & 1) ? sa : sb;
          if (c + 1 < BN / 32) tmem_ld32(s_base + (c + 1) * 32, nxt);
#pragma unroll
          for (int e = 0; e < 32; e += 2)
            tmax = fmax3(tmax, __uint_as_float(cur[e]), __uint_as_float(cur[e + 1]));
          tmem_wait_ld();
        }
        tmax *= args.scale_log2;
      } else {
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t sr[32];
          tmem_ld32(s_base + c * 32, sr);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e) tmax = fmaxf(tmax, score(sr[e], k0 + c * 32 + e));
        }
      }
      // lazy rescaling: the running max only moves when it grows by more than
      // 8 (log2 units; P stays <= 2^8, exact in fp16/bf16 range), so the O
      // correction below is rare after the first tiles.
      const float m_cand = fmaxf(m, tmax);
      const bool upd = m == -INFINITY || m_cand > m + 8.0f;
      const float m_new = upd ? m_cand : m;
      const float base = m_new == -INFINITY ? 0.0f : m_new;
      const float alpha = upd ? ex2(m - base) : 1.0f;  // 0 on the first tile
      // correction O *= exp(m_old - m_new) once per tile (warp-uniform decision:
      // tcgen05.ld/st are warp-collective; rows whose max did not move use 1)
      if (j > 0 && __any_sync(0xffffffffu, upd)) {
#pragma unroll 1
        for (int c = 0; c < D / 32; ++c) {
          uint32_t o[32];
          tmem_ld32(o_base + c * 32, o);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
          tmem_st32(o_base + c * 32, o);
        }
      }
      m = m_new;
      // pass 2: P = exp2(s - m) packed to 16 bit, written over S (cols 16c..)
      float tsum = 0.0f;
      const float nb = -base;
      uint32_t sa2[32], sb2[32];
      tmem_ld32(s_base, sa2);
      tmem_wait_ld();
#pragma unroll
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t(&sr)[32] = (c & 1) ? sb2 : sa2;
        uint32_t(&nxt)[32] = (c & 1) ? sa2 : sb2;
        // the next S chunk (columns 32(c+1)..) is not overwritten by P chunk c
        // (columns 16c..16c+15), so it can be loaded ahead
        if (c + 1 < BN / 32) tmem_ld32(s_base + (c + 1) * 32, nxt);
        uint32_t pk[16];
        if (fast) {
          const uint64_t sc2 = f2(args.scale_log2, args.scale_log2), nb2 = f2(nb, nb);
          uint64_t acc2 = f2(0.0f, 0.0f);
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            float x0, x1;
            f2split(ffma2(f2(__uint_as_float(sr[2 * e]), __uint_as_float(sr[2 * e + 1])), sc2, nb2),
                    x0, x1);
            const float p0 = ex2(x0), p1 = ex2(x1);
            acc2 = fadd2(acc2, f2(p0, p1));
            pk[e] = pack2(p0, p1, BF16);
          }
          float a0, a1;
          f2split(acc2, a0, a1);
          tsum += a0 + a1;
        } else {
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const float p0 = ex2(score(sr[2 * e], k0 + c * 32 + 2 * e) + nb);
            const float p1 = ex2(score(sr[2 * e + 1], k0 + c * 32 + 2 * e + 1) + nb);
            tsum += p0 + p1;
            pk[e] = pack2(p0, p1, BF16);
          }
        }
        tmem_st16(s_base + c * 16, pk);
        tmem_wait_ld();
      }
      tmem_wait_st();
      l = l * alpha + tsum;
      tc_fence_before();
      mbar_arrive(&p_full[g]);
    }
    // ---- epilogue: O / l -> global
    mbar_wait(o_done, 0);
    tc_fence_after();
    const float inv_l = l > 0.0f ? 1.0f / l : 0.0f;
    const bool valid = qi < args.Nq && nkv[g] > 0;
#pragma unroll 1
    for (int c = 0; c < D / 32; ++c) {
      uint32_t o[32];
      tmem_ld32(o_base + c * 32, o);
      tmem_wait_ld();
      if (!valid) continue;
      const int64_t base_idx = static_cast<int64_t>(bb) * args.o_bs +
                               static_cast<int64_t>(hh) * args.o_hs +
                               static_cast<int64_t>(qi) * args.o_ss + c * 32;
      if (args.o_dtype == AFG_F32) {
        float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(args.o) + base_idx);
#pragma unroll
        for (int v = 0; v < 8; ++v)
          dst[v] = make_float4(__uint_as_float(o[4 * v]) * inv_l, __uint_as_float(o[4 * v + 1]) * inv_l,
                               __uint_as_float(o[4 * v + 2]) * inv_l,
                               __uint_as_float(o[4 * v + 3]) * inv_l);
      } else {
        const bool ob = args.o_dtype == AFG_BF16;
        uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(args.o) + base_idx);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          uint4 u;
          u.x = pack2(__uint_as_float(o[8 * v + 0]) * inv_l, __uint_as_float(o[8 * v + 1]) * inv_l, ob);
          u.y = pack2(__uint_as_float(o[8 * v + 2]) * inv_l, __uint_as_float(o[8 * v + 3]) * inv_l, ob);
          u.z = pack2(__uint_as_float(o[8 * v + 4]) * inv_l, __uint_as_float(o[8 * v + 5]) * inv_l, ob);
          u.w = pack2(__uint_as_float(o[8 * v + 6]) * inv_l, __uint_as_float(o[8 * v + 7]) * inv_l, ob);
          dst[v] = u;
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<TMEM_COLS>(tmem);
  }
}

// ----------------------------------------------------------- SIMT fallback --
// Any D / dtype / length: one CTA per (bh, query row); scores staged in smem.
template <typename T>
__global__ void attn_simt_kernel(const T* __restrict__ q, const T* __restrict__ k,
                                 const T* __restrict__ v, const float* __restrict__ bias,
                                 void* __restrict__ o, int Nq, int Nk, int D, float scale,
                                 int causal, int o_dtype) {
  extern __shared__ float sc[];  // Nk scores + 32 reduction slots
  float* red = sc + Nk;
  const int i = blockIdx.x;
  const int64_t bh = blockIdx.y;
  const T* qr = q + (bh * Nq + i) * D;
  float mx = -INFINITY;
  for (int j = threadIdx.x; j < Nk; j += blockDim.x) {
    const T* kr = k + (bh * Nk + j) * D;
    float acc = 0.0f;
    for (int d = 0; d < D; ++d) acc = fmaf(OutCvt<T>::from(qr[d]), OutCvt<T>::from(kr[d]), acc);
    acc *= scale;
    if (bias) acc += bias[(bh * Nq + i) * Nk + j];
    if (causal && j > i) acc = -INFINITY;
    sc[j] = acc;
    mx = fmaxf(mx, acc);
  }
  for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = mx;
  __syncthreads();
  mx = -INFINITY;
  for (int w = 0; w < blockDim.x / 32; ++w) mx = fmaxf(mx, red[w]);
  __syncthreads();
  const float base = mx == -INFINITY ? 0.0f : mx;
  float sum = 0.0f;
  for (int j = threadIdx.x; j < Nk; j += blockDim.x) {
    const float e = expf(sc[j] - base);
    sc[j] = e;
    sum += e;
  }
  for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
  if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = sum;
  __syncthreads();
  sum = 0.0f;
  for (int w = 0; w < blockDim.x / 32; ++w) sum += red[w];
  const float inv = sum > 0.0f ? 1.0f / sum : 0.0f;
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    float acc = 0.0f;
    for (int j = 0; j < Nk; ++j) acc = fmaf(sc[j], OutCvt<T>::from(v[(bh * Nk + j) * D + d]), acc);
    acc *= inv;
    const int64_t idx = (bh * Nq + i) * D + d;
    if (o_dtype == AFG_F32)
      reinterpret_cast<float*>(o)[idx] = acc;
    else if (o_dtype == AFG_F16)
      reinterpret_cast<__half*>(o)[idx] = __float2half_rn(acc);
    else
      reinterpret_cast<__nv_bfloat16*>(o)[idx] = __float2bfloat16_rn(acc);
  }
}

template <int D, bool BF16>
cudaError_t launch_tc(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                      const AttnArgs& a, cudaStream_t s) {
  auto kern = attn_fwd_kernel<D, BF16>;
  constexpr int smem = AttnSmem<D>::TOTAL;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  dim3 grid((a.Nq + 2 * BM - 1) / (2 * BM), a.BH);
  kern<<<grid, 384, smem, s>>>(tq, tk, tv, a);
  count_launch();
  return cudaGetLastError();
}

}  // namespace
}  // namespace afg

using namespace afg;

namespace afg {
namespace {

// Strides in elements: s = sequence row, h = head, b = batch (d is unit).
struct Strides {
  int64_t s, h, b;
};

afg_status attention_core(const void* q, const void* k, const void* v, const float* bias, void* o,
                          int64_t B, int64_t H, int64_t Nq, int64_t Nk, int64_t D, float scale,
                          int causal, afg_dtype dt, afg_dtype od, Strides sq, Strides sk,
                          Strides sv, Strides so, bool contiguous, cudaStream_t s) {
  if (!q || !k || !v || !o) return set_error(AFG_ERR_INVALID_ARG, "afg_attention_fwd: null operand");
  if (B <= 0 || H <= 0 || Nq <= 0 || Nk <= 0 || D <= 0)
    return set_error(AFG_ERR_INVALID_ARG, "afg_attention_fwd: non-positive extent");
  if (!valid_dtype(dt) || !valid_dtype(od))
    return set_error(AFG_ERR_INVALID_ARG, "afg_attention_fwd: bad dtype");
  const int64_t BH = B * H;
  if (BH > 65535 || Nq >= (1 << 30) || Nk >= (1 << 30))
    return set_error(AFG_ERR_UNSUPPORTED, "afg_attention_fwd: extent too large");
  afg_status st = check_device();
  if (st != AFG_OK) return st;
  const bool strides_ok = (sq.s % 8 == 0) && (sq.h % 8 == 0) && (sq.b % 8 == 0) &&
                          (sk.s % 8 == 0) && (sk.h % 8 == 0) && (sk.b % 8 == 0) &&
                          (sv.s % 8 == 0) && (sv.h % 8 == 0) && (sv.b % 8 == 0);
  const bool tc = (dt == AFG_F16 || dt == AFG_BF16) && (D == 64 || D == 128) && aligned16(q) &&
                  aligned16(k) && aligned16(v) && aligned16(o) && strides_ok &&
                  (so.s % 8 == 0) && (so.h % 8 == 0) && (so.b % 8 == 0);
  if (tc) {
    const CUtensorMapDataType tdt =
        dt == AFG_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
    CUtensorMap tq, tk, tv;
    const uint32_t box[4] = {64, 128, 1, 1};
    auto map4 = [&](CUtensorMap* m, const void* base, int64_t N, Strides str) {
      const uint64_t dims[4] = {static_cast<uint64_t>(D), static_cast<uint64_t>(N),
                                static_cast<uint64_t>(H), static_cast<uint64_t>(B)};
      const uint64_t strides[3] = {static_cast<uint64_t>(str.s) * 2,
                                   static_cast<uint64_t>(str.h) * 2,
                                   static_cast<uint64_t>(str.b) * 2};
      return make_tmap(m, base, tdt, 4, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
    };
    if ((st = map4(&tq, q, Nq, sq)) != AFG_OK) return st;
    if ((st = map4(&tk, k, Nk, sk)) != AFG_OK) return st;
    if ((st = map4(&tv, v, Nk, sv)) != AFG_OK) return st;
    AttnArgs a;
    a.bias = bias;
    a.o = o;
    a.o_ss = so.s;
    a.o_hs = so.h;
    a.o_bs = so.b;
    a.BH = static_cast<int>(BH);
    a.H = static_cast<int>(H);
    a.Nq = static_cast<int>(Nq);
    a.Nk = static_cast<int>(Nk);
    a.scale_log2 = scale * 1.4426950408889634f;
    a.causal = causal;
    a.o_dtype = od;
    cudaError_t e;
    if (D == 128)
      e = dt == AFG_BF16 ? launch_tc<128, true>(tq, tk, tv, a, s) : launch_tc<128, false>(tq, tk, tv, a, s);
    else
      e = dt == AFG_BF16 ? launch_tc<64, true>(tq, tk, tv, a, s) : launch_tc<64, false>(tq, tk, tv, a, s);
    return cuda_status(e, "attention tc launch");
  }
  if (!contiguous)
    return set_error(AFG_ERR_UNSUPPORTED, "strided attention needs the tensor-core path "
                     "(f16/bf16, D in {64,128}, 16-byte strides)");
  const size_t smem = (static_cast<size_t>(Nk) + 32) * sizeof(float);
  if (smem > 200 * 1024) return set_error(AFG_ERR_UNSUPPORTED, "attention SIMT path: Nk too large");
  dim3 grid(static_cast<unsigned>(Nq), static_cast<unsigned>(BH));
#define AFG_ATT(T)                                                                              \
  do {                                                                                          \
    cudaFuncSetAttribute(attn_simt_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,      \
                         static_cast<int>(smem));                                               \
    attn_simt_kernel<T><<<grid, 128, smem, s>>>(                                                \
        reinterpret_cast<const T*>(q), reinterpret_cast<const T*>(k),                           \
        reinterpret_cast<const T*>(v), bias, o, (int)Nq, (int)Nk, (int)D, scale, causal, (int)od); \
  } while (0)
  if (dt == AFG_F32) AFG_ATT(float);
  else if (dt == AFG_F16) AFG_ATT(__half);
  else AFG_ATT(__nv_bfloat16);
#undef AFG_ATT
  count_launch();
  return cuda_status(cudaGetLastError(), "attention simt launch");
}

}  // namespace
}  // namespace afg

extern "C" afg_status afg_attention_fwd(const void* q, const void* k, const void* v,
                                        const float* bias, void* o, int64_t B, int64_t H,
                                        int64_t Nq, int64_t Nk, int64_t D, float scale,
                                        int causal, afg_dtype dt, afg_dtype od, void* stream) {
  const Strides sq{D, Nq * D, H * Nq * D}, sk{D, Nk * D, H * Nk * D};
  return attention_core(q, k, v, bias, o, B, H, Nq, Nk, D, scale, causal, dt, od, sq, sk, sk, sq,
                        true, static_cast<cudaStream_t>(stream));
}

extern "C" afg_status afg_attention_fwd_strided(
    const void* q, const void* k, const void* v, const float* bias, void* o, int64_t B,
    int64_t H, int64_t Nq, int64_t Nk, int64_t D, float scale, int causal, afg_dtype dt,
    afg_dtype od, const int64_t* q_strides, const int64_t* k_strides, const int64_t* v_strides,
    const int64_t* o_strides, void* stream) {
  if (!q_strides || !k_strides || !v_strides || !o_strides)
    return set_error(AFG_ERR_INVALID_ARG, "afg_attention_fwd_strided: null strides");
  auto S = [](const int64_t* p) { return Strides{p[0], p[1], p[2]}; };
  return attention_core(q, k, v, bias, o, B, H, Nq, Nk, D, scale, causal, dt, od, S(q_strides),
                        S(k_strides), S(v_strides), S(o_strides), false,
                        static_cast<cudaStream_t>(stream));
}
