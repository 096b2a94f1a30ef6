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
#include <cstdlib>
#include <map>
#include <mutex>
#include <queue>
#include <vector>

#include "afg_internal.h"
#include "epilogue.cuh"
#include "sm100.cuh"

namespace afg {
namespace {

using namespace sm100;

constexpr int BM = 128;  // query rows per CTA
constexpr int BN = 128;  // keys per KV tile
// Bit mask over the 8 pair slots of a 16-pair group: which exponential pairs
// use the FMA-pipe polynomial instead of MUFU ex2. Measured on B200 (round 2,
// with the S rows loaded as register pairs, `profiles/r02/attention/
// poly_pairs_ab.txt`): 1/8 of the pairs 1079 TFLOP/s non-causal, 903 causal;
// 0/8 the same; 2/8 1042 / 884; 3/8 986 / 804 and 4/8 929 / 745 (spills).
// The softmax is issue-bound, not MUFU-bound, once the pair moves are gone.
#ifndef AFG_POLY_PAIRS
#define AFG_POLY_PAIRS 0x02
#endif
constexpr unsigned POLY_PAIRS = AFG_POLY_PAIRS;


struct AttnArgs {
  const float* bias;  // [BH, Nq, Nk] or null
  void* o;
  int64_t o_ss, o_hs, o_bs;  // output strides (elements) of seq / head / batch
  int BH, H, Nq, Nk;
  float scale_log2;  // scale * log2(e)
  int causal;
  int o_dtype;
  int head_group;  // unit order: heads per group (see decode)
  // host-built schedule (attn_schedule): CTA c runs the unit codes
  // sched[sched_off[c] .. sched_off[c] + sched_cnt[c]), code = bh * n_pairs + qp
  const int* sched;
  const int* sched_off;
  const int* sched_cnt;
  int dyn;         // 0: static snake; else 1 + counter slot: units taken from a global
                   // atomic queue in `decode` order by whichever CTA is free
  int o_st32;      // 16-bit O rows 32-byte aligned: 256-bit stores
  int dbg;  // profiling aid (AFG_ATTN_DEBUG): 1 = no softmax math, 2 = no MMAs,
           // 3 = MMAs back to back (no softmax dependency)
};

// Dynamic unit queue, one counter pair per slot (stream_slot: one per stream,
// so concurrent launches on two streams never share a queue): [0] = next
// unit, [1] = CTA exits; the last CTA out resets both
// and the next launch on the stream touches them after griddepcontrol.wait.
constexpr int ATTN_SLOTS = 64;
__device__ unsigned int g_attn_queue[ATTN_SLOTS][2];

// Split rows (AFG_ATTN_SPLIT = 2): each query row's 128 scores are handled
// by two threads in two warpgroups (keys [0, 64) and [64, 128) of the KV
// tile), which exchange their partial row maxima through shared memory once
// per step; 16 softmax warps instead of 8, half the serial work per thread.
#ifndef AFG_ATTN_SPLIT
#define AFG_ATTN_SPLIT 1
#endif
constexpr int SPLIT = AFG_ATTN_SPLIT;
// Register split between the 4 TMA / MMA / TMEM warps and the 8 softmax
// warps: 128 x small + 256 x big must equal the CTA's launch allocation
// (384 x 168 = 64512; a larger sum never completes setmaxnreg.inc). 40 / 232
// spilled the MMA warp's descriptors to local memory inside the issue loop;
// 56 / 224 removes the spills: BERT D = 64 111.7 -> 105.0 us, D = 128
// 1109 -> 1132 TFLOP/s, causal 915 -> 937 (`profiles/r02/attention/regs_ab.txt`).
#ifndef AFG_ATTN_REGS_SMALL
#define AFG_ATTN_REGS_SMALL 56
#define AFG_ATTN_REGS_BIG 224
#endif
#ifndef AFG_ATTN_REGS_SMALL64  // D = 64: the MMA warp's issue loop spills at 56
#define AFG_ATTN_REGS_SMALL64 72   // (BERT attention 105-107 -> 103 us; 80 / 208
#define AFG_ATTN_REGS_BIG64 216    // spills the softmax instead: 112 us)
#endif
static_assert(SPLIT == 2 || (128 * AFG_ATTN_REGS_SMALL + 256 * AFG_ATTN_REGS_BIG <= 384 * 168 &&
                             128 * AFG_ATTN_REGS_SMALL64 + 256 * AFG_ATTN_REGS_BIG64 <= 384 * 168),
              "setmaxnreg split over the launch register allocation");
static_assert(SPLIT == 1 || SPLIT == 2, "AFG_ATTN_SPLIT");
constexpr int ATTN_THREADS = 128 + 256 * SPLIT;

template <int D>
struct AttnSmem {
  static constexpr int TILE = BM * D * 2;  // one Q / K / V tile (BM == BN rows)
  // K and V tiles share one ring (K(j), V(j), K(j+1), ...): 5 x 32 KB at D=128
  // keeps 2.5 KV tiles in flight next to the two resident Q tiles.
  // Q buffers: with two, the next unit's Q tiles load while the current unit
  // runs. Measured: +3% at D = 64 (BERT, 4-tile units); at D = 128 the two
  // K/V stages it would cost matter more (-1%), so one buffer there.
#ifndef AFG_ATTN_QBUF64
#define AFG_ATTN_QBUF64 2
#endif
  static constexpr int QBUF = D == 64 ? AFG_ATTN_QBUF64 : 1;
  // split rows need 8 KB of exchange buffers: one K/V stage fewer at D = 128
  static constexpr int STAGES = D == 64 ? (QBUF == 2 ? 8 : 10) : (QBUF == 2 ? 3 : (SPLIT == 2 ? 4 : 5));
  static constexpr int QA_OFF = 0;
  static constexpr int QB_OFF = TILE;
  static constexpr int QBUF_BYTES = 2 * TILE;
  static constexpr int RING_OFF = QBUF * QBUF_BYTES;
  // row-max exchange [step parity][tile][half][row] and row-sum exchange
  // [unit parity][tile][half][row] (floats), split rows only
  static constexpr int XCH_OFF = RING_OFF + STAGES * TILE;
  static constexpr int XCH_BYTES = SPLIT == 2 ? 2 * (2 * 2 * 2 * BM * 4) : 0;
  static constexpr int BAR_OFF = XCH_OFF + XCH_BYTES;
  // q_full[QBUF], q_empty[QBUF], kv_full[S], kv_empty[S], s_full[2], p_full[2][2],
  // o_full[OBUF][2], o_empty[OBUF][2], unit_full[UNIT_R], unit_empty[UNIT_R]
  static constexpr int UNIT_R = 4;  // dynamic schedule: unit ids in flight (TMA -> MMA, softmax)
  // O accumulators per tile: two (alternating units) when they fit in TMEM
  // next to S_A, S_B (D = 64): the next unit's PV MMAs then do not wait for
  // this unit's epilogue to read O out of TMEM
  static constexpr int OBUF = 2 * BN + 2 * 2 * D <= 512 ? 2 : 1;
  static constexpr int NUM_BARS = 2 * QBUF + 2 * STAGES + 6 + 4 * OBUF + 2 * UNIT_R;
  static constexpr int TOTAL = BAR_OFF + NUM_BARS * 8 + 16 + 4 * UNIT_R + 1024;
  static_assert(TOTAL <= 232448, "attention smem over the 227 KB opt-in limit");
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

// 2^x for a pair of floats on the FMA pipe (offloads the MUFU ex2 unit, which
// bounds the softmax): x = j + f with j = rint(x) by the 1.5*2^23 magic-number
// add, 2^f on [-0.5, 0.5] by a cubic minimax fit (max rel err 7.7e-5, below the
// 16-bit rounding of P), and j added to the exponent field. x is clamped at
// -120 (2^-120 rounds to 0 in fp16/bf16 P).
__device__ __forceinline__ void ex2_poly2(uint64_t x2, float& p0, float& p1) {
  constexpr float MAGIC = 12582912.0f;  // 1.5 * 2^23
  float x0, x1;
  f2split(x2, x0, x1);
  const uint64_t xx = f2(fmaxf(x0, -120.0f), fmaxf(x1, -120.0f));
  const uint64_t t = fadd2(xx, f2(MAGIC, MAGIC));
  const uint64_t j = fadd2(t, f2(-MAGIC, -MAGIC));
  const uint64_t fr = ffma2(j, f2(-1.0f, -1.0f), xx);  // x - j in [-0.5, 0.5]
  uint64_t p = ffma2(f2(0.05508886f, 0.05508886f), fr, f2(0.24260466f, 0.24260466f));
  p = ffma2(p, fr, f2(0.69327629f, 0.69327629f));
  p = ffma2(p, fr, f2(0.99992889f, 0.99992889f));
  float q0, q1, t0, t1;
  f2split(p, q0, q1);
  f2split(t, t0, t1);
  // the low bits of t hold j: (bits(t) << 23) == j << 23 (mod 2^32)
  p0 = __int_as_float(__float_as_int(q0) + (__float_as_int(t0) << 23));
  p1 = __int_as_float(__float_as_int(q1) + (__float_as_int(t1) << 23));
}

__device__ __forceinline__ uint32_t pack2(float a, float b, bool bf16) {
  return bf16 ? pack_bf16(a, b) : pack_f16(a, b);
}

// Persistent ping-pong kernel. A work unit = one (b, h) x two 128-row query
// tiles A and B: while the softmax warpgroup of one tile works, the tensor
// core runs the other tile's MMAs. One CTA per SM walks the units of the grid
// (snake order over a heavy-first list), so TMEM allocation, barrier set-up,
// the K/V stream and the output epilogue of one unit overlap the next unit's
// work instead of costing a CTA launch each.
// TMEM (512 columns): S_A [0,128) S_B [128,256) O_A, O_B after. P is written
// back over S as packed 16-bit values and consumed by the PV MMA straight from
// TMEM (A operand in tensor memory), so shared memory holds only Q_A, Q_B and
// the K / V ring. Each softmax thread reads its S row from TMEM once and keeps
// all 128 scores in registers: warpgroup 0 (TMA / MMA / TMEM alloc) gives
// registers to the two softmax warpgroups.
// Warps: 0 TMA, 1 MMA issuer, 2 TMEM allocator, 4-7 softmax A, 8-11 softmax B.
template <int D, bool BF16>
__global__ void __launch_bounds__(ATTN_THREADS, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tmQ,
                    const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const AttnArgs args) {
  using L = AttnSmem<D>;
  constexpr int NS = L::STAGES;
  constexpr int DB = D / 64;    // 128-byte swizzle atoms per row
  constexpr int NCH = BN / 32;  // 32-column chunks of an S row
  constexpr uint32_t TMEM_COLS = 512;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  constexpr int QBUF = L::QBUF;
  uint64_t* q_full = bars;            // [QBUF]
  uint64_t* q_empty = bars + QBUF;    // [QBUF]
  uint64_t* kv_full = bars + 2 * QBUF;
  uint64_t* kv_empty = kv_full + NS;
  uint64_t* s_full = kv_empty + NS;  // [2]
  uint64_t* p_full = s_full + 2;     // [tile][half]: P columns of keys [0,64) / [64,128)
  constexpr int OBUF = L::OBUF;
  uint64_t* o_full = p_full + 4;         // [OBUF][2]
  uint64_t* o_empty = o_full + 2 * OBUF;  // [OBUF][2]
  uint64_t* unit_full = o_empty + 2 * OBUF;        // [UNIT_R]
  uint64_t* unit_empty = unit_full + L::UNIT_R;    // [UNIT_R]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + L::NUM_BARS);
  int* unit_ring = reinterpret_cast<int*>(tmem_slot + 4);  // [UNIT_R]

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  const int n_pairs = (args.Nq + 2 * BM - 1) / (2 * BM);
  const int n_units = args.BH * n_pairs;
  const int nkv_all = (args.Nk + BN - 1) / BN;
  // Unit number u of this CTA -> linear unit index (snake over the grid:
  // rounds alternate direction so heavy and light units even out per CTA).
  // Linear order: heads in groups of HEAD_GROUP; inside a group the query-tile
  // pairs run from the last (heaviest under causal masking) down, all heads of
  // the group per pair (co-resident CTAs share the group's K/V in L2).
  // dynamic schedule, consumer side (MMA warp, softmax warps): the unit id the
  // TMA warp fetched for this CTA's u-th unit; one release arrival per warp
  auto unit_take = [&](int u) {
    const int slot = u % L::UNIT_R;
    mbar_wait(&unit_full[slot], (u / L::UNIT_R) & 1);
    const int lin = *reinterpret_cast<volatile int*>(&unit_ring[slot]);
    __syncwarp();
    if (lane == 0) mbar_arrive(&unit_empty[slot]);
    return lin;
  };
  auto unit_of = [&](int u) {
    if (args.dyn) return unit_take(u);
    if (args.sched) {  // host-balanced list of unit codes
      return u < args.sched_cnt[blockIdx.x] ? args.sched[args.sched_off[blockIdx.x] + u] : n_units;
    }
    const int G = static_cast<int>(gridDim.x);
    return u * G + ((u & 1) ? G - 1 - static_cast<int>(blockIdx.x) : static_cast<int>(blockIdx.x));
  };
  struct Unit {
    int bh, hh, bb, q0, nkv0, nkv1;
  };
  auto decode = [&](int lin) {
    const int HEAD_GROUP = args.head_group;
    Unit w;
    int qp;
    if (args.sched) {
      w.bh = lin / n_pairs;
      qp = lin % n_pairs;
    } else {
      const int grp = lin / (HEAD_GROUP * n_pairs);
      const int gsize = min(HEAD_GROUP, args.BH - grp * HEAD_GROUP);
      const int off = lin - grp * HEAD_GROUP * n_pairs;
      qp = n_pairs - 1 - off / gsize;
      w.bh = grp * HEAD_GROUP + off % gsize;
    }
    w.hh = w.bh % args.H;
    w.bb = w.bh / args.H;
    w.q0 = qp * 2 * BM;
    auto tiles_of = [&](int first) {
      return first >= args.Nq ? 0 : args.causal ? min(nkv_all, (first + BM - 1) / BN + 1) : nkv_all;
    };
    w.nkv0 = tiles_of(w.q0);
    w.nkv1 = tiles_of(w.q0 + BM);
    return w;
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    for (int b = 0; b < QBUF; ++b) {
      mbar_init(&q_full[b], 1);
      mbar_init(&q_empty[b], 1);
    }
    for (int s = 0; s < NS; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int g = 0; g < 2; ++g) {
      mbar_init(&s_full[g], 1);
      // one arrival per softmax warp of the tile; split rows: keys [0, 64)
      // (and every O correction) from both halves, keys [64, 128) from half 1
      mbar_init(&p_full[2 * g], 4 * SPLIT);
      mbar_init(&p_full[2 * g + 1], 4);
      for (int b = 0; b < OBUF; ++b) {
        mbar_init(&o_full[b * 2 + g], 1);
        mbar_init(&o_empty[b * 2 + g], 4 * SPLIT);
      }
    }
    for (int r = 0; r < L::UNIT_R; ++r) {
      mbar_init(&unit_full[r], 1);
      mbar_init(&unit_empty[r], 1 + 8 * SPLIT);  // the MMA warp + the softmax warps
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  griddep_wait();  // Q / K / V from the previous kernel are visible
  griddep_launch_dependents();
  auto s_col = [](int g) { return static_cast<uint32_t>(g * BN); };
  auto o_col = [](int g, int b) { return static_cast<uint32_t>(2 * BN + (b * 2 + g) * D); };

  if (warp >= 4) {
    if constexpr (SPLIT == 2) setmaxnreg_inc<112>();
    else setmaxnreg_inc<D == 64 ? AFG_ATTN_REGS_BIG64 : AFG_ATTN_REGS_BIG>();
    // --------------------------------- softmax / correction / epilogue (per tile)
    // warps 4-7: tile A, 8-11: tile B (split rows: keys [0, 64) of them; 12-15
    // / 16-19 the same rows' keys [64, 128))
    const int g = ((warp - 4) / 4) % 2;
    const int h = SPLIT == 2 ? (warp - 4) / 8 : 0;
    constexpr int SCH = NCH / SPLIT;  // 32-column S chunks per thread
    constexpr int OCH = D / 32 / SPLIT;  // 32-column O chunks per thread
    const int c0 = h * SCH;
    const int oc0 = h * OCH;
    const int w4 = warp % 4;
    const int row = w4 * 32 + lane;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(w4 * 32) << 16);
    const uint32_t s_base = lane_base + s_col(g);
    uint32_t s_phase = 0;  // s_full[g] completions consumed so far (parity)
    float* xmax = reinterpret_cast<float*>(smem + L::XCH_OFF);  // [2][2][2][BM]
    float* xsum = xmax + 2 * 2 * 2 * BM;                          // [2][2][2][BM]
    auto xidx = [&](int par, int hh) { return ((par * 2 + g) * 2 + hh) * BM + row; };
    // the two warps holding the same rows of the tile (split rows only)
    auto pair_sync = [&]() {
      asm volatile("bar.sync %0, 64;" ::"r"(1 + 4 * g + w4) : "memory");
    };
    int ks = 0;  // steps taken (exchange parity)
    // this warp's TMEM writes (P half / O reads) are complete: one arrival per warp
    auto warp_arrive = [&](uint64_t* bar) {
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar);
    };
    for (int u = 0;; ++u) {
      const int lin = unit_of(u);
      if (lin >= n_units) break;
      const Unit w = decode(lin);
      const int nkv_g = g ? w.nkv1 : w.nkv0;
      const int tile_first = w.q0 + g * BM;
      const int qi = tile_first + row;
      const float* brow =
          args.bias ? args.bias + (static_cast<int64_t>(w.bh) * args.Nq + min(qi, args.Nq - 1)) *
                                      args.Nk
                    : nullptr;
      const int ob = u % OBUF;  // this unit's O buffer
      const uint32_t o_base = lane_base + o_col(g, ob);
      float m = -INFINITY;  // running max (scaled log2 units)
      float l = 0.0f;       // this thread's part of the row sum
      for (int j = 0; j < (args.dbg >= 3 ? 0 : nkv_g); ++j, ++ks) {
        mbar_wait(&s_full[g], s_phase);  // also implies PV(g, j-1) completed (in-order MMAs)
        s_phase ^= 1;
        tc_fence_after();
        if (args.dbg == 1) {
          warp_arrive(&p_full[2 * g]);
          if (SPLIT == 1 || h == 1) warp_arrive(&p_full[2 * g + 1]);
          continue;
        }
        // this thread's S columns (all 128, or one half) into registers with
        // one TMEM pass, as column pairs (the f32x2 math takes them directly)
        uint64_t sp[SCH][16];
#pragma unroll
        for (int c = 0; c < SCH; ++c) tmem_ld32x2(s_base + (c0 + c) * 32, sp[c]);
        tmem_wait_ld();
        auto lo = [](uint64_t x) { return __uint_as_float(static_cast<uint32_t>(x)); };
        auto hi = [](uint64_t x) { return __uint_as_float(static_cast<uint32_t>(x >> 32)); };
        auto pk = [](float a, float b) {
          return static_cast<uint64_t>(__float_as_uint(a)) |
                 (static_cast<uint64_t>(__float_as_uint(b)) << 32);
        };
        const int k0 = j * BN + c0 * 32;  // first key of this thread's columns
        const bool need_mask = (args.causal && j * BN + BN - 1 > tile_first) || j * BN + BN > args.Nk;
        // Common path (no additive bias, scale > 0): the max is taken on the raw
        // scores, a causal-diagonal / key-tail tile masks by a per-row count of
        // valid columns (one compare + select per score), and each probability
        // is one FFMA + EX2. With a bias the scores are scaled / biased / masked
        // in place first.
        const bool fast = brow == nullptr && args.scale_log2 > 0.0f;
        float tmax, sc;
        if (fast) {
          if (need_mask) {
            const int lim = min(args.Nk, args.causal ? qi + 1 : args.Nk) - k0;  // valid columns
#pragma unroll
            for (int c = 0; c < SCH; ++c)
#pragma unroll
              for (int e = 0; e < 16; ++e) {
                const int col = c * 32 + 2 * e;
                sp[c][e] = pk(col >= lim ? -INFINITY : lo(sp[c][e]),
                              col + 1 >= lim ? -INFINITY : hi(sp[c][e]));
              }
          }
          float mc[SCH];
#pragma unroll
          for (int c = 0; c < SCH; ++c) {
            mc[c] = fmax3(lo(sp[c][0]), hi(sp[c][0]), lo(sp[c][1]));
            mc[c] = fmax3(mc[c], hi(sp[c][1]), lo(sp[c][2]));
#pragma unroll
            for (int e = 2; e < 15; ++e) mc[c] = fmax3(mc[c], hi(sp[c][e]), lo(sp[c][e + 1]));
            mc[c] = fmaxf(mc[c], hi(sp[c][15]));
          }
          float mm = mc[0];
#pragma unroll
          for (int c = 1; c < SCH; ++c) mm = fmaxf(mm, mc[c]);
          tmax = mm * args.scale_log2;
          sc = args.scale_log2;
        } else {
          tmax = -INFINITY;
#pragma unroll
          for (int c = 0; c < SCH; ++c)
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              float v2[2] = {lo(sp[c][e]), hi(sp[c][e])};
#pragma unroll
              for (int hh = 0; hh < 2; ++hh) {
                const int kj = k0 + c * 32 + 2 * e + hh;
                float v = v2[hh] * args.scale_log2;
                if (brow) v = kj < args.Nk ? fmaf(__ldg(brow + kj), 1.4426950408889634f, v) : v;
                if (need_mask && (kj >= args.Nk || (args.causal && kj > qi))) v = -INFINITY;
                v2[hh] = v;
                tmax = fmaxf(tmax, v);
              }
              sp[c][e] = pk(v2[0], v2[1]);
            }
          sc = 1.0f;
        }
        if constexpr (SPLIT == 2) {  // the row max over both halves
          xmax[xidx(ks & 1, h)] = tmax;
          pair_sync();
          tmax = fmaxf(tmax, xmax[xidx(ks & 1, h ^ 1)]);
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
        // tcgen05.ld/st are warp-collective; rows whose max did not move use 1).
        // Split rows: each half corrects its O columns.
        if (j > 0 && __any_sync(0xffffffffu, upd)) {
#pragma unroll 1
          for (int c = 0; c < OCH; ++c) {
            uint32_t o[32];
            tmem_ld32(o_base + (oc0 + c) * 32, o);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
            tmem_st32(o_base + (oc0 + c) * 32, o);
          }
        }
        m = m_new;
        // half 1's O columns are corrected: the first PV half may start once
        // half 0's P is written too
        if (SPLIT == 2 && h == 1) {
          tmem_wait_st();
          warp_arrive(&p_full[2 * g]);
        }
        // P = exp2(sc * s - base) packed to 16 bit, written over S (P chunk c
        // lands in columns 16c..16c+15; the scores are already in registers)
        const uint64_t sc2 = pk(sc, sc), nb2 = pk(-base, -base);
        uint64_t acc2[2] = {pk(0.0f, 0.0f), pk(0.0f, 0.0f)};  // two chains: half the add latency
#pragma unroll
        for (int c = 0; c < SCH; ++c) {
          uint32_t pkd[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const uint64_t x2 = ffma2(sp[c][e], sc2, nb2);
            float p0, p1;
            // pairs selected by POLY_PAIRS run on the FMA pipe, the rest on MUFU
            if ((POLY_PAIRS >> (e % 8)) & 1) {
              ex2_poly2(x2, p0, p1);
            } else {
              float x0, x1;
              f2split(x2, x0, x1);
              p0 = ex2(x0);
              p1 = ex2(x1);
            }
            acc2[e & 1] = fadd2(acc2[e & 1], pk(p0, p1));
            pkd[e] = pack2(p0, p1, BF16);
          }
          tmem_st16(s_base + (c0 + c) * 16, pkd);
          if (SPLIT == 1 && c == NCH / 2 - 1) {  // keys [0, 64) of P written: the PV MMA can start
            tmem_wait_st();
            warp_arrive(&p_full[2 * g]);
          }
        }
        float a0, a1, a2, a3;
        f2split(acc2[0], a0, a1);
        f2split(acc2[1], a2, a3);
        tmem_wait_st();
        l = l * alpha + ((a0 + a1) + (a2 + a3));
        warp_arrive(&p_full[2 * g + (SPLIT == 2 && h == 0 ? 0 : 1)]);
      }
      // ---- epilogue: O / l -> global, one 32-column chunk at a time; O_g is
      // released (o_empty) right after the last chunk's TMEM load, so the next
      // unit's first PV(g) does not wait for the global stores.
      if constexpr (SPLIT == 2) {  // the row sum over both halves
        xsum[xidx(u & 1, h)] = l;
        pair_sync();
        l += xsum[xidx(u & 1, h ^ 1)];
      }
      mbar_wait(&o_full[ob * 2 + g], (u / OBUF) & 1);
      tc_fence_after();
      const float inv_l = l > 0.0f ? 1.0f / l : 0.0f;
      const bool valid = qi < args.Nq && nkv_g > 0;
      const int64_t base_idx = static_cast<int64_t>(w.bb) * args.o_bs +
                               static_cast<int64_t>(w.hh) * args.o_hs +
                               static_cast<int64_t>(qi) * args.o_ss;
#pragma unroll 1
      for (int cc = 0; cc < OCH; ++cc) {
        const int c = oc0 + cc;
        uint32_t o[32];
        if (nkv_g > 0) {
          tmem_ld32(o_base + c * 32, o);
          tmem_wait_ld();
        }
        if (cc == OCH - 1) warp_arrive(&o_empty[ob * 2 + g]);
        if (!valid) continue;
        if (args.o_dtype == AFG_F32) {
          float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(args.o) + base_idx + c * 32);
#pragma unroll
          for (int v = 0; v < 8; ++v)
            dst[v] = make_float4(__uint_as_float(o[4 * v]) * inv_l, __uint_as_float(o[4 * v + 1]) * inv_l,
                                 __uint_as_float(o[4 * v + 2]) * inv_l,
                                 __uint_as_float(o[4 * v + 3]) * inv_l);
        } else {
          const bool ob = args.o_dtype == AFG_BF16;
          uint16_t* dst = reinterpret_cast<uint16_t*>(args.o) + base_idx + c * 32;
          uint32_t wv[16];
#pragma unroll
          for (int v = 0; v < 16; ++v)
            wv[v] = pack2(__uint_as_float(o[2 * v]) * inv_l, __uint_as_float(o[2 * v + 1]) * inv_l, ob);
          if (args.o_st32) {
            // 32-byte stores: each thread writes whole sectors of its row (the
            // rows of a warp are D * 2 bytes apart, so stores do not coalesce)
#pragma unroll
            for (int v = 0; v < 2; ++v)
              asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst + 16 * v),
                           "r"(wv[8 * v]), "r"(wv[8 * v + 1]), "r"(wv[8 * v + 2]), "r"(wv[8 * v + 3]),
                           "r"(wv[8 * v + 4]), "r"(wv[8 * v + 5]), "r"(wv[8 * v + 6]), "r"(wv[8 * v + 7])
                           : "memory");
          } else {
            uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
            for (int v = 0; v < 4; ++v) d4[v] = make_uint4(wv[4 * v], wv[4 * v + 1], wv[4 * v + 2], wv[4 * v + 3]);
          }
        }
      }
    }
  } else {
    if constexpr (SPLIT == 2) setmaxnreg_dec<32>();
    else setmaxnreg_dec<D == 64 ? AFG_ATTN_REGS_SMALL64 : AFG_ATTN_REGS_SMALL>();
    if (warp == 0) {
      // ------------------------------------------------------------- TMA --
      if (lane == 0) {
        int n = 0;  // K/V ring item counter across units (item 2j = K(j), 2j+1 = V(j))
        unsigned int* queue = args.dyn ? g_attn_queue[args.dyn - 1] : nullptr;
        for (int u = 0;; ++u) {
          const int qb = u % QBUF;
          // the S MMAs of the unit that last used this Q buffer are done
          mbar_wait(&q_empty[qb], ((u / QBUF) & 1) ^ 1);
          int lin;
          if (queue) {
            // take the next unit only now that its Q tiles can load: a CTA
            // never holds more than the unit it is about to start
            const int slot = u % L::UNIT_R;
            mbar_wait(&unit_empty[slot], ((u / L::UNIT_R) & 1) ^ 1);
            lin = min(static_cast<int>(atomicAdd(&queue[0], 1u)), n_units);
            unit_ring[slot] = lin;
            mbar_arrive(&unit_full[slot]);
          } else {
            lin = unit_of(u);
          }
          if (lin >= n_units) break;
          const Unit w = decode(lin);
          mbar_arrive_expect_tx(&q_full[qb], 2 * L::TILE);
          for (int g = 0; g < 2; ++g)
            for (int a = 0; a < DB; ++a)
              tma_load_4d(smem + qb * L::QBUF_BYTES + (g ? L::QB_OFF : L::QA_OFF) + a * (BM * 128),
                          &tmQ, &q_full[qb],
                          a * 64, w.q0 + g * BM, w.hh, w.bb);
          const int items = 2 * max(w.nkv0, w.nkv1);
          for (int it = 0; it < items; ++it, ++n) {
            const int st = n % NS;
            mbar_wait(&kv_empty[st], ((n / NS) & 1) ^ 1);
            mbar_arrive_expect_tx(&kv_full[st], L::TILE);
            const CUtensorMap* tm = (it & 1) ? &tmV : &tmK;
            for (int a = 0; a < DB; ++a)
              tma_load_4d(smem + L::RING_OFF + st * L::TILE + a * (BN * 128), tm, &kv_full[st],
                          a * 64, (it >> 1) * BN, w.hh, w.bb);
          }
        }
      }
    } else if (warp == 1) {
      // ------------------------------------------------------------- MMA --
      // The whole warp runs the issue loop (waits and descriptor arithmetic
      // stay warp-uniform, in uniform registers) and one elected lane issues:
      // a 128x128x16 MMA takes 64 tensor cycles, so per-MMA issue work must be
      // a handful of instructions (descriptors are base + immediate offsets).
      const bool leader = elect_one();
      constexpr uint32_t idesc_s = idesc_f16(BM, BN, BF16 ? 1u : 0u, 0u, 0u);
      constexpr uint32_t idesc_o = idesc_f16(BM, D, BF16 ? 1u : 0u, 0u, 1u);
      const uint64_t q_desc0 = desc_kmajor_sw128(smem_u32(smem + L::QA_OFF));
      const uint64_t k_desc0 = desc_kmajor_sw128(smem_u32(smem + L::RING_OFF));
      const uint64_t v_desc0 = desc_mnmajor_sw128(smem_u32(smem + L::RING_OFF), BN * 128);
      constexpr uint64_t QB_STEP = (L::QB_OFF - L::QA_OFF) >> 4;  // descriptor units (16 B)
      constexpr uint64_t SLOT_STEP = L::TILE >> 4;
      int nb = 0;                  // ring item index of this unit's K(0)
      uint32_t p_phase[2] = {0, 0};  // per tile; both halves complete once per step
      auto wait_item = [&](int n) {
        mbar_wait(&kv_full[n % NS], (n / NS) & 1);
        tc_fence_after();
      };
      int qb = 0;  // Q buffer of the current unit
      int ob = 0;  // O buffers of the current unit
      auto issue_s = [&](int g, int j) {
        const uint64_t qd =
            q_desc0 + (g ? QB_STEP : 0) + static_cast<uint64_t>(qb) * (L::QBUF_BYTES >> 4);
        const uint64_t kd = k_desc0 + static_cast<uint64_t>((nb + 2 * j) % NS) * SLOT_STEP;
        if (args.dbg != 2) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint64_t off =
                static_cast<uint64_t>(((kk / 4) * (BM * 128) + (kk % 4) * 32) >> 4);
            mma_f16_ss_if(leader, tmem + s_col(g), qd + off, kd + off, idesc_s, kk > 0 ? 1u : 0u);
          }
        }
        mma_commit_if(leader, &s_full[g]);
      };
      // O_g += P V over keys [64 h, 64 h + 64) (P half h)
      auto issue_pv_half = [&](int g, int j, int h) {
        const uint64_t vd = v_desc0 + static_cast<uint64_t>((nb + 2 * j + 1) % NS) * SLOT_STEP;
        if (args.dbg == 2) return;
#pragma unroll
        for (int k2 = 0; k2 < BN / 32; ++k2) {
          const int kk = h * (BN / 32) + k2;
          mma_f16_ts_if(leader, tmem + o_col(g, ob), tmem + s_col(g) + kk * 8,
                        vd + static_cast<uint64_t>((kk * 16 * 128) >> 4), idesc_o,
                        (j > 0 || kk > 0) ? 1u : 0u);
        }
      };
      for (int u = 0;; ++u) {
        const int lin = unit_of(u);
        if (lin >= n_units) break;
        const Unit w = decode(lin);
        const int nkv_max = max(w.nkv0, w.nkv1);
        qb = u % QBUF;
        ob = u % OBUF;
        mbar_wait(&q_full[qb], (u / QBUF) & 1);
        wait_item(nb);
        if (w.nkv0 > 0) issue_s(0, 0);
        if (w.nkv1 > 0) issue_s(1, 0);
        if (nkv_max <= 1) mma_commit_if(leader, &q_empty[qb]);  // last S of the unit issued
        mma_commit_if(leader, &kv_empty[nb % NS]);
        for (int j = 0; j < nkv_max; ++j) {
          const int jn = j + 1;
          bool k_next_ready = false;
          wait_item(nb + 2 * j + 1);
#pragma unroll
          for (int g = 0; g < 2; ++g) {
            const int nkv_g = g ? w.nkv1 : w.nkv0;
            if (j < nkv_g) {
              // the unit that last used this O buffer has read it out
              if (j == 0) mbar_wait(&o_empty[ob * 2 + g], ((u / OBUF) & 1) ^ 1);
              // PV in two halves: the first 64 keys as soon as their P is written
              if (args.dbg < 3) mbar_wait(&p_full[2 * g], p_phase[g]);
              tc_fence_after();
              issue_pv_half(g, j, 0);
              if (args.dbg < 3) mbar_wait(&p_full[2 * g + 1], p_phase[g]);
              p_phase[g] ^= 1;
              tc_fence_after();
              issue_pv_half(g, j, 1);
              if (jn < nkv_g) {
                if (!k_next_ready) {
                  wait_item(nb + 2 * jn);
                  k_next_ready = true;
                }
                issue_s(g, jn);  // runs after PV(g, j) on the tensor pipe: P(j) consumed first
              } else {
                mma_commit_if(leader, &o_full[ob * 2 + g]);  // O_g of this unit complete
              }
            }
          }
          if (jn == nkv_max - 1) mma_commit_if(leader, &q_empty[qb]);  // last S of the unit issued
          mma_commit_if(leader, &kv_empty[(nb + 2 * j + 1) % NS]);
          if (k_next_ready) mma_commit_if(leader, &kv_empty[(nb + 2 * jn) % NS]);
        }
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          if ((g ? w.nkv1 : w.nkv0) == 0) {  // empty tile: keep its O phases in step
            mbar_wait(&o_empty[ob * 2 + g], ((u / OBUF) & 1) ^ 1);
            mma_commit_if(leader, &o_full[ob * 2 + g]);
          }
        }
        nb += 2 * nkv_max;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<TMEM_COLS>(tmem);
  }
  if (args.dyn && threadIdx.x == 0) {
    unsigned int* queue = g_attn_queue[args.dyn - 1];
    __threadfence();
    if (atomicAdd(&queue[1], 1u) == gridDim.x - 1) {  // last CTA out: reset for the next launch
      atomicExch(&queue[0], 0u);
      atomicExch(&queue[1], 0u);
      __threadfence();
    }
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

// Unit schedule for the persistent grid (built on the host once per shape and
// device, kept in device memory): heads are taken in groups whose K / V fit
// comfortably in L2 (co-resident CTAs then share every K / V tile), and
// inside a group the units are dealt heaviest first to the CTA with the least
// accumulated work (greedy LPT, cost = KV tiles of the unit + one tile of
// per-unit overhead). Causal units differ 10x in cost, so the static snake
// order either broke the grouping (all 128 heads at once: 2-5x the K / V DRAM
// traffic) or the balance (groups of 16: the slowest CTA 19% over the mean);
// LPT per group keeps both.
struct Sched {
  int* dev = nullptr;  // [units] codes | [grid] offsets | [grid] counts
  int grid = 0, units = 0;
};

const Sched& attn_schedule(int BH, int Nq, int Nk, int D, int causal, int grid) {
  static std::mutex mu;
  static std::map<std::vector<int>, Sched> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const std::vector<int> key = {dev, BH, Nq, Nk, D, causal, grid};
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  const int n_pairs = (Nq + 2 * BM - 1) / (2 * BM);
  const int nkv_all = (Nk + BN - 1) / BN;
  auto tiles = [&](int first) {
    return first >= Nq ? 0 : causal ? std::min(nkv_all, (first + BM - 1) / BN + 1) : nkv_all;
  };
  // heads per group: K + V of the group <= ~40 MB of L2
  const int64_t kv_head = 2ll * Nk * D * 2;
  const int hg = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(BH, (40ll << 20) / kv_head)));
  std::vector<std::vector<int>> lists(grid);
  std::vector<double> load(grid, 0.0);
  for (int g0 = 0; g0 < BH; g0 += hg) {
    std::vector<std::pair<double, int>> items;
    for (int bh = g0; bh < std::min(BH, g0 + hg); ++bh)
      for (int qp = 0; qp < n_pairs; ++qp)
        items.push_back({tiles(qp * 2 * BM) + tiles(qp * 2 * BM + BM) + 1.0, bh * n_pairs + qp});
    std::stable_sort(items.begin(), items.end(),
                     [](const auto& x, const auto& y) { return x.first > y.first; });
    using E = std::pair<double, int>;
    std::priority_queue<E, std::vector<E>, std::greater<E>> heap;
    for (int c = 0; c < grid; ++c) heap.push({load[c], c});
    for (const auto& [cost, code] : items) {
      auto [l, c] = heap.top();
      heap.pop();
      lists[c].push_back(code);
      load[c] = l + cost;
      heap.push({load[c], c});
    }
  }
  std::vector<int> host;
  std::vector<int> off(grid), cnt(grid);
  for (int c = 0; c < grid; ++c) {
    off[c] = static_cast<int>(host.size());
    cnt[c] = static_cast<int>(lists[c].size());
    host.insert(host.end(), lists[c].begin(), lists[c].end());
  }
  Sched sc;
  sc.grid = grid;
  sc.units = static_cast<int>(host.size());
  host.insert(host.end(), off.begin(), off.end());
  host.insert(host.end(), cnt.begin(), cnt.end());
  if (cudaMalloc(&sc.dev, host.size() * sizeof(int)) == cudaSuccess &&
      cudaMemcpy(sc.dev, host.data(), host.size() * sizeof(int), cudaMemcpyHostToDevice) ==
          cudaSuccess)
    return cache[key] = sc;
  cudaGetLastError();
  return cache[key] = Sched{};
}

template <int D, bool BF16>
cudaError_t launch_tc(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                      AttnArgs a, cudaStream_t s) {
  auto kern = attn_fwd_kernel<D, BF16>;
  constexpr int smem = AttnSmem<D>::TOTAL;
  static std::atomic<uint64_t> configured{0};
  if (cudaError_t e = ensure_smem_optin(configured, kern, smem); e != cudaSuccess) return e;
  const int units = a.BH * ((a.Nq + 2 * BM - 1) / (2 * BM));
  const unsigned grid = static_cast<unsigned>(std::min(units, num_sms()));  // persistent
  static const int sched_env = [] {  // AFG_ATTN_SCHED=1: the LPT table (measured slower, §7b)
    const char* e = getenv("AFG_ATTN_SCHED");
    return e ? atoi(e) : 0;
  }();
  a.sched = a.sched_off = a.sched_cnt = nullptr;
  if (a.dyn) a.dyn = 1 + stream_slot(s, 1, ATTN_SLOTS);  // 0: the static walk
  if (!a.dyn && sched_env) {
    const Sched& sc = attn_schedule(a.BH, a.Nq, a.Nk, D, a.causal, static_cast<int>(grid));
    if (sc.dev) {
      a.sched = sc.dev;
      a.sched_off = sc.dev + sc.units;
      a.sched_cnt = sc.dev + sc.units + sc.grid;
    }
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(ATTN_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // see gemm_tc.cu
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tq, tk, tv, a);
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
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
  if (BH > 65535 || Nq >= (1 << 24) || Nk >= (1 << 30))
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
    uint32_t box[4] = {64, 128, 1, 1};
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
    a.o_st32 = (reinterpret_cast<uintptr_t>(o) % 32 == 0) && so.s % 16 == 0 && so.h % 16 == 0 &&
               so.b % 16 == 0;
    static const int dbg = [] {
      const char* e = getenv("AFG_ATTN_DEBUG");
      return e ? atoi(e) : 0;
    }();
    a.dbg = dbg;
    // Non-causal units are equal: group heads by 16 so co-resident CTAs share
    // K/V in L2. Causal: one group = a globally heaviest-first order (the K/V
    // of all heads ~ fits L2 at the BASELINE shape), which the snake walk
    // turns into balanced per-CTA totals with the lightest units last.
    static const int hg_env = [] {
      const char* e = getenv("AFG_ATTN_HEAD_GROUP");
      return e ? atoi(e) : 0;
    }();
    // AFG_ATTN_DYN=0: the static snake walk. The dynamic queue balances the
    // CTAs by their actual unit times, so causal units can stay grouped by
    // heads whose K / V fit in L2 without unbalancing the tail.
    static const int dyn_env = [] {
      const char* e = getenv("AFG_ATTN_DYN");
      return e ? atoi(e) : 1;
    }();
    a.dyn = dyn_env;
    // Measured at B8H16S2048D128 causal: 171.6 us static / all heads, 157-158
    // us dynamic with groups of 16 or 32 heads (K/V DRAM reads 513 -> 202 MB),
    // 164 us with groups of 8.
    a.head_group = hg_env > 0 ? hg_env : (a.dyn || !causal ? 16 : static_cast<int>(BH));
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
