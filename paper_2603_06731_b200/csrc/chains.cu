// chains.cu - K4/K5/K6: the memory-bound fused chains.
//
// The reference lowers softmax to four nests with global intermediates
// (.rowmax / .exp / .rowsum, frontend.cpp:564-625) and its fusion pass leaves
// them as four nests (probe 3). Here each chain is ONE pass
// over HBM: 128-bit vectorised coalesced loads (the reference's
// maxVectorWidthElems = 8 x 16-bit, ir.h:213), the row kept in registers,
// warp-shuffle reductions, one 128-bit store per chunk.
//
//   softmax_lastdim     : y = exp(x - max) / sum exp(x - max)   (oracles.cpp:175-190)
//   layernorm_residual  : y = (s - mean) * rsqrt(var + eps) * gamma + beta,
//                         s = x + residual, biased variance, fp32 statistics
//   elementwise / reduce / convert / transpose / fill: graph-executor tails
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <type_traits>

#include "afg_internal.h"
#include "epilogue.cuh"
#include "sm100.cuh"

namespace afg {
namespace {

// ------------------------------------------------------------ utilities --

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <typename T>
struct Vec {  // one 16-byte chunk
  static constexpr int N = 16 / sizeof(T);
  union {
    uint4 u;
    T e[N];
  };
};

__device__ __forceinline__ float ld_any(const void* p, int64_t i, int dt) {
  switch (dt) {
    case AFG_F32: return reinterpret_cast<const float*>(p)[i];
    case AFG_F16: return __half2float(reinterpret_cast<const __half*>(p)[i]);
    default: return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]);
  }
}
__device__ __forceinline__ void st_any(void* p, int64_t i, int dt, float v) {
  switch (dt) {
    case AFG_F32: reinterpret_cast<float*>(p)[i] = v; break;
    case AFG_F16: reinterpret_cast<__half*>(p)[i] = __float2half_rn(v); break;
    default: reinterpret_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(v); break;
  }
}

__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream(void* p, uint4 v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// -------------------------------------------------------------- softmax --

// One warp per row; each lane holds CH 16-byte chunks (chunk c = lane + 32 i).
template <typename TI, typename TO, int CH>
__global__ void __launch_bounds__(256) softmax_warp_kernel(const TI* __restrict__ x,
                                                           TO* __restrict__ y, int64_t rows,
                                                           int cols) {
  constexpr int E = Vec<TI>::N;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (row >= rows) return;
  const int nchunks = cols / E;
  const TI* xr = x + row * cols;
  float v[CH][E];
  float m = -INFINITY;
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    const int c = lane + 32 * i;
    if (c < nchunks) {
      Vec<TI> t;
      t.u = ld_stream(xr + c * E);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        v[i][e] = OutCvt<TI>::from(t.e[e]);
        m = fmaxf(m, v[i][e]);
      }
    }
  }
  m = warp_max(m);
  float s = 0.0f;
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    const int c = lane + 32 * i;
    if (c < nchunks) {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        v[i][e] = __expf(v[i][e] - m);
        s += v[i][e];
      }
    }
  }
  s = warp_sum(s);
  const float inv = 1.0f / s;
  TO* yr = y + row * cols;
  constexpr int EO = Vec<TO>::N;
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    const int c = lane + 32 * i;
    if (c < nchunks) {
      if constexpr (EO == E) {
        Vec<TO> o;
#pragma unroll
        for (int e = 0; e < E; ++e) o.e[e] = OutCvt<TO>::to(v[i][e] * inv);
        st_stream(yr + c * E, o.u);
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) yr[c * E + e] = OutCvt<TO>::to(v[i][e] * inv);
      }
    }
  }
}

// General fallback: one block per row, three sweeps (max, sum, write).
template <typename TI, typename TO>
__global__ void __launch_bounds__(256) softmax_block_kernel(const TI* __restrict__ x,
                                                            TO* __restrict__ y, int cols) {
  __shared__ float red[32];
  const int64_t row = blockIdx.x;
  const TI* xr = x + row * cols;
  TO* yr = y + row * cols;
  float m = -INFINITY;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) m = fmaxf(m, OutCvt<TI>::from(xr[c]));
  m = warp_max(m);
  if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : -INFINITY;
    t = warp_max(t);
    if (threadIdx.x == 0) red[31] = t;
  }
  __syncthreads();
  m = red[31];
  __syncthreads();
  float s = 0.0f;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) s += __expf(OutCvt<TI>::from(xr[c]) - m);
  s = warp_sum(s);
  if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0f;
    t = warp_sum(t);
    if (threadIdx.x == 0) red[31] = t;
  }
  __syncthreads();
  const float inv = 1.0f / red[31];
  for (int c = threadIdx.x; c < cols; c += blockDim.x)
    yr[c] = OutCvt<TO>::to(__expf(OutCvt<TI>::from(xr[c]) - m) * inv);
}

template <typename TI, typename TO>
cudaError_t softmax_launch(const void* x, void* y, int64_t rows, int64_t cols, cudaStream_t s);

template <typename TI, typename TO>
cudaError_t softmax_launch_direct(const void* x, void* y, int64_t rows, int64_t cols,
                                  cudaStream_t s) {
  constexpr int E = Vec<TI>::N;
  const bool vec_ok = (cols % E == 0) && (cols % Vec<TO>::N == 0) &&
                      ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) == 0;
  const int64_t nchunks = cols / E;
  const TI* xi = reinterpret_cast<const TI*>(x);
  TO* yo = reinterpret_cast<TO*>(y);
  const unsigned grid = static_cast<unsigned>((rows + 7) / 8);
  if (vec_ok && nchunks <= 32 * 16 && rows / 8 < (1ll << 31)) {
    if (nchunks <= 32)
      softmax_warp_kernel<TI, TO, 1><<<grid, 256, 0, s>>>(xi, yo, rows, (int)cols);
    else if (nchunks <= 64)
      softmax_warp_kernel<TI, TO, 2><<<grid, 256, 0, s>>>(xi, yo, rows, (int)cols);
    else if (nchunks <= 128)
      softmax_warp_kernel<TI, TO, 4><<<grid, 256, 0, s>>>(xi, yo, rows, (int)cols);
    else if (nchunks <= 256)
      softmax_warp_kernel<TI, TO, 8><<<grid, 256, 0, s>>>(xi, yo, rows, (int)cols);
    else
      softmax_warp_kernel<TI, TO, 16><<<grid, 256, 0, s>>>(xi, yo, rows, (int)cols);
  } else {
    if (rows >= (1ll << 31)) return cudaErrorInvalidValue;
    softmax_block_kernel<TI, TO><<<static_cast<unsigned>(rows), 256, 0, s>>>(xi, yo, (int)cols);
  }
  count_launch();
  return cudaGetLastError();
}

// --------------------------------------------------- TMA-streamed chains --
// Persistent CTA per SM: warp 8 (one lane) streams whole rows global -> smem
// with 1-D bulk copies into an NS-deep ring (mbarrier complete_tx); warps 0-7
// each reduce every 8th row out of shared memory and write the result with
// coalesced 16-byte stores. In-flight bytes live in shared memory (~160 KB
// per SM), not in registers, so HBM stays saturated.
// 15 consumer warps + 1 producer (128 registers per thread). The chains are
// bound by the bytes in flight per SM (layernorm, measured: a 48 / 96 / 192
// KB ring gives 0.36 / 0.75 / 0.78 of HBM); 12 consumer warps with a 216 KB
// ring (36 slots) measured worse (0.75 layernorm, 0.85 softmax): the consumer
// parallelism matters as much.
constexpr int STREAM_WARPS = 15;
constexpr int STREAM_SMEM = 160 * 1024;
constexpr int STREAM_SMEM_LN = 192 * 1024;  // layernorm: 2 rows x (x, residual) per slot

__device__ __forceinline__ float ex2f_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// max over the 8 16-bit values of a chunk with packed (x2) compares
template <typename T>
__device__ __forceinline__ float chunk_max(const Vec<T>& t) {
  if constexpr (sizeof(T) == 2) {
    using T2 = typename std::conditional<std::is_same<T, __half>::value, __half2, __nv_bfloat162>::type;
    const T2* p = reinterpret_cast<const T2*>(&t.u);
    T2 m = __hmax2(__hmax2(p[0], p[1]), __hmax2(p[2], p[3]));
    return fmaxf(OutCvt<T>::from(m.x), OutCvt<T>::from(m.y));
  } else {
    float m = -INFINITY;
#pragma unroll
    for (int e = 0; e < Vec<T>::N; ++e) m = fmaxf(m, OutCvt<T>::from(t.e[e]));
    return m;
  }
}

// 16-bit pair <-> packed f32x2 (the low element in the low half)
template <typename T>
__device__ __forceinline__ uint64_t unpack_pair(uint32_t w) {
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    return sm100::f2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
  } else {
    const __half2 h = *reinterpret_cast<const __half2*>(&w);
    const float2 f = __half22float2(h);
    return sm100::f2(f.x, f.y);
  }
}
template <typename T>
__device__ __forceinline__ uint32_t pack_pair(uint64_t v) {
  float a, b;
  sm100::f2split(v, a, b);
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
  } else {
    const __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
  }
}

// Tail balancing: the last `pool` rows are not assigned to a CTA; producers
// claim them slot by slot from a global counter pair owned by the stream
// (stream_slot): [0] = rows claimed, [1] = producer exits; the last producer
// out resets both, the next launch touches them after griddepcontrol.wait.
// The per-SM DRAM rates differ, so a static split ends with the slowest SM
// alone (layernorm: SM active 45.4 k cycles on average, 48.7 k at most).
constexpr int ROW_SLOTS = 64;
__device__ unsigned int g_row_pool[ROW_SLOTS][2];

// What a ring slot holds: rows [row, row + n) (n > 0), nothing (n = 0: skip
// it), or the end of the stream for the consumer warp that reads it (n < 0).
struct SlotDesc {
  int64_t row;
  int n, pad;
};

#ifndef AFG_LN_ROWS  // layernorm rows per ring slot / per consumer warp step (rows <= 1024)
#define AFG_LN_ROWS 2
#endif

template <typename TI, typename TO, int MODE, int CH>  // MODE 0 softmax, 1 layernorm
__global__ void __launch_bounds__((STREAM_WARPS + 1) * 32, 1)
    stream_rows_kernel(const TI* __restrict__ x, const TI* __restrict__ res,
                       const float* __restrict__ gamma, const float* __restrict__ beta,
                       TO* __restrict__ y, TO* __restrict__ sum_out, int64_t rows, int cols,
                       float eps, int ns, int slot_bytes, int grp, unsigned int* pool_ctr,
                       int64_t pool) {
  using namespace sm100;
  constexpr int E = Vec<TI>::N;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) &
                                             ~uintptr_t(127));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(ns) * slot_bytes);
  uint64_t* empty = full + ns;
  SlotDesc* desc = reinterpret_cast<SlotDesc*>(empty + ns);
  float* gb = reinterpret_cast<float*>(desc + ns + 2);  // layernorm: gamma | beta
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t srows = rows - pool;  // statically split rows
  const int64_t per = (srows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * per;
  const int64_t nr = max(static_cast<int64_t>(0), min(per, srows - r0));
  // a ring slot holds `grp` consecutive rows (of x, then of the residual):
  // fewer, larger bulk copies (the per-copy cost bounds 1.5 KB rows)
  const int64_t nslots = (nr + grp - 1) / grp;
  const uint32_t row_bytes = static_cast<uint32_t>(cols) * sizeof(TI);
  if (threadIdx.x == 0) {
    for (int i = 0; i < ns; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    desc[ns].row = -1;  // producer control words (see the producer)
    desc[ns].n = 0;
    desc[ns + 1].row = -1;
    fence_barrier_init();
  }
  __syncthreads();  // barriers initialised: the producer starts streaming at once
  griddep_wait();   // the previous kernel's output (our input) is visible
  griddep_launch_dependents();
  if constexpr (MODE == 1) {
    if (warp < STREAM_WARPS) {  // gamma / beta staged by the consumers meanwhile
      for (int c = threadIdx.x; c < cols; c += STREAM_WARPS * 32) {
        gb[c] = gamma[c];
        gb[cols + c] = beta[c];
      }
      asm volatile("bar.sync 1, %0;" ::"n"(STREAM_WARPS * 32) : "memory");
    }
  }
  if (warp == STREAM_WARPS) {
    // Every ring slot belongs to one producer lane (slots lane, lane + 32,
    // lane + 64 < ns), which issues that slot's uses k = 0, 1, ... in order,
    // each after the consumers released use k-1 (empty parity (k & 1) ^ 1).
    // Lanes run independently: a slot is refilled the moment it is released.
    // (Issuing in warp-wide lock-step batches of `ns` rows drained the whole
    // ring before each refill -- on the 151 MB layernorm the DRAM read rate
    // stayed at ~3.6 TB/s.) One lane owning a slot means no wait can see a
    // phase two laps stale. Stream index i = k * ns + slot: the CTA's static
    // rows first, then rows claimed from the pool; the first index a lane
    // cannot fill becomes a skip. With B = the largest such index in the
    // warp, every index <= B is then data or a skip and (B, B + STREAM_WARPS]
    // -- one index per consumer warp -- holds the end marker.
    int64_t k = 0;
    int sj = 0;  // this lane's slot = lane + 32 sj
    auto advance_p = [&]() {
      if (lane + 32 * (++sj) >= ns) {
        sj = 0;
        ++k;
      }
    };
    auto fill = [&](int64_t i, int64_t row, int n) {
      const int slot = static_cast<int>(i - k * ns);
      mbar_wait(&empty[slot], static_cast<uint32_t>(k & 1) ^ 1u);
      desc[slot].row = row;
      desc[slot].n = n;
      if (n > 0) {
        const uint32_t bytes = static_cast<uint32_t>(n) * row_bytes;
        uint8_t* dst = smem + static_cast<size_t>(slot) * slot_bytes;
        mbar_arrive_expect_tx(&full[slot], MODE == 1 && res ? 2 * bytes : bytes);
        bulk_load(dst, x + row * cols, bytes, &full[slot]);
        if (MODE == 1 && res) bulk_load(dst + grp * row_bytes, res + row * cols, bytes, &full[slot]);
      } else {
        mbar_arrive(&full[slot]);
      }
    };
    // ctl[0].row: the highest index any lane has started to fill; ctl[1].row:
    // the highest exhaustion index; ctl[0].n: lanes exhausted. An exhausted
    // lane fills skips only below the highest started index (every index a
    // blocked fill transitively waits for lies below it), and places the end
    // markers once all lanes are exhausted -- no warp-wide barrier, which
    // could wait on a lane whose fill waits on a skip of the waiting lane.
    SlotDesc* ctl = desc + ns;
    auto* prog = reinterpret_cast<long long*>(&ctl[0].row);
    auto* bexh = reinterpret_cast<long long*>(&ctl[1].row);
    const bool use_pool = pool_ctr != nullptr && pool > 0;
    if (!use_pool) {
      // static rows only: the consumers know the count, no markers needed
      for (;;) {
        const int64_t i = k * ns + lane + 32 * sj;
        if (lane >= ns || i >= nslots) break;
        fill(i, r0 + i * grp, static_cast<int>(min(static_cast<int64_t>(grp), nr - i * grp)));
        advance_p();
      }
      return;
    }
    if (lane < ns) {
      // the pool claim for a lane's next dynamic fill is issued right after
      // the previous fill, so its round trip overlaps the wait for the slot
      unsigned int claim = 0;
      bool claimed = false;
      // a claim past the pool end is answered by a plain load once the pool is
      // drained: every lane's final (failing) claim would otherwise queue on
      // the one counter behind the real ones
      auto claim_rows = [&]() -> unsigned int {
        const unsigned int seen = *reinterpret_cast<volatile unsigned int*>(&pool_ctr[0]);
        if (seen >= static_cast<unsigned int>(pool)) return seen;
        return atomicAdd(&pool_ctr[0], static_cast<unsigned int>(grp));
      };
      for (;;) {
        const int64_t i = k * ns + lane + 32 * sj;
        int64_t row = 0;
        int n = 0;
        if (i < nslots) {
          row = r0 + i * grp;
          n = static_cast<int>(min(static_cast<int64_t>(grp), nr - i * grp));
        } else if (use_pool) {
          if (!claimed) claim = claim_rows();
          claimed = false;
          row = srows + static_cast<int64_t>(claim);
          n = static_cast<int>(max(static_cast<int64_t>(0), min(static_cast<int64_t>(grp), rows - row)));
        }
        atomicMax(prog, static_cast<long long>(i));
        fill(i, row, n);
        advance_p();
        if (n == 0) {
          atomicMax(bexh, static_cast<long long>(i));
          __threadfence_block();
          atomicAdd(&ctl[0].n, 1);
          break;
        }
        if (use_pool && k * ns + lane + 32 * sj >= nslots) {
          claim = claim_rows();
          claimed = true;
        }
      }
      const int lanes = ns < 32 ? ns : 32;
      for (;;) {
        const int64_t i = k * ns + lane + 32 * sj;
        if (*reinterpret_cast<volatile int*>(&ctl[0].n) == lanes) break;
        if (i < *reinterpret_cast<volatile long long*>(prog)) {
          fill(i, 0, 0);
          advance_p();
        } else {
          __nanosleep(64);
        }
      }
      __threadfence_block();
      const int64_t bmax = *reinterpret_cast<volatile long long*>(bexh);
      for (;;) {
        const int64_t i = k * ns + lane + 32 * sj;
        if (i > bmax + STREAM_WARPS) break;
        fill(i, 0, i <= bmax ? 0 : -1);
        advance_p();
      }
    }
    if (pool_ctr != nullptr && lane == 0) {
      __threadfence();
      if (atomicAdd(&pool_ctr[1], 1u) == gridDim.x - 1) {  // last producer out: reset
        atomicExch(&pool_ctr[0], 0u);
        atomicExch(&pool_ctr[1], 0u);
        __threadfence();
      }
    }
    return;
  }
  const int nchunks = cols / E;
  // consumer ring position (slot, phase) advanced by STREAM_WARPS per row /
  // slot: ns is a multiple of STREAM_WARPS, so it wraps exactly
  int cslot = warp;
  uint32_t cph = 0;
  int64_t ci = warp;  // stream index of the slot this warp reads next
  // without a pool the stream is the CTA's static slots: stop after them
  const int64_t cend = pool_ctr != nullptr && pool > 0 ? INT64_MAX : nslots;
  auto advance = [&]() {
    ci += STREAM_WARPS;
    cslot += STREAM_WARPS;
    if (cslot >= ns) {
      cslot -= ns;
      cph ^= 1;
    }
  };
  const float inv_cols = 1.0f / static_cast<float>(cols);
  if constexpr (MODE == 0) {
    for (;; advance()) {
      if (ci >= cend) break;
      const int slot = cslot;
      mbar_wait(&full[slot], cph);
      const int dn = reinterpret_cast<volatile SlotDesc*>(desc)[slot].n;
      if (dn < 0) break;  // end of this warp's stream
      if (dn == 0) {      // skip
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        continue;
      }
      const uint32_t sx = smem_u32(smem + static_cast<size_t>(slot) * slot_bytes);
      const int64_t row = reinterpret_cast<volatile SlotDesc*>(desc)[slot].row;
      TO* yr = y + row * cols;
      Vec<TI> raw[CH];
        float mx = -INFINITY;
#pragma unroll
        for (int k = 0; k < CH; ++k) {
          const int c = lane + 32 * k;
          if (c < nchunks) {
            raw[k].u = ld_shared_v4(sx + c * 16);
            mx = fmaxf(mx, chunk_max<TI>(raw[k]));
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);  // row consumed: the slot can be refilled
        const float nm = -warp_max(mx) * 1.4426950408889634f;
        float v[CH][E];
        float sm = 0.0f;
#pragma unroll
        for (int k = 0; k < CH; ++k)
          if (lane + 32 * k < nchunks)
#pragma unroll
            for (int e = 0; e < E; ++e) {
              v[k][e] = ex2f_approx(fmaf(OutCvt<TI>::from(raw[k].e[e]), 1.4426950408889634f, nm));
              sm += v[k][e];
            }
        const float inv = 1.0f / warp_sum(sm);
#pragma unroll
        for (int k = 0; k < CH; ++k) {
          const int c = lane + 32 * k;
          if (c < nchunks) {
            Vec<TO> o;
#pragma unroll
            for (int e = 0; e < E; ++e) o.e[e] = OutCvt<TO>::to(v[k][e] * inv);
            st_stream(yr + c * E, o.u);
          }
        }
    }
  } else {
    // residual + layernorm, the R rows of a slot per warp: the rows' reduction
    // chains interleave, which hides the shuffle / smem latency a single row
    // per warp leaves exposed.
    constexpr int R = CH <= 4 ? AFG_LN_ROWS : 1;  // rows per slot (= grp at launch); long rows: 1
    const uint32_t gb_addr = smem_u32(gb);
    // a lane always owns the same columns (chunks lane + 32 k): its gamma / beta
    // live in registers for the whole kernel (rows of <= 768 16-bit columns)
    constexpr bool GB_REGS = CH <= 3;
    float greg[GB_REGS ? CH : 1][E], breg[GB_REGS ? CH : 1][E];
    if constexpr (GB_REGS) {
#pragma unroll
      for (int k = 0; k < CH; ++k) {
        const int c = lane + 32 * k;
#pragma unroll
        for (int e = 0; e < E; e += 4) {
          uint4 g4 = make_uint4(0, 0, 0, 0), b4 = make_uint4(0, 0, 0, 0);
          if (c < nchunks) {
            g4 = ld_shared_v4(gb_addr + (c * E + e) * 4);
            b4 = ld_shared_v4(gb_addr + (cols + c * E + e) * 4);
          }
          greg[k][e] = __uint_as_float(g4.x); greg[k][e + 1] = __uint_as_float(g4.y);
          greg[k][e + 2] = __uint_as_float(g4.z); greg[k][e + 3] = __uint_as_float(g4.w);
          breg[k][e] = __uint_as_float(b4.x); breg[k][e + 1] = __uint_as_float(b4.y);
          breg[k][e + 2] = __uint_as_float(b4.z); breg[k][e + 3] = __uint_as_float(b4.w);
        }
      }
    }
    if constexpr (sizeof(TI) == 2 && sizeof(TO) == 2 && GB_REGS) {
      // 16-bit rows: all arithmetic on packed f32x2 pairs (FADD2 / FFMA2), the
      // 16-bit <-> f32 conversions per pair: ~11 instructions per pair of
      // values instead of ~40 (the scalar version was issue-bound: 490
      // instructions per 768-column row, ncu profiles/r02/full_layernorm_*).
      uint64_t gp[CH][E / 2], bp[CH][E / 2];
#pragma unroll
      for (int k = 0; k < CH; ++k)
#pragma unroll
        for (int p = 0; p < E / 2; ++p) {
          gp[k][p] = sm100::f2(greg[k][2 * p], greg[k][2 * p + 1]);
          bp[k][p] = sm100::f2(breg[k][2 * p], breg[k][2 * p + 1]);
        }
      for (;; advance()) {
        if (ci >= cend) break;
        const int slot = cslot;
        mbar_wait(&full[slot], cph);
        const int dn = reinterpret_cast<volatile SlotDesc*>(desc)[slot].n;
        if (dn < 0) break;  // end of this warp's stream
        if (dn == 0) {      // skip
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[slot]);
          continue;
        }
        const int64_t row0 = reinterpret_cast<volatile SlotDesc*>(desc)[slot].row;
        const uint32_t sx = smem_u32(smem + static_cast<size_t>(slot) * slot_bytes);
        uint64_t v[R][CH][E / 2];
        bool have[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          have[r] = r < dn;
#pragma unroll
          for (int k = 0; k < CH; ++k) {
            const int c = lane + 32 * k;
            if (have[r] && c < nchunks) {
              const uint4 t = ld_shared_v4(sx + r * row_bytes + c * 16);
              const uint32_t tw[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
              for (int p = 0; p < 4; ++p) v[r][k][p] = unpack_pair<TI>(tw[p]);
              if (res) {
                const uint4 q = ld_shared_v4(sx + (R + r) * row_bytes + c * 16);
                const uint32_t qw[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
                for (int p = 0; p < 4; ++p) v[r][k][p] = sm100::fadd2(v[r][k][p], unpack_pair<TI>(qw[p]));
              }
            } else {
#pragma unroll
              for (int p = 0; p < 4; ++p) v[r][k][p] = 0ull;  // +0.0f pairs: neutral in the sums
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);  // slot consumed: it refills
        float s[R], q[R], mean[R], rstd[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          uint64_t a = 0ull, b = 0ull;
#pragma unroll
          for (int k = 0; k < CH; ++k) {
            a = sm100::fadd2(a, sm100::fadd2(v[r][k][0], v[r][k][1]));
            b = sm100::fadd2(b, sm100::fadd2(v[r][k][2], v[r][k][3]));
          }
          float x0, x1;
          sm100::f2split(sm100::fadd2(a, b), x0, x1);
          s[r] = x0 + x1;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int r = 0; r < R; ++r) s[r] += __shfl_xor_sync(0xffffffffu, s[r], o);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          mean[r] = s[r] * inv_cols;
          const uint64_t nm = sm100::f2(-mean[r], -mean[r]);
          uint64_t a = 0ull, b = 0ull;
#pragma unroll
          for (int k = 0; k < CH; ++k) {
            if (lane + 32 * k >= nchunks) continue;  // padded lanes hold zeros, not the mean
            const uint64_t d0 = sm100::fadd2(v[r][k][0], nm), d1 = sm100::fadd2(v[r][k][1], nm);
            const uint64_t d2 = sm100::fadd2(v[r][k][2], nm), d3 = sm100::fadd2(v[r][k][3], nm);
            a = sm100::ffma2(d0, d0, a);
            b = sm100::ffma2(d1, d1, b);
            a = sm100::ffma2(d2, d2, a);
            b = sm100::ffma2(d3, d3, b);
          }
          float x0, x1;
          sm100::f2split(sm100::fadd2(a, b), x0, x1);
          q[r] = x0 + x1;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int r = 0; r < R; ++r) q[r] += __shfl_xor_sync(0xffffffffu, q[r], o);
#pragma unroll
        for (int r = 0; r < R; ++r) rstd[r] = rsqrtf(fmaf(q[r], inv_cols, eps));
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (!have[r]) continue;
          const int64_t row = row0 + r;
          // y = ((v - mean) * rstd) * g + b = (v * rstd + (-mean * rstd)) * g + b
          const uint64_t ra = sm100::f2(rstd[r], rstd[r]);
          const float c0 = -mean[r] * rstd[r];
          const uint64_t rc = sm100::f2(c0, c0);
#pragma unroll
          for (int k = 0; k < CH; ++k) {
            const int c = lane + 32 * k;
            if (c >= nchunks) continue;
            uint32_t ow[4], sw[4];
#pragma unroll
            for (int p = 0; p < 4; ++p) {
              const uint64_t t = sm100::ffma2(v[r][k][p], ra, rc);
              ow[p] = pack_pair<TO>(sm100::ffma2(t, gp[k][p], bp[k][p]));
              if (sum_out) sw[p] = pack_pair<TO>(v[r][k][p]);
            }
            st_stream(y + row * cols + c * E, make_uint4(ow[0], ow[1], ow[2], ow[3]));
            if (sum_out)
              st_stream(sum_out + row * cols + c * E, make_uint4(sw[0], sw[1], sw[2], sw[3]));
          }
        }
      }
    } else {
    for (;; advance()) {
      if (ci >= cend) break;
      const int slot = cslot;
      mbar_wait(&full[slot], cph);
      const int dn = reinterpret_cast<volatile SlotDesc*>(desc)[slot].n;
      if (dn < 0) break;  // end of this warp's stream
      if (dn == 0) {      // skip
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        continue;
      }
      const int64_t row0 = reinterpret_cast<volatile SlotDesc*>(desc)[slot].row;
      const uint32_t sx = smem_u32(smem + static_cast<size_t>(slot) * slot_bytes);
      float v[R][CH][E];
      bool have[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        have[r] = r < dn;
        if (!have[r]) continue;
#pragma unroll
        for (int k = 0; k < CH; ++k) {
          const int c = lane + 32 * k;
          if (c < nchunks) {
            Vec<TI> t;
            t.u = ld_shared_v4(sx + r * row_bytes + c * 16);
#pragma unroll
            for (int e = 0; e < E; ++e) v[r][k][e] = OutCvt<TI>::from(t.e[e]);
            if (res) {
              Vec<TI> q;
              q.u = ld_shared_v4(sx + (R + r) * row_bytes + c * 16);
#pragma unroll
              for (int e = 0; e < E; ++e) v[r][k][e] += OutCvt<TI>::from(q.e[e]);
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);  // slot consumed: it refills
      // sums as short trees (one partial per chunk), both rows' shuffles interleaved
      float s[R], q[R], mean[R], rstd[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        float part[CH];
#pragma unroll
        for (int k = 0; k < CH; ++k) {
          part[k] = 0.0f;
          if (lane + 32 * k < nchunks) {
            float a = v[r][k][0] + v[r][k][1], b = v[r][k][2] + v[r][k][3];
#pragma unroll
            for (int e = 4; e < E; e += 4) {
              a += v[r][k][e] + v[r][k][e + 1];
              b += v[r][k][e + 2] + v[r][k][e + 3];
            }
            part[k] = a + b;
          }
        }
        s[r] = part[0];
#pragma unroll
        for (int k = 1; k < CH; ++k) s[r] += part[k];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int r = 0; r < R; ++r) s[r] += __shfl_xor_sync(0xffffffffu, s[r], o);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        mean[r] = s[r] * inv_cols;
        float part[CH];
#pragma unroll
        for (int k = 0; k < CH; ++k) {
          part[k] = 0.0f;
          if (lane + 32 * k < nchunks) {
            float a = 0.0f, b = 0.0f;
#pragma unroll
            for (int e = 0; e < E; e += 2) {
              const float d0 = v[r][k][e] - mean[r], d1 = v[r][k][e + 1] - mean[r];
              a = fmaf(d0, d0, a);
              b = fmaf(d1, d1, b);
            }
            part[k] = a + b;
          }
        }
        q[r] = part[0];
#pragma unroll
        for (int k = 1; k < CH; ++k) q[r] += part[k];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int r = 0; r < R; ++r) q[r] += __shfl_xor_sync(0xffffffffu, q[r], o);
#pragma unroll
      for (int r = 0; r < R; ++r) rstd[r] = rsqrtf(fmaf(q[r], inv_cols, eps));
#pragma unroll
      for (int k = 0; k < CH; ++k) {
        const int c = lane + 32 * k;
        if (c >= nchunks) continue;
        float gg[E], bb[E];
        if constexpr (GB_REGS) {
#pragma unroll
          for (int e = 0; e < E; ++e) {
            gg[e] = greg[k][e];
            bb[e] = breg[k][e];
          }
        } else {
#pragma unroll
          for (int e = 0; e < E; e += 4) {
            const uint4 g4 = ld_shared_v4(gb_addr + (c * E + e) * 4);
            const uint4 b4 = ld_shared_v4(gb_addr + (cols + c * E + e) * 4);
            gg[e] = __uint_as_float(g4.x); gg[e + 1] = __uint_as_float(g4.y);
            gg[e + 2] = __uint_as_float(g4.z); gg[e + 3] = __uint_as_float(g4.w);
            bb[e] = __uint_as_float(b4.x); bb[e + 1] = __uint_as_float(b4.y);
            bb[e + 2] = __uint_as_float(b4.z); bb[e + 3] = __uint_as_float(b4.w);
          }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (!have[r]) continue;
          const int64_t row = row0 + r;
          Vec<TO> o, so;
#pragma unroll
          for (int e = 0; e < E; ++e) {
            o.e[e] = OutCvt<TO>::to(fmaf((v[r][k][e] - mean[r]) * rstd[r], gg[e], bb[e]));
            so.e[e] = OutCvt<TO>::to(v[r][k][e]);
          }
          st_stream(y + row * cols + c * E, o.u);
          if (sum_out) st_stream(sum_out + row * cols + c * E, so.u);
        }
      }
    }
    }
  }
}

// Launches the streamed kernel when the shape allows it (16-bit rows whose
// chunks fit CH <= 16 per lane); returns cudaErrorNotSupported otherwise.
template <typename TI, typename TO, int MODE>
cudaError_t stream_launch(const void* x, const void* r, const float* g, const float* b, void* y,
                          void* so, int64_t rows, int64_t cols, float eps, cudaStream_t s) {
  constexpr int E = Vec<TI>::N;
  if (sizeof(TI) != sizeof(TO) || cols % E != 0) return cudaErrorNotSupported;
  const uintptr_t addr_or = reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(r) |
                            reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(so);
  if (addr_or & 15) return cudaErrorNotSupported;
  const int64_t nchunks = cols / E;
  // layernorm rows of <= 1024 16-bit values: two consecutive rows per ring
  // slot (one bulk copy each for x and the residual) and per consumer warp
  const int grp = MODE == 1 && nchunks <= 128 ? AFG_LN_ROWS : 1;
  const int64_t row_bytes = cols * static_cast<int64_t>(sizeof(TI));
  const int slot_bytes =
      static_cast<int>(((MODE == 1 && r ? 2 : 1) * grp * row_bytes + 127) / 128 * 128);
  // Ring depth is a multiple of the consumer-warp count: consumer warp w takes
  // slots w, w+15, ..., so the slot use one lap before slot i (i - ns) is its
  // own and was already consumed (loaded) when it waits on slot i. Otherwise a
  // warp can poll slot i % ns while use i - ns's bulk copy is still in flight
  // (copies complete out of order) and the parity wait passes a phase early.
  static const int64_t ln_budget_env = [] {  // AFG_LN_SMEM_KB: ring size (A/B measurements)
    const char* e = getenv("AFG_LN_SMEM_KB");
    return e ? static_cast<int64_t>(atoi(e)) * 1024 : 0;
  }();
  // AFG_STREAM_CPS = CTAs per SM (A/B): each with 1/cps of the ring budget.
  // Measured: 2 per SM layernorm 0.80 -> 0.66, softmax 0.98 -> 0.955 of HBM.
  static const int cps_env = [] {
    const char* e = getenv("AFG_STREAM_CPS");
    return e ? std::max(1, atoi(e)) : 1;
  }();
  const int64_t budget = (MODE == 1 ? (ln_budget_env > 0 ? ln_budget_env : STREAM_SMEM_LN)
                                    : STREAM_SMEM) / cps_env;
  const int ns = static_cast<int>(std::min<int64_t>(90, budget / slot_bytes)) /
                 STREAM_WARPS * STREAM_WARPS;
  if (ns < STREAM_WARPS || rows < 8ll * num_sms()) return cudaErrorNotSupported;
  const int smem = ns * slot_bytes + ns * 16 + (ns + 2) * static_cast<int>(sizeof(SlotDesc)) + 128 +
                   (MODE == 1 ? static_cast<int>(cols) * 8 + 16 : 0);
  // tail pool (AFG_STREAM_POOL = denominator, 0 = off). Measured: softmax
  // [262144, 2048] 370 -> 333 us with 1/4 of the rows pooled (1/16: no
  // change); layernorm [32768, 768] 30.2 -> 31.8-33 us with any pool (a 30 us
  // kernel cannot hide the claims' round trips), so it stays static.
  static const int pool_env = [] {
    const char* e = getenv("AFG_STREAM_POOL");
    return e ? atoi(e) : -1;
  }();
  const int pool_div = pool_env >= 0 ? pool_env : (MODE == 0 ? 4 : 0);
  unsigned int* pool_ctr = nullptr;
  int64_t pool = 0;
  if (pool_div > 0) {
    pool = rows / pool_div / grp * grp;
    static unsigned int* bases[64] = {};  // per device
    int dev = 0;
    cudaGetDevice(&dev);
    unsigned int*& base = bases[dev & 63];
    if (!base && cudaGetSymbolAddress(reinterpret_cast<void**>(&base), g_row_pool) != cudaSuccess)
      base = nullptr;
    const int slot = base ? stream_slot(s, 2, ROW_SLOTS) : -1;
    if (slot >= 0) {
      pool_ctr = base + 2 * slot;
    } else {
      cudaGetLastError();
      pool = 0;
    }
  }
  const TI* xi = reinterpret_cast<const TI*>(x);
  const TI* ri = reinterpret_cast<const TI*>(r);
  TO* yo = reinterpret_cast<TO*>(y);
  TO* soo = reinterpret_cast<TO*>(so);
  const unsigned grid = static_cast<unsigned>(num_sms() * cps_env);
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3((STREAM_WARPS + 1) * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // see gemm_tc.cu
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, xi, ri, g, b, yo, soo, rows, (int)cols, eps, ns,
                                       slot_bytes, grp, pool_ctr, pool);
    return e != cudaSuccess ? e : cudaGetLastError();
  };
  cudaError_t e;
  if (nchunks <= 32) e = go(stream_rows_kernel<TI, TO, MODE, 1>);
  else if (nchunks <= 64) e = go(stream_rows_kernel<TI, TO, MODE, 2>);
  else if (nchunks <= 96) e = go(stream_rows_kernel<TI, TO, MODE, 3>);
  else if (nchunks <= 128) e = go(stream_rows_kernel<TI, TO, MODE, 4>);
  else if (nchunks <= 256) e = go(stream_rows_kernel<TI, TO, MODE, 8>);
  else return cudaErrorNotSupported;  // longer rows: direct kernels
  count_launch();
  return e;
}

// ------------------------------------------------------------ layernorm --

template <typename T, int CH>
__global__ void __launch_bounds__(256) layernorm_warp_kernel(
    const T* __restrict__ x, const T* __restrict__ res, const float* __restrict__ gamma,
    const float* __restrict__ beta, T* __restrict__ y, T* __restrict__ sum_out, int64_t rows,
    int cols, float eps) {
  constexpr int E = Vec<T>::N;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (row >= rows) return;
  const int nchunks = cols / E;
  float v[CH][E];
  float s = 0.0f;
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    const int c = lane + 32 * i;
    if (c < nchunks) {
      Vec<T> a;
      a.u = ld_stream(x + row * cols + c * E);
      if (res) {
        Vec<T> b;
        b.u = ld_stream(res + row * cols + c * E);
#pragma unroll
        for (int e = 0; e < E; ++e) v[i][e] = OutCvt<T>::from(a.e[e]) + OutCvt<T>::from(b.e[e]);
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) v[i][e] = OutCvt<T>::from(a.e[e]);
      }
#pragma unroll
      for (int e = 0; e < E; ++e) s += v[i][e];
    }
  }
  const float mean = warp_sum(s) / cols;
  float q = 0.0f;
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    const int c = lane + 32 * i;
    if (c < nchunks) {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const float d = v[i][e] - mean;
        q = fmaf(d, d, q);
      }
    }
  }
  const float rstd = rsqrtf(warp_sum(q) / cols + eps);
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    const int c = lane + 32 * i;
    if (c < nchunks) {
      Vec<T> o, so;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int col = c * E + e;
        o.e[e] = OutCvt<T>::to((v[i][e] - mean) * rstd * __ldg(gamma + col) + __ldg(beta + col));
        so.e[e] = OutCvt<T>::to(v[i][e]);
      }
      st_stream(y + row * cols + c * E, o.u);
      if (sum_out) st_stream(sum_out + row * cols + c * E, so.u);
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256) layernorm_block_kernel(
    const T* __restrict__ x, const T* __restrict__ res, const float* __restrict__ gamma,
    const float* __restrict__ beta, T* __restrict__ y, T* __restrict__ sum_out, int cols,
    float eps) {
  __shared__ float red[33];
  const int64_t row = blockIdx.x;
  auto val = [&](int c) {
    float v = OutCvt<T>::from(x[row * cols + c]);
    if (res) v += OutCvt<T>::from(res[row * cols + c]);
    return v;
  };
  auto block_sum = [&](float v) {
    v = warp_sum(v);
    __syncthreads();
    if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
      float t = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0f;
      t = warp_sum(t);
      if (threadIdx.x == 0) red[32] = t;
    }
    __syncthreads();
    return red[32];
  };
  float s = 0.0f;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) s += val(c);
  const float mean = block_sum(s) / cols;
  float q = 0.0f;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) {
    const float d = val(c) - mean;
    q = fmaf(d, d, q);
  }
  const float rstd = rsqrtf(block_sum(q) / cols + eps);
  for (int c = threadIdx.x; c < cols; c += blockDim.x) {
    const float v = val(c);
    y[row * cols + c] = OutCvt<T>::to((v - mean) * rstd * gamma[c] + beta[c]);
    if (sum_out) sum_out[row * cols + c] = OutCvt<T>::to(v);
  }
}

template <typename T>
cudaError_t layernorm_launch(const void* x, const void* r, const float* g, const float* b,
                             void* y, void* so, int64_t rows, int64_t cols, float eps,
                             cudaStream_t s) {
  if (sizeof(T) == 2) {
    const cudaError_t e = stream_launch<T, T, 1>(x, r, g, b, y, so, rows, cols, eps, s);
    if (e != cudaErrorNotSupported) return e;
  }
  constexpr int E = Vec<T>::N;
  const uintptr_t addr_or = reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(r) |
                            reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(so);
  const bool vec_ok = cols % E == 0 && (addr_or & 15) == 0;
  const int64_t nchunks = cols / E;
  const T* xi = reinterpret_cast<const T*>(x);
  const T* ri = reinterpret_cast<const T*>(r);
  T* yo = reinterpret_cast<T*>(y);
  T* soo = reinterpret_cast<T*>(so);
  const unsigned grid = static_cast<unsigned>((rows + 7) / 8);
  if (vec_ok && nchunks <= 32 * 16) {
#define AFG_LN(CH) \
  layernorm_warp_kernel<T, CH><<<grid, 256, 0, s>>>(xi, ri, g, b, yo, soo, rows, (int)cols, eps)
    if (nchunks <= 32) AFG_LN(1);
    else if (nchunks <= 64) AFG_LN(2);
    else if (nchunks <= 96) AFG_LN(3);
    else if (nchunks <= 128) AFG_LN(4);
    else if (nchunks <= 256) AFG_LN(8);
    else AFG_LN(16);
#undef AFG_LN
  } else {
    layernorm_block_kernel<T><<<static_cast<unsigned>(rows), 256, 0, s>>>(xi, ri, g, b, yo, soo,
                                                                         (int)cols, eps);
  }
  count_launch();
  return cudaGetLastError();
}

template <typename TI, typename TO>
cudaError_t softmax_launch(const void* x, void* y, int64_t rows, int64_t cols, cudaStream_t s) {
  if (sizeof(TI) == 2 && sizeof(TO) == 2) {
    const cudaError_t e =
        stream_launch<TI, TO, 0>(x, nullptr, nullptr, nullptr, y, nullptr, rows, cols, 0.f, s);
    if (e != cudaErrorNotSupported) return e;
  }
  return softmax_launch_direct<TI, TO>(x, y, rows, cols, s);
}

// ----------------------------------------------------------- elementwise --

__global__ void elementwise_kernel(const void* __restrict__ a, const void* __restrict__ b,
                                   void* __restrict__ out, int64_t n, int64_t b_period, int op,
                                   int adt, int bdt, int odt) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float x = ld_any(a, i, adt);
    float r;
    if (op == AFG_OP_EXP) {
      r = expf(x);
    } else {
      const float y = ld_any(b, b_period > 0 ? i % b_period : i, bdt);
      switch (op) {
        case AFG_OP_ADD: r = x + y; break;
        case AFG_OP_SUB: r = x - y; break;
        case AFG_OP_MUL: r = x * y; break;
        default: r = fmaxf(x, y); break;
      }
    }
    st_any(out, i, odt, r);
  }
}

__global__ void reduce_kernel(const void* __restrict__ x, void* __restrict__ out, int64_t rows,
                              int64_t cols, int kind, int xdt, int odt) {
  const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (row >= rows) return;
  float acc = kind == AFG_REDUCE_MAX ? -INFINITY : 0.0f;
  bool nan = false;
  for (int64_t c = lane; c < cols; c += 32) {
    const float v = ld_any(x, row * cols + c, xdt);
    if (kind == AFG_REDUCE_MAXABS) {
      nan |= isnan(v);
      acc = fmaxf(acc, fabsf(v));
    } else {
      acc = kind == AFG_REDUCE_MAX ? fmaxf(acc, v) : acc + v;
    }
  }
  acc = kind == AFG_REDUCE_SUM ? warp_sum(acc) : warp_max(acc);
  if (kind == AFG_REDUCE_MAXABS && __any_sync(0xffffffffu, nan)) acc = NAN;
  if (lane == 0) st_any(out, row, odt, acc);
}

__global__ void convert_kernel(const void* __restrict__ x, void* __restrict__ y, int64_t n,
                               int xdt, int ydt) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    st_any(y, i, ydt, ld_any(x, i, xdt));
}

struct BroadcastArgs {
  int out_rank;
  int64_t out_shape[6];
  int64_t in_stride_for_out[6];  // 0 for broadcast output dims
};

__global__ void broadcast_kernel(const void* __restrict__ x, void* __restrict__ y, int64_t n,
                                 BroadcastArgs b, int xdt, int ydt) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t rem = i, src = 0;
    for (int d = b.out_rank - 1; d >= 0; --d) {
      const int64_t idx = rem % b.out_shape[d];
      rem /= b.out_shape[d];
      src += idx * b.in_stride_for_out[d];
    }
    st_any(y, i, ydt, ld_any(x, src, xdt));
  }
}

__global__ void quantize_kernel(const void* __restrict__ x, void* __restrict__ y, int64_t n,
                                float scale, int mode, int xdt, int ydt) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float v = ld_any(x, i, xdt);
    float r;
    if (mode == 0) {
      r = fminf(fmaxf(roundf(v / scale), -128.0f), 127.0f);  // std::round: half away from 0
    } else if (mode == 1) {
      r = v * scale;
    } else if (mode == 2) {
      r = fminf(fmaxf(rintf(v), -128.0f), 127.0f);
    } else {
      r = fminf(fmaxf(rintf(v), -2147483648.0f), 2147483647.0f);
    }
    st_any(y, i, ydt, r);
  }
}

__global__ void epilogue_apply_kernel(const void* __restrict__ acc, const float* __restrict__ bias,
                                      const void* __restrict__ res, void* __restrict__ out,
                                      int64_t rows, int64_t cols, int64_t ld, int epi, int adt,
                                      int odt) {
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / cols, c = i % cols;
    const int64_t idx = r * ld + c;
    float v = ld_any(acc, idx, adt);
    if (epi != AFG_EPI_NONE) v = apply_act_rt(epi, v + bias[c]);
    if (res) v += ld_any(res, idx, odt);
    st_any(out, idx, odt, v);
  }
}

struct TransposeArgs {
  int rank;
  int64_t out_shape[6];
  int64_t in_stride_for_out[6];  // input stride of the input dim mapped to out dim d
};

__global__ void transpose_kernel(const void* __restrict__ x, void* __restrict__ y, int64_t n,
                                 TransposeArgs t, int esize) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t rem = i, src = 0;
    for (int d = t.rank - 1; d >= 0; --d) {
      const int64_t idx = rem % t.out_shape[d];
      rem /= t.out_shape[d];
      src += idx * t.in_stride_for_out[d];
    }
    if (esize == 4)
      reinterpret_cast<float*>(y)[i] = reinterpret_cast<const float*>(x)[src];
    else
      reinterpret_cast<uint16_t*>(y)[i] = reinterpret_cast<const uint16_t*>(x)[src];
  }
}

// splitmix64 as in makeRandomTensor (interp.cpp:817-844): the i-th draw of a
// stream seeded with s0 is mix(s0 + (i + 1) * golden), so the whole tensor is
// generated in parallel and bit-identical to the reference generator.
__device__ __forceinline__ uint64_t splitmix_at(uint64_t s0, uint64_t i) {
  uint64_t z = s0 + (i + 1) * 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__global__ void fill_uniform_kernel(void* __restrict__ x, int64_t n, uint64_t seed, double lo,
                                    double hi, int dt) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t bits = splitmix_at(seed, static_cast<uint64_t>(i));
    const double u = static_cast<double>(bits >> 11) * (1.0 / 9007199254740992.0);
    const double v = lo + u * (hi - lo);
    switch (dt) {
      case AFG_F32: reinterpret_cast<float*>(x)[i] = static_cast<float>(v); break;
      case AFG_F16:
        reinterpret_cast<__half*>(x)[i] = __float2half_rn(static_cast<float>(v));
        break;
      default:
        reinterpret_cast<__nv_bfloat16*>(x)[i] = __float2bfloat16_rn(static_cast<float>(v));
        break;
    }
  }
}

unsigned grid_for(int64_t n, int per_block = 256) {
  int64_t g = (n + per_block - 1) / per_block;
  const int64_t cap = static_cast<int64_t>(num_sms()) * 32;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<unsigned>(g);
}

bool valid_dt(int t) { return t == AFG_F32 || t == AFG_F16 || t == AFG_BF16; }

}  // namespace
}  // namespace afg

using namespace afg;

extern "C" {

afg_status afg_softmax_lastdim(const void* x, void* y, int64_t rows, int64_t cols,
                               afg_dtype xd, afg_dtype yd, void* stream) {
  if (!x || !y || rows <= 0 || cols <= 0 || !valid_dt(xd) || !valid_dt(yd))
    return set_error(AFG_ERR_INVALID_ARG, "afg_softmax_lastdim: bad arguments");
  if (cols >= (1ll << 31)) return set_error(AFG_ERR_UNSUPPORTED, "softmax: cols too large");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
#define AFG_SM(TI, TO) e = softmax_launch<TI, TO>(x, y, rows, cols, s)
  if (xd == AFG_F32 && yd == AFG_F32) AFG_SM(float, float);
  else if (xd == AFG_F16 && yd == AFG_F16) AFG_SM(__half, __half);
  else if (xd == AFG_BF16 && yd == AFG_BF16) AFG_SM(__nv_bfloat16, __nv_bfloat16);
  else if (xd == AFG_F16 && yd == AFG_F32) AFG_SM(__half, float);
  else if (xd == AFG_BF16 && yd == AFG_F32) AFG_SM(__nv_bfloat16, float);
  else if (xd == AFG_F32 && yd == AFG_F16) AFG_SM(float, __half);
  else AFG_SM(float, __nv_bfloat16);
#undef AFG_SM
  return cuda_status(e, "softmax launch");
}

afg_status afg_layernorm_residual(const void* x, const void* residual, const float* gamma,
                                  const float* beta, void* y, void* sum_out, int64_t rows,
                                  int64_t cols, float eps, afg_dtype dtype, void* stream) {
  if (!x || !y || !gamma || !beta || rows <= 0 || cols <= 0 || !valid_dt(dtype))
    return set_error(AFG_ERR_INVALID_ARG, "afg_layernorm_residual: bad arguments");
  if (cols >= (1ll << 31) || rows >= (1ll << 31))
    return set_error(AFG_ERR_UNSUPPORTED, "layernorm: extent too large");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (dtype == AFG_F32)
    e = layernorm_launch<float>(x, residual, gamma, beta, y, sum_out, rows, cols, eps, s);
  else if (dtype == AFG_F16)
    e = layernorm_launch<__half>(x, residual, gamma, beta, y, sum_out, rows, cols, eps, s);
  else
    e = layernorm_launch<__nv_bfloat16>(x, residual, gamma, beta, y, sum_out, rows, cols, eps,
                                        s);
  return cuda_status(e, "layernorm launch");
}

afg_status afg_elementwise(const void* a, const void* b, void* out, int64_t n, int64_t b_period,
                           afg_binop op, afg_dtype ad, afg_dtype bd, afg_dtype od,
                           void* stream) {
  if (!a || !out || n <= 0 || (op != AFG_OP_EXP && !b) || op < AFG_OP_ADD || op > AFG_OP_EXP ||
      !valid_dt(ad) || !valid_dt(od) || (op != AFG_OP_EXP && !valid_dt(bd)))
    return set_error(AFG_ERR_INVALID_ARG, "afg_elementwise: bad arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  elementwise_kernel<<<grid_for(n), 256, 0, s>>>(a, b, out, n, b_period, op, ad, bd, od);
  count_launch();
  return cuda_status(cudaGetLastError(), "elementwise launch");
}

afg_status afg_reduce_lastdim(const void* x, void* out, int64_t rows, int64_t cols,
                              afg_reduce_kind kind, afg_dtype xd, afg_dtype od, void* stream) {
  if (!x || !out || rows <= 0 || cols <= 0 || !valid_dt(xd) || !valid_dt(od))
    return set_error(AFG_ERR_INVALID_ARG, "afg_reduce_lastdim: bad arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  reduce_kernel<<<static_cast<unsigned>((rows + 7) / 8), 256, 0, s>>>(x, out, rows, cols, kind,
                                                                     xd, od);
  count_launch();
  return cuda_status(cudaGetLastError(), "reduce launch");
}

afg_status afg_broadcast_in_dim(const void* x, void* y, int in_rank, const int64_t* in_shape,
                                int out_rank, const int64_t* out_shape, const int64_t* dims,
                                afg_dtype xd, afg_dtype yd, void* stream) {
  if (!x || !y || !out_shape || out_rank <= 0 || out_rank > 6 || in_rank < 0 ||
      in_rank > out_rank || (in_rank > 0 && (!in_shape || !dims)) || !valid_dt(xd) ||
      !valid_dt(yd))
    return set_error(AFG_ERR_INVALID_ARG, "afg_broadcast_in_dim: bad arguments");
  BroadcastArgs b;
  b.out_rank = out_rank;
  int64_t n = 1;
  for (int d = 0; d < out_rank; ++d) {
    b.out_shape[d] = out_shape[d];
    b.in_stride_for_out[d] = 0;
    n *= out_shape[d];
  }
  int64_t st = 1;
  for (int d = in_rank - 1; d >= 0; --d) {
    if (dims[d] < 0 || dims[d] >= out_rank || out_shape[dims[d]] != in_shape[d])
      return set_error(AFG_ERR_INVALID_ARG, "afg_broadcast_in_dim: dims/extents mismatch");
    b.in_stride_for_out[dims[d]] = st;
    st *= in_shape[d];
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  broadcast_kernel<<<grid_for(n), 256, 0, s>>>(x, y, n, b, xd, yd);
  count_launch();
  return cuda_status(cudaGetLastError(), "broadcast launch");
}

afg_status afg_epilogue_apply(const void* acc, const float* bias, const void* residual, void* out,
                              int64_t rows, int64_t cols, int64_t ld, afg_epilogue epi,
                              afg_dtype ad, afg_dtype od, void* stream) {
  if (!acc || !out || rows <= 0 || cols <= 0 || ld < cols || !valid_dt(ad) || !valid_dt(od) ||
      epi < AFG_EPI_NONE || epi > AFG_EPI_BIAS_GELU_ERF || (epi != AFG_EPI_NONE && !bias))
    return set_error(AFG_ERR_INVALID_ARG, "afg_epilogue_apply: bad arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  epilogue_apply_kernel<<<grid_for(rows * cols), 256, 0, s>>>(acc, bias, residual, out, rows, cols,
                                                             ld, epi, ad, od);
  count_launch();
  return cuda_status(cudaGetLastError(), "epilogue_apply launch");
}

afg_status afg_quantize(const void* x, void* y, int64_t n, float scale, int mode, afg_dtype xd,
                        afg_dtype yd, void* stream) {
  if (!x || !y || n <= 0 || mode < 0 || mode > 3 || (mode == 0 && scale == 0.0f) ||
      !valid_dt(xd) || !valid_dt(yd))
    return set_error(AFG_ERR_INVALID_ARG, "afg_quantize: bad arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  quantize_kernel<<<grid_for(n), 256, 0, s>>>(x, y, n, scale, mode, xd, yd);
  count_launch();
  return cuda_status(cudaGetLastError(), "quantize launch");
}

afg_status afg_convert(const void* x, void* y, int64_t n, afg_dtype xd, afg_dtype yd,
                       void* stream) {
  if (!x || !y || n <= 0 || !valid_dt(xd) || !valid_dt(yd))
    return set_error(AFG_ERR_INVALID_ARG, "afg_convert: bad arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  convert_kernel<<<grid_for(n), 256, 0, s>>>(x, y, n, xd, yd);
  count_launch();
  return cuda_status(cudaGetLastError(), "convert launch");
}

afg_status afg_transpose(const void* x, void* y, int rank, const int64_t* shape,
                         const int64_t* perm, afg_dtype dtype, void* stream) {
  if (!x || !y || !shape || !perm || rank <= 0 || rank > 6 || !valid_dt(dtype))
    return set_error(AFG_ERR_INVALID_ARG, "afg_transpose: bad arguments");
  TransposeArgs t;
  t.rank = rank;
  int64_t in_stride[6];
  int64_t st = 1, n = 1;
  for (int d = rank - 1; d >= 0; --d) {
    in_stride[d] = st;
    st *= shape[d];
  }
  bool seen[6] = {false, false, false, false, false, false};
  for (int d = 0; d < rank; ++d) {
    if (perm[d] < 0 || perm[d] >= rank || seen[perm[d]])
      return set_error(AFG_ERR_INVALID_ARG, "afg_transpose: bad perm");
    seen[perm[d]] = true;
    t.out_shape[d] = shape[perm[d]];
    t.in_stride_for_out[d] = in_stride[perm[d]];
    n *= shape[d];
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  transpose_kernel<<<grid_for(n), 256, 0, s>>>(x, y, n, t, dtype_bytes(dtype));
  count_launch();
  return cuda_status(cudaGetLastError(), "transpose launch");
}

afg_status afg_fill_uniform(void* x, int64_t n, uint64_t seed, float lo, float hi,
                            afg_dtype dtype, void* stream) {
  if (!x || n <= 0 || !valid_dt(dtype))
    return set_error(AFG_ERR_INVALID_ARG, "afg_fill_uniform: bad arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  fill_uniform_kernel<<<grid_for(n), 256, 0, s>>>(x, n, seed, lo, hi, dtype);
  count_launch();
  return cuda_status(cudaGetLastError(), "fill launch");
}

}  // extern "C"
