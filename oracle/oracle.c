/*
 * oracle.c - TEST INFRASTRUCTURE ONLY: plain-C restatement of the reference's
 * CPU arithmetic for the operator path. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / reference arm use it, as the checker. It is
 * never linked into libafg.so.
 *
 * Every function cites the reference code it restates (paths relative to
 * /root/reference/proj). Conventions follow the reference: values are
 * doubles, arithmetic is done in double, and results are rounded to the
 * declared element type at every store (interp.cpp:335-347).
 *
 * Pinning: tests/test_oracle.py checks these functions against (a) the
 * reference tests' known-answer vectors (test_interp.cpp:50-94, :221-255,
 * test_frontend.cpp graphs) committed under tests/golden/, and (b) the real
 * reference library compiled in oracle/_ref/ (af::interpret,
 * oracle::evalGraphReference, makeRandomInputs, roundToType).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Element type codes: the reference's ElementType order (ir.h:29) plus BF16. */
enum { T_F32 = 0, T_F16 = 1, T_I8 = 2, T_I32 = 3, T_BF16 = 10, T_F64 = 11 };
/* Epilogue codes (include/afg.h afg_epilogue). */
enum { E_NONE = 0, E_BIAS = 1, E_RELU = 2, E_GELU_TANH = 3, E_GELU_ERF = 4 };

/* ------------------------------------------------------------ rounding --- */

/* roundToF16, interp.cpp:25-86: via float, RNE incl. subnormals, overflow->inf */
double orc_round_f16(double v) {
  if (isnan(v) || isinf(v)) return v;
  float f = (float)v;
  uint32_t bits;
  memcpy(&bits, &f, 4);
  uint32_t sign = (bits >> 16) & 0x8000u;
  int32_t exponent = (int32_t)((bits >> 23) & 0xff) - 127 + 15;
  uint32_t mant = bits & 0x7fffffu;
  uint16_t half;
  if (exponent >= 31) {
    half = (uint16_t)(sign | 0x7c00u);
  } else if (exponent <= 0) {
    if (exponent < -10) {
      half = (uint16_t)sign;
    } else {
      mant |= 0x800000u;
      int shift = 14 - exponent;
      uint32_t m = mant >> shift;
      uint32_t rem = mant & ((1u << shift) - 1);
      uint32_t halfway = 1u << (shift - 1);
      if (rem > halfway || (rem == halfway && (m & 1))) ++m;
      half = (uint16_t)(sign | m);
    }
  } else {
    uint32_t m = mant >> 13;
    uint32_t rem = mant & 0x1fffu;
    if (rem > 0x1000u || (rem == 0x1000u && (m & 1))) ++m;
    uint32_t combined = ((uint32_t)exponent << 10) + m;
    if (combined >= 0x7c00u) combined = 0x7c00u;
    half = (uint16_t)(sign | combined);
  }
  uint32_t hs = (half & 0x8000u) << 16, he = (half >> 10) & 0x1f, hm = half & 0x3ffu, ob;
  if (he == 0) {
    if (hm == 0) {
      ob = hs;
    } else {
      int e = -1;
      uint32_t m = hm;
      do {
        ++e;
        m <<= 1;
      } while (!(m & 0x400u));
      ob = hs | ((uint32_t)(127 - 15 - e) << 23) | ((m & 0x3ffu) << 13);
    }
  } else if (he == 31) {
    ob = hs | 0x7f800000u | (hm << 13);
  } else {
    ob = hs | ((he - 15 + 127) << 23) | (hm << 13);
  }
  float out;
  memcpy(&out, &ob, 4);
  return (double)out;
}

/* bf16 (extension; the reference carries bf16 values in f32 tensors):
 * round to f32 first (as roundToType(F32)), then RNE to 8 mantissa bits,
 * matching __float2bfloat16_rn on the device. */
double orc_round_bf16(double v) {
  float f = (float)v;
  if (isnan(f) || isinf(f)) return (double)f;
  uint32_t b;
  memcpy(&b, &f, 4);
  uint32_t lsb = (b >> 16) & 1u;
  b += 0x7fffu + lsb;
  b &= 0xffff0000u;
  memcpy(&f, &b, 4);
  return (double)f;
}

/* roundToType, interp.cpp:88-104 */
double orc_round_to_type(double v, int t) {
  switch (t) {
    case T_F32: return (double)(float)v;
    case T_F16: return orc_round_f16(v);
    case T_I8: {
      double r = nearbyint(v);
      return r < -128.0 ? -128.0 : (r > 127.0 ? 127.0 : r);
    }
    case T_I32: {
      double r = nearbyint(v);
      return r < -2147483648.0 ? -2147483648.0 : (r > 2147483647.0 ? 2147483647.0 : r);
    }
    case T_BF16: return orc_round_bf16(v);
    default: return v;
  }
}

void orc_round_array(double* x, int64_t n, int t) {
  for (int64_t i = 0; i < n; ++i) x[i] = orc_round_to_type(x[i], t);
}

/* ------------------------------------------------------------------ RNG --- */

/* std::hash<std::string> of libstdc++ (_Hash_bytes, seed 0xc70f6907), which
 * makeRandomTensor mixes into its seed (interp.cpp:833). */
static uint64_t shift_mix(uint64_t v) { return v ^ (v >> 47); }
uint64_t orc_std_hash(const char* s) {
  const uint64_t mul = (((uint64_t)0xc6a4a793UL) << 32) + (uint64_t)0x5bd1e995UL;
  const size_t len = strlen(s);
  const size_t len_aligned = len & ~(size_t)7;
  uint64_t hash = 0xc70f6907UL ^ ((uint64_t)len * mul);
  for (size_t i = 0; i < len_aligned; i += 8) {
    uint64_t d;
    memcpy(&d, s + i, 8);
    d = shift_mix(d * mul) * mul;
    hash ^= d;
    hash *= mul;
  }
  if (len & 7) {
    uint64_t d = 0;
    for (int j = (int)(len & 7) - 1; j >= 0; --j) d = (d << 8) + (unsigned char)s[len_aligned + j];
    hash ^= d;
    hash *= mul;
  }
  hash = shift_mix(hash) * mul;
  return shift_mix(hash);
}

/* splitmix64, interp.cpp:808-815 */
static uint64_t splitmix64(uint64_t* state) {
  *state += 0x9e3779b97f4a7c15ull;
  uint64_t z = *state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

uint64_t orc_stream_seed(const char* buffer_id, uint64_t seed) {
  return seed ^ orc_std_hash(buffer_id);
}

/* makeRandomTensor, interp.cpp:817-844 (buffer_id includes the '%' prefix,
 * as lowered programs name buffers). Values are NOT rounded to the type. */
void orc_random_tensor(double* out, int64_t n, const char* buffer_id, uint64_t seed, double lo,
                       double hi, int is_int) {
  uint64_t state = orc_stream_seed(buffer_id, seed);
  for (int64_t i = 0; i < n; ++i) {
    uint64_t bits = splitmix64(&state);
    if (is_int) {
      out[i] = (double)((int64_t)(bits % 9) - 4);
    } else {
      double u = (double)(bits >> 11) * (1.0 / 9007199254740992.0);
      out[i] = lo + u * (hi - lo);
    }
  }
}

/* The raw stream from state s0 (s0 = seed ^ hash(id)), for sharded checks. */
void orc_random_stream(double* out, int64_t n, uint64_t s0, double lo, double hi) {
  uint64_t state = s0;
  for (int64_t i = 0; i < n; ++i) {
    uint64_t bits = splitmix64(&state);
    double u = (double)(bits >> 11) * (1.0 / 9007199254740992.0);
    out[i] = lo + u * (hi - lo);
  }
}

/* ------------------------------------------------------- parallel for --- */

typedef void (*range_fn)(void* ctx, int64_t begin, int64_t end);
typedef struct {
  range_fn fn;
  void* ctx;
  int64_t b, e;
} job_t;
static void* job_main(void* p) {
  job_t* j = (job_t*)p;
  j->fn(j->ctx, j->b, j->e);
  return NULL;
}
static void parallel_for(int64_t n, int threads, range_fn fn, void* ctx) {
  if (threads <= 1 || n < 2) {
    fn(ctx, 0, n);
    return;
  }
  if (threads > 256) threads = 256;
  if (threads > n) threads = (int)n;
  pthread_t th[256];
  job_t jobs[256];
  for (int t = 0; t < threads; ++t) {
    jobs[t].fn = fn;
    jobs[t].ctx = ctx;
    jobs[t].b = n * t / threads;
    jobs[t].e = n * (t + 1) / threads;
    pthread_create(&th[t], NULL, job_main, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
}

/* ----------------------------------------------------------- epilogue --- */

static double gelu_tanh_d(double x) {
  double u = 0.7978845608028654 * (x + 0.044715 * x * x * x);
  return x / (1.0 + exp(-2.0 * u));
}
static double gelu_erf_d(double x) { return 0.5 * x * (1.0 + erf(x / sqrt(2.0))); }

/* The bias / activation nests after a matmul (frontend.cpp:447-500: add of a
 * broadcast_in_dim bias, max with a zeros tensor), each a store rounded to
 * `t`. GELU is the closed form of the composite in SURVEY.md App. B. */
static double apply_epi(double acc, double bias, int epi, int t) {
  if (epi == E_NONE) return acc;
  double v = orc_round_to_type(acc + bias, t);
  switch (epi) {
    case E_RELU: return orc_round_to_type(v > 0.0 ? v : 0.0, t);
    case E_GELU_TANH: return orc_round_to_type(gelu_tanh_d(v), t);
    case E_GELU_ERF: return orc_round_to_type(gelu_erf_d(v), t);
    default: return v;
  }
}

/* -------------------------------------------------------------- matmul --- */

typedef struct {
  const double *A, *B, *bias;
  double* C;
  const int64_t* rows; /* optional row subset */
  int64_t M, N, K;
  int epi, acc_t, out_t, b_nk, interp;
} mm_ctx;

static void mm_range(void* p, int64_t b, int64_t e) {
  mm_ctx* c = (mm_ctx*)p;
  for (int64_t r = b; r < e; ++r) {
    const int64_t i = c->rows ? c->rows[r] : r;
    for (int64_t j = 0; j < c->N; ++j) {
      double acc = 0.0;
      for (int64_t k = 0; k < c->K; ++k) {
        const double a = c->A[i * c->K + k];
        const double bb = c->b_nk ? c->B[j * c->K + k] : c->B[k * c->N + j];
        if (c->interp)
          acc = orc_round_to_type(a * bb + acc, c->acc_t); /* interp.cpp:335-347 */
        else
          acc += a * bb; /* oracles.cpp:122-134 */
      }
      if (!c->interp) acc = orc_round_to_type(acc, T_F32); /* oracles.cpp:131 */
      const double bv = c->bias ? c->bias[j] : 0.0;
      double y = apply_epi(acc, bv, c->epi, c->out_t);
      if (c->epi == E_NONE) y = orc_round_to_type(y, c->out_t);
      c->C[r * c->N + j] = y;
    }
  }
}

/* C[M,N] = epi(A[M,K] . B + bias). A, B must already hold values on their
 * storage grid. interp = 1: sequential accumulation rounded to acc_t at every
 * k (the lowered matmul nest, frontend.cpp:679-733, run by interp.cpp:440-561);
 * interp = 0: double accumulation rounded once to f32 (matmulReference,
 * oracles.cpp:122-134). b_nk: B stored [N,K]. rows/n_rows: optional subset of
 * output rows (C then holds n_rows x N). */
void orc_matmul(const double* A, const double* B, const double* bias, double* C, int64_t M,
                int64_t N, int64_t K, int epi, int acc_t, int out_t, int b_nk, int interp,
                const int64_t* rows, int64_t n_rows, int threads) {
  mm_ctx c = {A, B, bias, C, rows, M, N, K, epi, acc_t, out_t, b_nk, interp};
  parallel_for(rows ? n_rows : M, threads, mm_range, &c);
}

/* batchMatmulReference, oracles.cpp:150-173 */
void orc_batch_matmul(const double* A, const double* B, double* C, int64_t batch, int64_t M,
                      int64_t N, int64_t K) {
  for (int64_t g = 0; g < batch; ++g)
    for (int64_t i = 0; i < M; ++i)
      for (int64_t j = 0; j < N; ++j) {
        double acc = 0;
        for (int64_t k = 0; k < K; ++k) acc += A[(g * M + i) * K + k] * B[(g * K + k) * N + j];
        C[(g * M + i) * N + j] = orc_round_to_type(acc, T_F32);
      }
}

/* ---------------------------------------------------------------- conv --- */

/* convGeometry, frontend.cpp:115-149 (also oracles.cpp:38-76). */
void orc_conv_geometry(int64_t inH, int64_t inW, int64_t kH, int64_t kW, int64_t sY, int64_t sX,
                       int64_t dY, int64_t dX, int same, int transposed, int64_t* out4) {
  int64_t oh, ow, py = 0, px = 0;
  if (!transposed) {
    if (same) {
      oh = (inH + sY - 1) / sY;
      ow = (inW + sX - 1) / sX;
      int64_t ty = (oh - 1) * sY + (kH - 1) * dY + 1 - inH;
      int64_t tx = (ow - 1) * sX + (kW - 1) * dX + 1 - inW;
      if (ty < 0) ty = 0;
      if (tx < 0) tx = 0;
      py = ty / 2;
      px = tx / 2;
    } else {
      oh = (inH - (kH - 1) * dY - 1) / sY + 1;
      ow = (inW - (kW - 1) * dX - 1) / sX + 1;
    }
  } else {
    if (same) {
      oh = inH * sY;
      ow = inW * sX;
      py = ((kH - 1) * dY + 1 - sY) / 2;
      px = ((kW - 1) * dX + 1 - sX) / 2;
    } else {
      oh = (inH - 1) * sY + (kH - 1) * dY + 1;
      ow = (inW - 1) * sX + (kW - 1) * dX + 1;
    }
  }
  out4[0] = oh;
  out4[1] = ow;
  out4[2] = py;
  out4[3] = px;
}

/* convReference, oracles.cpp:78-120: NCHW in, OIHW (transposed: IOHW) w,
 * double accumulation, output rounded to out_t. Explicit begin pads. */
void orc_conv_nchw(const double* in, const double* w, double* out, int64_t B, int64_t IC,
                   int64_t H, int64_t W, int64_t OC, int64_t KH, int64_t KW, int64_t sY,
                   int64_t sX, int64_t dY, int64_t dX, int64_t padY, int64_t padX,
                   int transposed, int64_t OH, int64_t OW, int out_t) {
  for (int64_t b = 0; b < B; ++b)
    for (int64_t oc = 0; oc < OC; ++oc)
      for (int64_t oy = 0; oy < OH; ++oy)
        for (int64_t ox = 0; ox < OW; ++ox) {
          double acc = 0;
          for (int64_t ic = 0; ic < IC; ++ic)
            for (int64_t ky = 0; ky < KH; ++ky)
              for (int64_t kx = 0; kx < KW; ++kx) {
                if (!transposed) {
                  int64_t iy = oy * sY + ky * dY - padY, ix = ox * sX + kx * dX - padX;
                  if (iy < 0 || iy >= H || ix < 0 || ix >= W) continue;
                  acc += in[((b * IC + ic) * H + iy) * W + ix] *
                         w[((oc * IC + ic) * KH + ky) * KW + kx];
                } else {
                  int64_t ny = oy + padY - ky * dY, nx = ox + padX - kx * dX;
                  if (ny % sY != 0 || nx % sX != 0) continue;
                  int64_t iy = ny / sY, ix = nx / sX;
                  if (iy < 0 || iy >= H || ix < 0 || ix >= W) continue;
                  acc += in[((b * IC + ic) * H + iy) * W + ix] *
                         w[((ic * OC + oc) * KH + ky) * KW + kx];
                }
              }
          out[((b * OC + oc) * OH + oy) * OW + ox] = orc_round_to_type(acc, out_t);
        }
}

typedef struct {
  const double *x, *w, *bias;
  double* y;
  const int64_t* images;
  int64_t H, W, C, OC, KH, KW, sY, sX, pT, pL, dY, dX, OH, OW;
  int epi, out_t;
} cv_ctx;

static void cv_range(void* p, int64_t b0, int64_t b1) {
  cv_ctx* c = (cv_ctx*)p;
  for (int64_t r = b0; r < b1; ++r) {
    const int64_t b = c->images ? c->images[r] : r;
    for (int64_t oy = 0; oy < c->OH; ++oy)
      for (int64_t ox = 0; ox < c->OW; ++ox)
        for (int64_t oc = 0; oc < c->OC; ++oc) {
          double acc = 0;
          for (int64_t ky = 0; ky < c->KH; ++ky) {
            const int64_t iy = oy * c->sY + ky * c->dY - c->pT;
            if (iy < 0 || iy >= c->H) continue;
            for (int64_t kx = 0; kx < c->KW; ++kx) {
              const int64_t ix = ox * c->sX + kx * c->dX - c->pL;
              if (ix < 0 || ix >= c->W) continue;
              const double* xp = c->x + ((b * c->H + iy) * c->W + ix) * c->C;
              const double* wp = c->w + ((oc * c->KH + ky) * c->KW + kx) * c->C;
              for (int64_t ic = 0; ic < c->C; ++ic) acc += xp[ic] * wp[ic];
            }
          }
          acc = orc_round_to_type(acc, T_F32);
          const double bv = c->bias ? c->bias[oc] : 0.0;
          double y = apply_epi(acc, bv, c->epi, c->out_t);
          if (c->epi == E_NONE) y = orc_round_to_type(y, c->out_t);
          c->y[((r * c->OH + oy) * c->OW + ox) * c->OC + oc] = y;
        }
  }
}

/* The same arithmetic as convReference (oracles.cpp:78-120: zero outside the
 * input, double accumulation, f32 result) in the NHWC / OHWI layout the B200
 * kernel uses, with explicit begin pads and the fused bias/act epilogue.
 * images/n_images: optional subset of batch images (y holds n_images). */
void orc_conv_nhwc(const double* x, const double* w, const double* bias, double* y, int64_t B,
                   int64_t H, int64_t W, int64_t C, int64_t OC, int64_t KH, int64_t KW,
                   int64_t sY, int64_t sX, int64_t pT, int64_t pL, int64_t dY, int64_t dX,
                   int64_t OH, int64_t OW, int epi, int out_t, const int64_t* images,
                   int64_t n_images, int threads) {
  cv_ctx c = {x, w, bias, y, images, H, W, C, OC, KH, KW, sY, sX, pT, pL, dY, dX, OH, OW, epi,
              out_t};
  parallel_for(images ? n_images : B, threads, cv_range, &c);
}

/* ----------------------------------------------------------- attention --- */

typedef struct {
  const double *q, *k, *v, *bias;
  double* o;
  const int64_t* heads;
  int64_t H, Nq, Nk, D;
  double scale;
  int causal;
} at_ctx;

static void at_range(void* p, int64_t h0, int64_t h1) {
  at_ctx* c = (at_ctx*)p;
  double* s = (double*)malloc(sizeof(double) * c->Nk);
  for (int64_t r = h0; r < h1; ++r) {
    const int64_t bh = c->heads ? c->heads[r] : r;
    const double* q = c->q + bh * c->Nq * c->D;
    const double* k = c->k + bh * c->Nk * c->D;
    const double* v = c->v + bh * c->Nk * c->D;
    for (int64_t i = 0; i < c->Nq; ++i) {
      double m = -INFINITY;
      for (int64_t j = 0; j < c->Nk; ++j) {
        double acc = 0;
        for (int64_t d = 0; d < c->D; ++d) acc += q[i * c->D + d] * k[j * c->D + d];
        acc *= c->scale;
        if (c->bias) acc += c->bias[(bh * c->Nq + i) * c->Nk + j];
        if (c->causal && j > i) acc = -INFINITY;
        s[j] = acc;
        if (acc > m) m = acc;
      }
      double sum = 0;
      for (int64_t j = 0; j < c->Nk; ++j) sum += exp(s[j] - m);
      for (int64_t d = 0; d < c->D; ++d) {
        double acc = 0;
        for (int64_t j = 0; j < c->Nk; ++j) acc += exp(s[j] - m) / sum * v[j * c->D + d];
        c->o[(r * c->Nq + i) * c->D + d] = acc;
      }
    }
  }
  free(s);
}

/* attentionReference, oracles.cpp:192-227 (softmax(QK^T + bias) V in double,
 * output not rounded), extended with a scale on QK^T (1 = the reference) and
 * causal masking (= the -inf upper-triangular additive bias). q/k/v [BH,N,D];
 * heads/n_heads: optional subset of flattened (b,h) indices (o holds n_heads). */
void orc_attention(const double* q, const double* k, const double* v, const double* bias,
                   double* o, int64_t BH, int64_t Nq, int64_t Nk, int64_t D, double scale,
                   int causal, const int64_t* heads, int64_t n_heads, int threads) {
  at_ctx c = {q, k, v, bias, o, heads, BH, Nq, Nk, D, scale, causal};
  parallel_for(heads ? n_heads : BH, threads, at_range, &c);
}

/* ------------------------------------------------------- memory chains --- */

/* softmaxReference, oracles.cpp:175-190 (double; caller rounds). */
void orc_softmax(const double* x, double* y, int64_t rows, int64_t cols) {
  for (int64_t r = 0; r < rows; ++r) {
    double m = -INFINITY;
    for (int64_t c = 0; c < cols; ++c) m = x[r * cols + c] > m ? x[r * cols + c] : m;
    double s = 0;
    for (int64_t c = 0; c < cols; ++c) s += exp(x[r * cols + c] - m);
    for (int64_t c = 0; c < cols; ++c) y[r * cols + c] = exp(x[r * cols + c] - m) / s;
  }
}

/* Layernorm (no reference op; restatement in the interpreter's conventions,
 * SURVEY.md §8c): s = x + res, mean, biased variance, all in double;
 * y = (s - mean) / sqrt(var + eps) * gamma + beta (caller rounds). */
void orc_layernorm(const double* x, const double* res, const double* gamma, const double* beta,
                   double* y, double* sum_out, int64_t rows, int64_t cols, double eps) {
  for (int64_t r = 0; r < rows; ++r) {
    double mean = 0, var = 0;
    for (int64_t c = 0; c < cols; ++c) {
      const double s = x[r * cols + c] + (res ? res[r * cols + c] : 0.0);
      mean += s;
    }
    mean /= (double)cols;
    for (int64_t c = 0; c < cols; ++c) {
      const double d = x[r * cols + c] + (res ? res[r * cols + c] : 0.0) - mean;
      var += d * d;
    }
    var /= (double)cols;
    const double rstd = 1.0 / sqrt(var + eps);
    for (int64_t c = 0; c < cols; ++c) {
      const double s = x[r * cols + c] + (res ? res[r * cols + c] : 0.0);
      y[r * cols + c] = (s - mean) * rstd * gamma[c] + beta[c];
      if (sum_out) sum_out[r * cols + c] = s;
    }
  }
}

/* ----------------------------------------------------------- compare --- */

/* compareTensors, interp.cpp:698-730: pass iff |a-b| <= tol * max(|a|,|b|,1)
 * everywhere (tol = 0: exact) and all values are finite. */
int orc_compare(const double* a, const double* b, int64_t n, double tol, double* max_abs,
                double* max_rel, int64_t* worst) {
  int passed = 1;
  double ma = 0, mr = 0;
  int64_t w = -1;
  for (int64_t i = 0; i < n; ++i) {
    const double av = a[i], bv = b[i];
    const double ab = fabs(av - bv);
    double den = fabs(av) > fabs(bv) ? fabs(av) : fabs(bv);
    if (den < 1.0) den = 1.0;
    const double rel = ab / den;
    if (ab > ma) ma = ab;
    if (rel > mr) {
      mr = rel;
      w = i;
    }
    const int ok = tol == 0.0 ? (ab == 0.0) : (ab <= tol * den);
    if (!ok) passed = 0;
    if (!isfinite(av) || !isfinite(bv)) passed = 0;
  }
  if (max_abs) *max_abs = ma;
  if (max_rel) *max_rel = mr;
  if (worst) *worst = w;
  return passed;
}
