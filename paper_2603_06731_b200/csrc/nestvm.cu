// nestvm.cu - the nest VM: executes one top-level loop nest of a lowered
// program (af::Program, ir.h) on the GPU with the reference interpreter's
// semantics (interp.cpp:164-696).
//
// Design (B200): the outermost perfectly nested loops whose iterations write
// provably disjoint elements are flattened into the thread index (mixed
// radix, innermost level fastest, so row-major stores coalesce); each thread
// then runs the remaining nest from a compact instruction stream: loops with
// affine max/min bounds, loads / stores through affine access maps (postfix
// index programs, mathematical floordiv / non-negative mod as affine.h), and
// the interpreter's scalar arithmetic in double precision with no FMA
// contraction (interp.cpp:502-561: fma is a*b+c, two roundings). Every store
// rounds to the buffer's declared type exactly as roundToType
// (interp.cpp:88-104; f16 through f32 as roundToF16 does) and is kept in that
// native type in HBM, so loads return exactly the interpreter's values.
// Out-of-bounds accesses raise the interpreter's InterpError. Scratch buffers
// in shared / register space referenced by one nest only are privatised per
// thread. An optional counting mode reproduces the interpreter's Metrics.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <set>
#include <sstream>
#include <stdexcept>
#include <dlfcn.h>
#include <mutex>
#include <thread>
#include <vector>
#include <nvrtc.h>
#include <type_traits>

#include "nestvm.h"

namespace afg {
namespace vm {

using gpu::ArithOp;
using gpu::ElementType;
using gpu::IndexExpr;
using gpu::InterpError;
using gpu::MemSpace;
using gpu::NestOp;
using gpu::NestOpKind;
using gpu::NestOperand;

namespace {

constexpr int MAX_RANK = 8;
constexpr int MAX_PAR = 8;
constexpr int NIV = 32;
constexpr int64_t EXPR_END = -1;
constexpr int64_t EXPR_IV = 101;  // resolved Dim: immediate = iv slot
constexpr size_t kErrBytes = 8 + 8 + 8 * NIV;
// threads x instructions above which a nest is compiled instead of interpreted
constexpr double kJitWork = 1 << 21;

enum VmOp : int32_t {
  OP_LOOP = 1, OP_END, OP_LOAD, OP_STORE, OP_ARITH, OP_IVVAL, OP_MMA_LOAD, OP_MMA_COMPUTE,
  OP_MMA_STORE
};

struct Ins {
  int32_t op, a, b, c, d, e;
  double imm;
};

struct VmBuf {
  char* ptr;
  int64_t shape[MAX_RANK];
  int64_t stride[MAX_RANK];
  int64_t priv;  // elements per thread when privatised, else 0
  int32_t type, rank, space, counter;
};

struct VmArgs {
  const Ins* code;
  const int64_t* expr;
  const int32_t* lists;
  const double* consts;
  const VmBuf* bufs;
  int32_t ncode, npar, nbufs;
  int64_t par_lo[MAX_PAR], par_ext[MAX_PAR], par_step[MAX_PAR];
  int32_t par_slot[MAX_PAR];
  int64_t total;
  unsigned long long* counters;
  int* err;
};

// ------------------------------------------------------------- device ----

__device__ __forceinline__ int64_t floordiv_d(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return q;
}
__device__ __forceinline__ int64_t floormod_d(int64_t a, int64_t b) {
  int64_t r = a % b;
  if (r != 0 && ((r < 0) != (b < 0))) r += b;
  return r;
}

__device__ int64_t eval_expr(const int64_t* e, const int64_t* iv) {
  int64_t st[16];
  int sp = 0;
  for (;;) {
    const int64_t op = *e++;
    switch (op) {
      case EXPR_END: return st[0];
      case IndexExpr::Const: st[sp++] = *e++; break;
      case EXPR_IV: st[sp++] = iv[*e++]; break;
      case IndexExpr::Add: --sp; st[sp - 1] += st[sp]; break;
      case IndexExpr::MulConst: st[sp - 1] *= *e++; break;
      case IndexExpr::FloorDiv: st[sp - 1] = floordiv_d(st[sp - 1], *e++); break;
      case IndexExpr::Mod: st[sp - 1] = floormod_d(st[sp - 1], *e++); break;
      default: return 0;
    }
  }
}

__device__ int64_t eval_list(const VmArgs& p, int list, const int64_t* iv, bool take_max) {
  const int32_t n = p.lists[list];
  int64_t best = 0;
  for (int i = 0; i < n; ++i) {
    const int64_t v = eval_expr(p.expr + p.lists[list + 1 + i], iv);
    if (i == 0 || (take_max ? v > best : v < best)) best = v;
  }
  return best;
}

// roundToType (interp.cpp:88-104) + bf16 (through f32, like f16)
__device__ __forceinline__ double round_to(double v, int t) {
  switch (t) {
    case VT_F32: return static_cast<double>(__double2float_rn(v));
    case VT_F16: return static_cast<double>(__half2float(__float2half_rn(__double2float_rn(v))));
    case VT_BF16:
      return static_cast<double>(__bfloat162float(__float2bfloat16_rn(__double2float_rn(v))));
    case VT_I8: return fmin(fmax(rint(v), -128.0), 127.0);
    case VT_I32: return fmin(fmax(rint(v), -2147483648.0), 2147483647.0);
    default: return v;
  }
}

__device__ __forceinline__ double ld_native(const char* p, int t) {
  switch (t) {
    case VT_F32: return *reinterpret_cast<const float*>(p);
    case VT_F16: return __half2float(*reinterpret_cast<const __half*>(p));
    case VT_BF16: return __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(p));
    case VT_I8: return *reinterpret_cast<const int8_t*>(p);
    case VT_I32: return *reinterpret_cast<const int32_t*>(p);
    default: return *reinterpret_cast<const double*>(p);
  }
}

// v is already on the type's grid
__device__ __forceinline__ void st_native(char* p, int t, double v) {
  switch (t) {
    case VT_F32: *reinterpret_cast<float*>(p) = static_cast<float>(v); break;
    case VT_F16: *reinterpret_cast<__half*>(p) = __float2half_rn(static_cast<float>(v)); break;
    case VT_BF16:
      *reinterpret_cast<__nv_bfloat16*>(p) = __float2bfloat16_rn(static_cast<float>(v));
      break;
    case VT_I8: *reinterpret_cast<int8_t*>(p) = static_cast<int8_t>(v); break;
    case VT_I32: *reinterpret_cast<int32_t*>(p) = static_cast<int32_t>(v); break;
    default: *reinterpret_cast<double*>(p) = v; break;
  }
}

__device__ __forceinline__ int type_bytes_d(int t) {
  return t == VT_I8 ? 1 : (t == VT_F16 || t == VT_BF16) ? 2 : t == VT_F64 ? 8 : 4;
}

// err: int code, int info, then (at byte 8) the live-iv mask and the 32 iv
// values of the failing thread (the interpreter's "[ivs: ...]" trace)
__device__ void fail(const VmArgs& p, int code, int info, const int64_t* iv = nullptr,
                     uint32_t live = 0) {
  if (atomicCAS(p.err, 0, code) == 0) {
    p.err[1] = info;
    int64_t* t = reinterpret_cast<int64_t*>(p.err + 2);
    t[0] = iv ? live : 0;
    if (iv)
      for (int i = 0; i < NIV; ++i) t[1 + i] = iv[i];
  }
}

// Counting mode: per-thread counters (the NestMetrics slots, then 4 per
// buffer of the nest's table for the first LOCAL_BUFS buffers), flushed with
// one atomic per non-zero slot when the thread finishes.
constexpr int LOCAL_BUFS = 16;
constexpr int LOCAL_SLOTS = 17 + 4 * LOCAL_BUFS;

template <bool COUNT>
__device__ __forceinline__ void count_access(const VmArgs& p, unsigned long long* cnt, int bi,
                                             const VmBuf& b, bool store, long long n) {
  if constexpr (COUNT) {
    const unsigned long long bytes = static_cast<unsigned long long>(n * type_bytes_d(b.type));
    cnt[4 * b.space + (store ? 1 : 0)] += static_cast<unsigned long long>(n);
    cnt[4 * b.space + (store ? 3 : 2)] += bytes;
    if (bi < LOCAL_BUFS) {
      cnt[17 + 4 * bi + (store ? 1 : 0)] += static_cast<unsigned long long>(n);
      cnt[17 + 4 * bi + (store ? 3 : 2)] += bytes;
    } else if (b.counter >= 0) {
      unsigned long long* q = p.counters + C_PER_BUFFER + 4 * b.counter;
      atomicAdd(q + (store ? 1 : 0), static_cast<unsigned long long>(n));
      atomicAdd(q + (store ? 3 : 2), bytes);
    }
  }
}

template <bool COUNT>
__device__ void flush_counts(const VmArgs& p, const unsigned long long* cnt) {
  if constexpr (COUNT) {
    for (int i = 0; i < 17; ++i)
      if (cnt[i]) atomicAdd(p.counters + i, cnt[i]);
    for (int bi = 0; bi < LOCAL_BUFS && bi < p.nbufs; ++bi) {
      const int c = p.bufs[bi].counter;
      if (c < 0) continue;
      for (int j = 0; j < 4; ++j)
        if (cnt[17 + 4 * bi + j]) atomicAdd(p.counters + C_PER_BUFFER + 4 * c + j, cnt[17 + 4 * bi + j]);
    }
  }
}

// element offset of an access, or -1 (and the InterpError flag) when out of bounds
__device__ int64_t address(const VmArgs& p, const VmBuf& b, int list, const int64_t* iv,
                           int buf_index, uint32_t live, int64_t row_extra = 0,
                           int64_t col_extra = 0) {
  const int32_t n = p.lists[list];
  if (n != b.rank) {
    fail(p, 2, buf_index, iv, live);
    return -1;
  }
  int64_t off = 0;
  for (int d = 0; d < n; ++d) {
    int64_t x = eval_expr(p.expr + p.lists[list + 1 + d], iv);
    if (d == n - 2) x += row_extra;
    if (d == n - 1) x += col_extra;
    if (x < 0 || x >= b.shape[d]) {
      fail(p, 1, buf_index, iv, live);
      return -1;
    }
    off += x * b.stride[d];
  }
  return off;
}

__device__ __forceinline__ const char* base_of(const VmBuf& b, int64_t tid) {
  return b.ptr + (b.priv ? tid * b.priv * type_bytes_d(b.type) : 0);
}

__device__ __forceinline__ double operand(int32_t x, const double* r, const double* k) {
  return x >= 0 ? r[x] : k[-x - 1];
}

template <int NR, int NF, bool COUNT>
__global__ void __launch_bounds__(128) nest_vm_kernel(const VmArgs p) {
  unsigned long long cnt[COUNT ? LOCAL_SLOTS : 1];
  if constexpr (COUNT)
    for (int i = 0; i < LOCAL_SLOTS; ++i) cnt[i] = 0;
  double r[NR];
  double frag[NF > 0 ? NF : 1][NF > 0 ? 256 : 1];
  int fragt[NF > 0 ? NF : 1];
  int64_t iv[NIV], ub[NIV];
  const int64_t nthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  for (int64_t t = tid; t < p.total; t += nthreads) {
    int64_t rem = t;
    for (int l = p.npar - 1; l >= 0; --l) {
      iv[p.par_slot[l]] = p.par_lo[l] + (rem % p.par_ext[l]) * p.par_step[l];
      rem /= p.par_ext[l];
    }
    if (*reinterpret_cast<volatile int*>(p.err) != 0) break;
    uint32_t live = 0;  // ivs currently bound (for the failure trace)
    for (int l = 0; l < p.npar; ++l) live |= 1u << p.par_slot[l];
    int pc = 0;
    while (pc < p.ncode) {
      const Ins in = p.code[pc];
      switch (in.op) {
        case OP_LOOP: {
          const int64_t lb = eval_list(p, in.b, iv, true);
          const int64_t hi = eval_list(p, in.c, iv, false);
          if (lb >= hi) {
            pc = in.e + 1;
          } else {
            iv[in.a] = lb;
            ub[in.a] = hi;
            live |= 1u << in.a;
            ++pc;
          }
          break;
        }
        case OP_END: {
          const int64_t v = iv[in.a] + in.d;
          if (v < ub[in.a]) {
            iv[in.a] = v;
            pc = in.b + 1;
          } else {
            live &= ~(1u << in.a);
            ++pc;
          }
          break;
        }
        case OP_IVVAL: r[in.a] = static_cast<double>(iv[in.b]); ++pc; break;
        case OP_LOAD: {
          const VmBuf& b = p.bufs[in.b];
          const int64_t off = address(p, b, in.c, iv, in.b, live);
          if (off < 0) goto done;
          r[in.a] = ld_native(base_of(b, tid) + off * type_bytes_d(b.type), b.type);
          count_access<COUNT>(p, cnt, in.b, b, false, 1);
          ++pc;
          break;
        }
        case OP_STORE: {
          const VmBuf& b = p.bufs[in.b];
          const int64_t off = address(p, b, in.c, iv, in.b, live);
          if (off < 0) goto done;
          const double v = round_to(operand(in.a, r, p.consts), b.type);
          st_native(const_cast<char*>(base_of(b, tid)) + off * type_bytes_d(b.type), b.type, v);
          count_access<COUNT>(p, cnt, in.b, b, true, 1);
          ++pc;
          break;
        }
        case OP_ARITH: {
          const int kind = in.b & 0xff, cast = (in.b >> 8) & 0xff;
          const double x = in.c != INT32_MIN ? operand(in.c, r, p.consts) : 0.0;
          const double y = in.d != INT32_MIN ? operand(in.d, r, p.consts) : 0.0;
          const double z = in.e != INT32_MIN ? operand(in.e, r, p.consts) : 0.0;
          double v = 0.0;
          switch (static_cast<ArithOp>(kind)) {
            case ArithOp::Add: v = __dadd_rn(x, y); break;
            case ArithOp::Mul: v = __dmul_rn(x, y); break;
            case ArithOp::Sub: v = __dsub_rn(x, y); break;
            case ArithOp::Div: v = __ddiv_rn(x, y); break;
            case ArithOp::Max: v = (x < y) ? y : x; break;  // std::max(a, b)
            case ArithOp::Exp: v = exp(x); break;
            case ArithOp::Negate: v = -x; break;
            case ArithOp::Cast:
              v = (cast == VT_I8 || cast == VT_I32) ? round_to(trunc(x), cast) : round_to(x, cast);
              break;
            case ArithOp::Fma: v = __dadd_rn(__dmul_rn(x, y), z); break;
            case ArithOp::Select: v = x != 0.0 ? y : z; break;
            case ArithOp::CmpEq: v = x == y ? 1.0 : 0.0; break;
            case ArithOp::CmpLt: v = x < y ? 1.0 : 0.0; break;
            case ArithOp::CmpLe: v = x <= y ? 1.0 : 0.0; break;
            case ArithOp::Quant:  // interp.cpp:547-552: round half away, clamp to i8
              v = fmin(fmax(round(__ddiv_rn(x, in.imm)), -128.0), 127.0);
              break;
            case ArithOp::Dequant: v = __dmul_rn(x, in.imm); break;
            case ArithOp::Round: v = round_to(x, cast); break;
          }
          r[in.a] = v;
          if constexpr (COUNT) {
            cnt[C_FLOPS] += (in.b >> 16) & 0xff;
            cnt[C_CORRECTION] += (in.b >> 24) & 1;
          }
          ++pc;
          break;
        }
        case OP_MMA_LOAD: {  // interp.cpp:563-583
          if (NF == 0) goto done;
          const VmBuf& b = p.bufs[in.b];
          double* f = frag[in.a < NF ? in.a : 0];
          fragt[in.a < NF ? in.a : 0] = b.type;
          for (int rr = 0; rr < 16; ++rr)
            for (int cc = 0; cc < 16; ++cc) {
              const int64_t off = address(p, b, in.c, iv, in.b, live, rr, cc);
              if (off < 0) goto done;
              f[rr * 16 + cc] = ld_native(base_of(b, tid) + off * type_bytes_d(b.type), b.type);
            }
          count_access<COUNT>(p, cnt, in.b, b, false, 256);
          if constexpr (COUNT) cnt[C_FRAG_LOADS] += 1;
          ++pc;
          break;
        }
        case OP_MMA_COMPUTE: {  // interp.cpp:585-600: exact 16x16x16, rounded once
          if (NF == 0) goto done;
          const double* fa = frag[in.c];
          const double* fb = frag[in.d];
          const int ct = fragt[in.e];
          double out[256];
          for (int rr = 0; rr < 16; ++rr)
            for (int cc = 0; cc < 16; ++cc) {
              double acc = frag[in.e][rr * 16 + cc];
              for (int k = 0; k < 16; ++k)
                acc = __dadd_rn(acc, __dmul_rn(fa[rr * 16 + k], fb[k * 16 + cc]));
              out[rr * 16 + cc] = round_to(acc, ct);
            }
          for (int i = 0; i < 256; ++i) frag[in.a][i] = out[i];
          fragt[in.a] = ct;
          if constexpr (COUNT) cnt[C_FRAG_COMPUTES] += 1;
          ++pc;
          break;
        }
        case OP_MMA_STORE: {  // interp.cpp:602-619
          if (NF == 0) goto done;
          const VmBuf& b = p.bufs[in.b];
          const double* f = frag[in.a];
          for (int rr = 0; rr < 16; ++rr)
            for (int cc = 0; cc < 16; ++cc) {
              const int64_t off = address(p, b, in.c, iv, in.b, live, rr, cc);
              if (off < 0) goto done;
              st_native(const_cast<char*>(base_of(b, tid)) + off * type_bytes_d(b.type), b.type,
                        round_to(f[rr * 16 + cc], b.type));
            }
          count_access<COUNT>(p, cnt, in.b, b, true, 256);
          if constexpr (COUNT) cnt[C_FRAG_STORES] += 1;
          ++pc;
          break;
        }
        default: fail(p, 3, pc, iv, live); goto done;
      }
    }
  }
done:
  flush_counts<COUNT>(p, cnt);
}

__global__ void f64_to_native_kernel(const double* __restrict__ x, char* __restrict__ y, int64_t n,
                                     int t) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    st_native(y + i * type_bytes_d(t), t, round_to(x[i], t));
}

__global__ void native_to_f64_kernel(const char* __restrict__ x, double* __restrict__ y, int64_t n,
                                     int t) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    y[i] = ld_native(x + i * type_bytes_d(t), t);
}

unsigned grid_for(int64_t n, int per_block = 256) {
  const int64_t g = (n + per_block - 1) / per_block;
  const int64_t cap = static_cast<int64_t>(num_sms()) * 8;
  return static_cast<unsigned>(std::max<int64_t>(1, std::min(g, cap)));
}

// ------------------------------------------------------------- host ------

int64_t floordiv_h(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return q;
}
int64_t floormod_h(int64_t a, int64_t b) {
  int64_t r = a % b;
  if (r != 0 && ((r < 0) != (b < 0))) r += b;
  return r;
}

// constant value of a bound list (no dims), or false
bool const_list(const std::vector<IndexExpr>& rs, bool take_max, int64_t* out) {
  if (rs.empty()) return false;
  int64_t best = 0;
  for (size_t i = 0; i < rs.size(); ++i) {
    std::vector<int64_t> st;
    const auto& c = rs[i].code;
    for (size_t k = 0; k < c.size();) {
      const int64_t op = c[k++];
      switch (op) {
        case IndexExpr::Const: st.push_back(c[k++]); break;
        case IndexExpr::Dim: return false;
        case IndexExpr::Add: {
          const int64_t b = st.back();
          st.pop_back();
          st.back() += b;
          break;
        }
        case IndexExpr::MulConst: st.back() *= c[k++]; break;
        case IndexExpr::FloorDiv: st.back() = floordiv_h(st.back(), c[k++]); break;
        case IndexExpr::Mod: st.back() = floormod_h(st.back(), c[k++]); break;
        default: return false;
      }
    }
    if (st.size() != 1) return false;
    if (i == 0 || (take_max ? st[0] > best : st[0] < best)) best = st[0];
  }
  *out = best;
  return true;
}

struct Encoder {
  std::vector<Ins> code;
  std::vector<int64_t> expr;
  std::vector<int32_t> lists;
  std::vector<double> consts;
  std::map<std::string, int> iv, reg, frag;
  std::map<std::string, int> buf;  // id -> index into bufs
  std::vector<std::string> bufs;

  int iv_slot(const std::string& n) {
    auto it = iv.find(n);
    if (it != iv.end()) return it->second;
    const int s = static_cast<int>(iv.size());
    if (s >= NIV) throw InterpError("afg nest vm: more than 32 loop ivs in one nest");
    iv[n] = s;
    return s;
  }
  int reg_slot(const std::string& n) {
    auto it = reg.find(n);
    if (it != reg.end()) return it->second;
    const int s = static_cast<int>(reg.size());
    reg[n] = s;
    return s;
  }
  int temp() { return reg_slot("$t" + std::to_string(reg.size())); }
  int frag_slot(const std::string& n) {
    auto it = frag.find(n);
    if (it != frag.end()) return it->second;
    const int s = static_cast<int>(frag.size());
    frag[n] = s;
    return s;
  }
  int buf_index(const std::string& id) {
    auto it = buf.find(id);
    if (it != buf.end()) return it->second;
    const int s = static_cast<int>(bufs.size());
    buf[id] = s;
    bufs.push_back(id);
    return s;
  }
  int32_t expr_of(const IndexExpr& e, const std::vector<std::string>& operands) {
    const int32_t off = static_cast<int32_t>(expr.size());
    for (size_t k = 0; k < e.code.size();) {
      const int64_t op = e.code[k++];
      if (op == IndexExpr::Dim) {
        const int64_t d = e.code[k++];
        if (d < 0 || d >= static_cast<int64_t>(operands.size()))
          throw InterpError("afg nest vm: access map dim without operand");
        auto it = iv.find(operands[d]);
        if (it == iv.end()) throw InterpError("unbound iv " + operands[d]);
        expr.push_back(EXPR_IV);
        expr.push_back(it->second);
      } else {
        expr.push_back(op);
        if (op == IndexExpr::Const || op == IndexExpr::MulConst || op == IndexExpr::FloorDiv ||
            op == IndexExpr::Mod) {
          if ((op == IndexExpr::FloorDiv || op == IndexExpr::Mod) && e.code[k] <= 0)
            throw InterpError("non-positive divisor");
          expr.push_back(e.code[k++]);
        }
      }
    }
    expr.push_back(EXPR_END);
    return off;
  }
  int32_t list_of(const std::vector<IndexExpr>& rs, const std::vector<std::string>& operands) {
    std::vector<int32_t> offs;
    for (const auto& r : rs) offs.push_back(expr_of(r, operands));
    const int32_t at = static_cast<int32_t>(lists.size());
    lists.push_back(static_cast<int32_t>(offs.size()));
    for (int32_t o : offs) lists.push_back(o);
    return at;
  }
  int32_t operand(const NestOperand& o) {
    if (o.isImm) {
      consts.push_back(o.imm);
      return -static_cast<int32_t>(consts.size());
    }
    auto it = reg.find(o.value);
    if (it != reg.end()) return it->second;
    auto jt = iv.find(o.value);
    if (jt != iv.end()) {  // an iv used as a value (interp.cpp:367-374)
      const int t = temp();
      code.push_back({OP_IVVAL, t, jt->second, 0, 0, 0, 0.0});
      return t;
    }
    throw InterpError("use of undefined value " + o.value);
  }
  void loop(const std::string& name, const std::vector<IndexExpr>& lo,
            const std::vector<IndexExpr>& hi, const std::vector<std::string>& ops, int64_t step,
            const std::vector<NestOp>& body) {
    const int32_t lb = list_of(lo, ops), hb = list_of(hi, ops);
    const int slot = iv_slot(name);
    const int at = static_cast<int>(code.size());
    code.push_back({OP_LOOP, slot, lb, hb, static_cast<int32_t>(step), 0, 0.0});
    for (const auto& c : body) emit(c);
    const int end = static_cast<int>(code.size());
    code.push_back({OP_END, slot, at, 0, static_cast<int32_t>(step), 0, 0.0});
    code[at].e = end;
  }
  void emit_parallel(const NestOp& op, size_t i) {
    if (i == op.ivs.size()) {
      for (const auto& c : op.body) emit(c);
      return;
    }
    NestOp inner;  // loop i wraps loops i+1.. and the body
    const int32_t lb = list_of(op.lowers[i], op.boundOperands);
    const int32_t hb = list_of(op.uppers[i], op.boundOperands);
    const int slot = iv_slot(op.ivs[i]);
    const int at = static_cast<int>(code.size());
    code.push_back({OP_LOOP, slot, lb, hb, 1, 0, 0.0});
    emit_parallel(op, i + 1);
    const int end = static_cast<int>(code.size());
    code.push_back({OP_END, slot, at, 0, 1, 0, 0.0});
    code[at].e = end;
  }
  void emit(const NestOp& op) {
    switch (op.kind) {
      case NestOpKind::For:
        if (op.step <= 0 || op.step > INT32_MAX) throw InterpError("afg nest vm: bad loop step");
        loop(op.ivs.at(0), op.lowers.at(0), op.uppers.at(0), op.boundOperands, op.step, op.body);
        break;
      case NestOpKind::Parallel: emit_parallel(op, 0); break;
      case NestOpKind::Load: {
        const int32_t l = list_of(op.access, op.accessOperands);
        code.push_back({OP_LOAD, reg_slot(op.result), buf_index(op.buffer), l, 0, 0, 0.0});
        break;
      }
      case NestOpKind::Store: {
        const int32_t v = operand(op.operands.at(0));
        const int32_t l = list_of(op.access, op.accessOperands);
        code.push_back({OP_STORE, v, buf_index(op.buffer), l, 0, 0, 0.0});
        break;
      }
      case NestOpKind::Arith: {
        int32_t x[3] = {INT32_MIN, INT32_MIN, INT32_MIN};
        for (size_t i = 0; i < op.operands.size() && i < 3; ++i) x[i] = operand(op.operands[i]);
        const int k = static_cast<int>(op.arith);
        const int fl = op.arith == ArithOp::Fma ? 2
                       : (op.arith == ArithOp::Select || op.arith == ArithOp::CmpEq ||
                          op.arith == ArithOp::CmpLt || op.arith == ArithOp::CmpLe ||
                          op.arith == ArithOp::Cast || op.arith == ArithOp::Round)
                           ? 0
                           : 1;
        const int corr = op.attrs.count("correction") ? 1 : 0;
        const int32_t packed = k | (vm_type(op.castType) << 8) | (fl << 16) | (corr << 24);
        code.push_back({OP_ARITH, reg_slot(op.result), packed, x[0], x[1], x[2], op.scale});
        break;
      }
      case NestOpKind::MmaLoad: {
        const int32_t l = list_of(op.access, op.accessOperands);
        code.push_back({OP_MMA_LOAD, frag_slot(op.result), buf_index(op.buffer), l, 0, 0, 0.0});
        break;
      }
      case NestOpKind::MmaCompute: {
        auto f = [&](int i) {
          auto it = frag.find(op.operands.at(i).value);
          if (it == frag.end()) throw InterpError("scalar value where fragment expected");
          return it->second;
        };
        const int a = f(0), b = f(1), c = f(2);
        code.push_back({OP_MMA_COMPUTE, frag_slot(op.result), 0, a, b, c, 0.0});
        break;
      }
      case NestOpKind::MmaStore: {
        auto it = frag.find(op.operands.at(0).value);
        if (it == frag.end()) throw InterpError("scalar value where fragment expected");
        const int32_t l = list_of(op.access, op.accessOperands);
        code.push_back({OP_MMA_STORE, it->second, buf_index(op.buffer), l, 0, 0, 0.0});
        break;
      }
      case NestOpKind::AsyncCopy:  // completion-at-await == eager for a src no one rewrites
        for (const auto& c : op.body) emit(c);
        break;
      case NestOpKind::AwaitCopies:
      case NestOpKind::Alloc:
      case NestOpKind::Dealloc: break;
    }
  }
};

// ---- parallel-level analysis ----

struct AccessRec {
  std::string buf;
  std::vector<Linear> lin;
  bool store = false;
  bool mma = false;
};

void collect_accesses(const NestOp& op, std::vector<AccessRec>& out) {
  switch (op.kind) {
    case NestOpKind::Load:
    case NestOpKind::Store:
    case NestOpKind::MmaLoad:
    case NestOpKind::MmaStore: {
      AccessRec a;
      a.buf = op.buffer;
      a.store = op.kind == NestOpKind::Store || op.kind == NestOpKind::MmaStore;
      a.mma = op.kind == NestOpKind::MmaLoad || op.kind == NestOpKind::MmaStore;
      for (const auto& e : op.access) a.lin.push_back(linearize(e, op.accessOperands));
      out.push_back(std::move(a));
      break;
    }
    default: break;
  }
  for (const auto& c : op.body) collect_accesses(c, out);
}

void collect_buffers(const NestOp& op, std::set<std::string>& out) {
  if (!op.buffer.empty()) out.insert(op.buffer);
  if (!op.srcBuffer.empty()) out.insert(op.srcBuffer);
  for (const auto& c : op.body) collect_buffers(c, out);
}

// Do the iterations of the parallel ivs P write disjoint elements, and does
// every thread read back only elements it writes itself?
bool disjoint(const std::vector<AccessRec>& acc, const std::vector<std::string>& P,
              const std::set<std::string>& privatised) {
  std::set<std::string> written;
  for (const auto& a : acc)
    if (a.store) written.insert(a.buf);
  for (const std::string& X : written) {
    if (privatised.count(X)) continue;
    // pinned positions: result r == c*p + k for a parallel iv p
    struct Pin {
      std::string p;
      int64_t c, k;
      bool operator==(const Pin& o) const { return p == o.p && c == o.c && k == o.k; }
    };
    bool first = true;
    std::map<size_t, Pin> pins;
    for (const auto& a : acc) {
      if (!a.store || a.buf != X) continue;
      std::map<size_t, Pin> mine;
      std::set<std::string> covered;
      for (size_t r = 0; r < a.lin.size(); ++r) {
        const Linear& L = a.lin[r];
        if (!L.affine || L.coef.size() != 1) continue;
        const auto& [name, c] = *L.coef.begin();
        if (std::find(P.begin(), P.end(), name) == P.end() || c == 0) continue;
        if (a.mma && r + 2 >= a.lin.size() && std::llabs(c) < 16) continue;
        mine[r] = Pin{name, c, L.c};
        covered.insert(name);
      }
      if (covered.size() != P.size()) return false;
      if (first) {
        pins = mine;
        first = false;
      } else {
        if (mine.size() != pins.size()) return false;
        for (const auto& [r, pin] : mine) {
          auto it = pins.find(r);
          if (it == pins.end() || !(it->second == pin)) return false;
        }
      }
    }
    for (const auto& a : acc) {
      if (a.store || a.buf != X) continue;
      for (const auto& [r, pin] : pins) {
        if (r >= a.lin.size()) return false;
        const Linear& L = a.lin[r];
        if (!L.affine || L.coef.size() != 1 || L.c != pin.k) return false;
        const auto& [name, c] = *L.coef.begin();
        if (name != pin.p || c != pin.c) return false;
      }
    }
  }
  return true;
}

template <int NR, int NF>
cudaError_t launch_vm(const VmArgs& a, unsigned grid, cudaStream_t s) {
  if (a.counters)
    nest_vm_kernel<NR, NF, true><<<grid, 128, 0, s>>>(a);
  else
    nest_vm_kernel<NR, NF, false><<<grid, 128, 0, s>>>(a);
  return cudaGetLastError();
}


// ------------------------------------------------------------- JIT -------
// The same encoded nest, compiled: the instruction stream is translated to
// CUDA C (loops -> for loops, loads / stores -> typed accesses with the bounds
// check, arithmetic -> the interpreter's double operations with explicit
// _rn intrinsics, no contraction) and compiled once per distinct nest with
// NVRTC for sm_100a (-fmad=false), cached per device. Same semantics as the
// interpreting kernel, at memory speed: the graph planner's fused regions and
// the program executor's large nests run through it; small nests, counting
// mode and fragment ops stay on the interpreter.

namespace jit {

struct Nvrtc {
  bool ok = false;
  std::string why;
  nvrtcResult (*create)(nvrtcProgram*, const char*, const char*, int, const char* const*,
                        const char* const*) = nullptr;
  nvrtcResult (*compile)(nvrtcProgram, int, const char* const*) = nullptr;
  nvrtcResult (*cubin_size)(nvrtcProgram, size_t*) = nullptr;
  nvrtcResult (*cubin)(nvrtcProgram, char*) = nullptr;
  nvrtcResult (*log_size)(nvrtcProgram, size_t*) = nullptr;
  nvrtcResult (*log)(nvrtcProgram, char*) = nullptr;
  nvrtcResult (*destroy)(nvrtcProgram*) = nullptr;
};

const Nvrtc& nvrtc() {
  static Nvrtc n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnvrtc.so.12", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("/usr/local/cuda/lib64/libnvrtc.so.12", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      n.why = "libnvrtc.so.12 not loadable";
      return;
    }
    auto sym = [&](auto& f, const char* name) {
      f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name));
      return f != nullptr;
    };
    n.ok = sym(n.create, "nvrtcCreateProgram") && sym(n.compile, "nvrtcCompileProgram") &&
           sym(n.cubin_size, "nvrtcGetCUBINSize") && sym(n.cubin, "nvrtcGetCUBIN") &&
           sym(n.log_size, "nvrtcGetProgramLogSize") && sym(n.log, "nvrtcGetProgramLog") &&
           sym(n.destroy, "nvrtcDestroyProgram");
    if (!n.ok) n.why = "libnvrtc lacks a symbol";
  });
  return n;
}

constexpr int MAX_BUFS = 48;
struct JitArgs {
  char* ptr[MAX_BUFS];
  int* err;
  long long total;
};

std::string lit(double v) {
  uint64_t u;
  std::memcpy(&u, &v, 8);
  char b[64];
  std::snprintf(b, sizeof(b), "__longlong_as_double(0x%016llxLL)", static_cast<unsigned long long>(u));
  return b;
}

const char* kPrelude = R"(
typedef long long LL;
__device__ __forceinline__ LL fdiv(LL a, LL b) { LL q = a / b; if ((a % b != 0) && ((a < 0) != (b < 0))) --q; return q; }
__device__ __forceinline__ LL fmd(LL a, LL b) { LL r = a % b; if (r != 0 && ((r < 0) != (b < 0))) r += b; return r; }
__device__ __forceinline__ float h2f(unsigned short h) { float f; asm("cvt.f32.f16 %0, %1;" : "=f"(f) : "h"(h)); return f; }
__device__ __forceinline__ unsigned short f2h(float f) { unsigned short h; asm("cvt.rn.f16.f32 %0, %1;" : "=h"(h) : "f"(f)); return h; }
__device__ __forceinline__ float b2f(unsigned short h) { return __uint_as_float(((unsigned)h) << 16); }
__device__ __forceinline__ unsigned short f2b(float f) { unsigned short h; asm("cvt.rn.bf16.f32 %0, %1;" : "=h"(h) : "f"(f)); return h; }
__device__ __forceinline__ double rt0(double v) { return (double)__double2float_rn(v); }
__device__ __forceinline__ double rt1(double v) { return (double)h2f(f2h(__double2float_rn(v))); }
__device__ __forceinline__ double rt2(double v) { return (double)b2f(f2b(__double2float_rn(v))); }
__device__ __forceinline__ double rt3(double v) { return fmin(fmax(rint(v), -128.0), 127.0); }
__device__ __forceinline__ double rt4(double v) { return fmin(fmax(rint(v), -2147483648.0), 2147483647.0); }
__device__ __forceinline__ double rt5(double v) { return v; }
struct JitArgs { char* ptr[48]; int* err; LL total; };
)";

const char* ld_expr(int t) {
  switch (t) {
    case VT_F32: return "(double)((const float*)%s)[%s]";
    case VT_F16: return "(double)h2f(((const unsigned short*)%s)[%s])";
    case VT_BF16: return "(double)b2f(((const unsigned short*)%s)[%s])";
    case VT_I8: return "(double)((const signed char*)%s)[%s]";
    case VT_I32: return "(double)((const int*)%s)[%s]";
    default: return "((const double*)%s)[%s]";
  }
}
std::string st_stmt(int t, const std::string& p, const std::string& off, const std::string& v) {
  switch (t) {
    case VT_F32: return "((float*)" + p + ")[" + off + "] = (float)(" + v + ");";
    case VT_F16: return "((unsigned short*)" + p + ")[" + off + "] = f2h((float)(" + v + "));";
    case VT_BF16: return "((unsigned short*)" + p + ")[" + off + "] = f2b((float)(" + v + "));";
    case VT_I8: return "((signed char*)" + p + ")[" + off + "] = (signed char)(" + v + ");";
    case VT_I32: return "((int*)" + p + ")[" + off + "] = (int)(" + v + ");";
    default: return "((double*)" + p + ")[" + off + "] = " + v + ";";
  }
}

// postfix index program -> C expression
std::string cexpr(const std::vector<int64_t>& ex, int32_t off) {
  std::vector<std::string> st;
  for (size_t k = static_cast<size_t>(off);;) {
    const int64_t op = ex[k++];
    if (op == EXPR_END) break;
    switch (op) {
      case IndexExpr::Const: st.push_back("(" + std::to_string(ex[k++]) + "LL)"); break;
      case EXPR_IV: st.push_back("i" + std::to_string(ex[k++])); break;
      case IndexExpr::Add: {
        const std::string b = st.back();
        st.pop_back();
        st.back() = "(" + st.back() + " + " + b + ")";
        break;
      }
      case IndexExpr::MulConst: st.back() = "(" + st.back() + " * " + std::to_string(ex[k++]) + "LL)"; break;
      case IndexExpr::FloorDiv: st.back() = "fdiv(" + st.back() + ", " + std::to_string(ex[k++]) + "LL)"; break;
      case IndexExpr::Mod: st.back() = "fmd(" + st.back() + ", " + std::to_string(ex[k++]) + "LL)"; break;
      default: throw InterpError("afg nest jit: bad index code");
    }
  }
  return st.at(0);
}

// Source of the nest kernel, or "" when the program uses what the JIT does
// not translate (fragments).
std::string source(const Encoder& enc, const std::vector<VmBuf>& bt, const VmArgs& a) {
  std::ostringstream o;
  o << kPrelude;
  o << "extern \"C\" __global__ void __launch_bounds__(128) nest_jit(JitArgs p) {\n";
  o << "  const LL nth = (LL)gridDim.x * blockDim.x;\n";
  o << "  const LL tid = (LL)blockIdx.x * blockDim.x + threadIdx.x;\n";
  const int niv = static_cast<int>(enc.iv.size());
  const int nreg = static_cast<int>(enc.reg.size());
  for (int i = 0; i < niv; ++i) o << "  LL i" << i << " = 0;\n";
  for (int r = 0; r < nreg; ++r) o << "  double r" << r << " = 0.0;\n";
  for (size_t b = 0; b < bt.size(); ++b) {
    o << "  char* P" << b << " = p.ptr[" << b << "]";
    if (bt[b].priv) o << " + tid * " << bt[b].priv * vm_type_bytes(static_cast<VmType>(bt[b].type)) << "LL";
    o << ";\n";
  }
  o << "  for (LL t = tid; t < p.total; t += nth) {\n    LL rem = t;\n";
  uint32_t live = 0;
  for (int l = a.npar - 1; l >= 0; --l) {
    o << "    i" << a.par_slot[l] << " = " << a.par_lo[l] << "LL + (rem % " << a.par_ext[l]
      << "LL) * " << a.par_step[l] << "LL; rem /= " << a.par_ext[l] << "LL;\n";
    live |= 1u << a.par_slot[l];
  }
  std::vector<uint32_t> live_stack;
  auto operand = [&](int32_t x) {
    return x >= 0 ? "r" + std::to_string(x) : lit(enc.consts.at(-x - 1));
  };
  // f32 fast path. A register is "f32-exact" when every definition of it
  // yields a value on the f32 grid (loads of f32 / f16 / bf16 / i8 buffers,
  // roundings to those types, the fused ops below). For + - * / max of two
  // f32-exact values immediately rounded to f32 (and used nowhere else), the
  // interpreter's double op + roundToType(F32) equals the f32 op: double
  // rounding through 53 bits is innocuous for these operations (53 >= 2*24+2),
  // so the generated code uses the f32 instruction -- still bit-exact.
  std::vector<int> uses(nreg, 0), defs_exact(nreg, 0), defs(nreg, 0);
  auto use = [&](int32_t x) {
    if (x >= 0 && x != INT32_MIN) ++uses[x];
  };
  auto grid32 = [](int t) { return t == VT_F32 || t == VT_F16 || t == VT_BF16 || t == VT_I8; };
  for (const Ins& in : enc.code) {
    if (in.op == OP_STORE) use(in.a);
    if (in.op == OP_ARITH) {
      use(in.c);
      use(in.d);
      use(in.e);
    }
  }
  for (size_t pc = 0; pc < enc.code.size(); ++pc) {
    const Ins& in = enc.code[pc];
    if (in.op == OP_LOAD) {
      ++defs[in.a];
      defs_exact[in.a] += grid32(bt[in.b].type);
    } else if (in.op == OP_IVVAL) {
      ++defs[in.a];
    } else if (in.op == OP_ARITH) {
      ++defs[in.a];
      const int kind = in.b & 0xff, cast = (in.b >> 8) & 0xff;
      if ((static_cast<ArithOp>(kind) == ArithOp::Round || static_cast<ArithOp>(kind) == ArithOp::Cast) &&
          grid32(cast))
        ++defs_exact[in.a];
    }
  }
  auto exact = [&](int32_t x) {
    if (x == INT32_MIN) return false;
    if (x < 0) {
      const double v = enc.consts.at(-x - 1);
      return static_cast<double>(static_cast<float>(v)) == v || v != v;
    }
    return defs[x] > 0 && defs[x] == defs_exact[x];
  };
  std::vector<bool> fused(enc.code.size(), false);  // arith folded into the next Round(F32)
  for (size_t pc = 0; pc + 1 < enc.code.size(); ++pc) {
    const Ins& in = enc.code[pc];
    const Ins& nx = enc.code[pc + 1];
    if (in.op != OP_ARITH || nx.op != OP_ARITH) continue;
    const auto k = static_cast<ArithOp>(in.b & 0xff);
    const bool f32op = k == ArithOp::Add || k == ArithOp::Sub || k == ArithOp::Mul ||
                       k == ArithOp::Div || k == ArithOp::Max;
    if (!f32op || static_cast<ArithOp>(nx.b & 0xff) != ArithOp::Round ||
        ((nx.b >> 8) & 0xff) != VT_F32 || nx.c != in.a || uses[in.a] != 1 || !exact(in.c) ||
        !exact(in.d))
      continue;
    fused[pc] = true;
  }
  auto list = [&](int32_t at, const char* fn) {
    const int32_t n = enc.lists.at(at);
    std::string e = cexpr(enc.expr, enc.lists.at(at + 1));
    for (int32_t i = 1; i < n; ++i)
      e = std::string(fn) + "(" + e + ", " + cexpr(enc.expr, enc.lists.at(at + 1 + i)) + ")";
    return e;
  };
  auto fail = [&](int code, int buf) {
    std::ostringstream f;
    f << "{ if (atomicCAS(p.err, 0, " << code << ") == 0) { p.err[1] = " << buf
      << "; LL* tr = (LL*)(p.err + 2); tr[0] = " << live << "LL;";
    for (int i = 0; i < niv; ++i) f << " tr[" << 1 + i << "] = i" << i << ";";
    f << " } return; }";
    return f.str();
  };
  auto address = [&](int32_t list_at, int b, int64_t row_extra = 0, int64_t col_extra = 0) {
    const VmBuf& vb = bt.at(b);
    const int32_t n = enc.lists.at(list_at);
    std::ostringstream s2;
    if (n != vb.rank) {
      s2 << fail(2, b);
      return std::make_pair(s2.str(), std::string("0"));
    }
    std::string off = "0LL";
    for (int d = 0; d < n; ++d) {
      std::string x = cexpr(enc.expr, enc.lists.at(list_at + 1 + d));
      (void)row_extra;
      (void)col_extra;
      s2 << "const LL x" << d << " = " << x << "; if (x" << d << " < 0 || x" << d << " >= "
         << vb.shape[d] << "LL) " << fail(1, b) << "\n";
      off = off + " + x" + std::to_string(d) + " * " + std::to_string(vb.stride[d]) + "LL";
    }
    return std::make_pair(s2.str(), off);
  };
  for (size_t pc = 0; pc < enc.code.size(); ++pc) {
    const Ins& in = enc.code[pc];
    switch (in.op) {
      case OP_LOOP:
        o << "    { const LL lb" << pc << " = " << list(in.b, "max") << "; const LL ub" << pc
          << " = " << list(in.c, "min") << ";\n    for (i" << in.a << " = lb" << pc << "; i" << in.a
          << " < ub" << pc << "; i" << in.a << " += " << in.d << "LL) {\n";
        live_stack.push_back(live);
        live |= 1u << in.a;
        break;
      case OP_END:
        o << "    } }\n";
        live = live_stack.back();
        live_stack.pop_back();
        break;
      case OP_IVVAL: o << "    r" << in.a << " = (double)i" << in.b << ";\n"; break;
      case OP_LOAD: {
        const auto [chk, off] = address(in.c, in.b);
        char buf[512];
        std::snprintf(buf, sizeof(buf), ld_expr(bt[in.b].type), ("P" + std::to_string(in.b)).c_str(),
                      "o_");
        o << "    { " << chk << " const LL o_ = " << off << "; r" << in.a << " = " << buf << "; }\n";
        break;
      }
      case OP_STORE: {
        const auto [chk, off] = address(in.c, in.b);
        const std::string v = "rt" + std::to_string(bt[in.b].type) + "(" + operand(in.a) + ")";
        o << "    { " << chk << " const LL o_ = " << off << "; "
          << st_stmt(bt[in.b].type, "P" + std::to_string(in.b), "o_", v) << " }\n";
        break;
      }
      case OP_ARITH: {
        const int kind = in.b & 0xff, cast = (in.b >> 8) & 0xff;
        const std::string x = in.c != INT32_MIN ? operand(in.c) : "0.0";
        const std::string y = in.d != INT32_MIN ? operand(in.d) : "0.0";
        const std::string z = in.e != INT32_MIN ? operand(in.e) : "0.0";
        if (fused[pc]) {  // f32 op + Round(F32) in one f32 instruction (see above)
          const Ins& nx = enc.code[pc + 1];
          const std::string fx = "(float)(" + x + ")", fy = "(float)(" + y + ")";
          std::string v;
          switch (static_cast<ArithOp>(kind)) {
            case ArithOp::Add: v = "__fadd_rn(" + fx + ", " + fy + ")"; break;
            case ArithOp::Sub: v = "__fsub_rn(" + fx + ", " + fy + ")"; break;
            case ArithOp::Mul: v = "__fmul_rn(" + fx + ", " + fy + ")"; break;
            case ArithOp::Div: v = "__fdiv_rn(" + fx + ", " + fy + ")"; break;
            default: v = "((" + x + ") < (" + y + ") ? " + fy + " : " + fx + ")"; break;  // Max
          }
          o << "    r" << nx.a << " = (double)(" << v << ");\n";
          ++pc;  // the Round is done
          break;
        }
        std::string v;
        switch (static_cast<ArithOp>(kind)) {
          case ArithOp::Add: v = "__dadd_rn(" + x + ", " + y + ")"; break;
          case ArithOp::Mul: v = "__dmul_rn(" + x + ", " + y + ")"; break;
          case ArithOp::Sub: v = "__dsub_rn(" + x + ", " + y + ")"; break;
          case ArithOp::Div: v = "__ddiv_rn(" + x + ", " + y + ")"; break;
          case ArithOp::Max: v = "((" + x + ") < (" + y + ") ? (" + y + ") : (" + x + "))"; break;
          case ArithOp::Exp: v = "exp(" + x + ")"; break;
          case ArithOp::Negate: v = "(-(" + x + "))"; break;
          case ArithOp::Cast:
            v = (cast == VT_I8 || cast == VT_I32)
                    ? "rt" + std::to_string(cast) + "(trunc(" + x + "))"
                    : "rt" + std::to_string(cast) + "(" + x + ")";
            break;
          case ArithOp::Fma: v = "__dadd_rn(__dmul_rn(" + x + ", " + y + "), " + z + ")"; break;
          case ArithOp::Select: v = "((" + x + ") != 0.0 ? (" + y + ") : (" + z + "))"; break;
          case ArithOp::CmpEq: v = "((" + x + ") == (" + y + ") ? 1.0 : 0.0)"; break;
          case ArithOp::CmpLt: v = "((" + x + ") < (" + y + ") ? 1.0 : 0.0)"; break;
          case ArithOp::CmpLe: v = "((" + x + ") <= (" + y + ") ? 1.0 : 0.0)"; break;
          case ArithOp::Quant:
            v = "fmin(fmax(round(__ddiv_rn(" + x + ", " + lit(in.imm) + ")), -128.0), 127.0)";
            break;
          case ArithOp::Dequant: v = "__dmul_rn(" + x + ", " + lit(in.imm) + ")"; break;
          case ArithOp::Round: v = "rt" + std::to_string(cast) + "(" + x + ")"; break;
        }
        o << "    r" << in.a << " = " << v << ";\n";
        break;
      }
      default: return "";  // fragment ops: interpreter only
    }
  }
  o << "  }\n}\n";
  return o.str();
}

struct Compiled {
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kern = nullptr;
};

// compile-once cache per (device, source)
cudaKernel_t get(const std::string& src) {
  static std::mutex mu;
  static std::map<std::pair<int, std::string>, Compiled> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_pair(dev, src);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second.kern;
  const Nvrtc& n = nvrtc();
  if (!n.ok) return nullptr;
  nvrtcProgram prog;
  if (n.create(&prog, src.c_str(), "afg_nest.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) return nullptr;
  const char* opts[] = {"--gpu-architecture=sm_100a", "-fmad=false", "--std=c++17"};
  const nvrtcResult r = n.compile(prog, 3, opts);
  Compiled c;
  if (r == NVRTC_SUCCESS) {
    size_t sz = 0;
    n.cubin_size(prog, &sz);
    std::vector<char> bin(sz);
    n.cubin(prog, bin.data());
    if (cudaLibraryLoadData(&c.lib, bin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) ==
            cudaSuccess &&
        cudaLibraryGetKernel(&c.kern, c.lib, "nest_jit") == cudaSuccess) {
      // compiled
    } else {
      cudaGetLastError();
      c.kern = nullptr;
    }
  } else {
    size_t ls = 0;
    n.log_size(prog, &ls);
    std::string log(ls, '\0');
    n.log(prog, log.data());
    std::fprintf(stderr, "afg nest jit: NVRTC failed (falling back to the interpreter):\n%s\n",
                 log.c_str());
  }
  n.destroy(&prog);
  cache[key] = c;
  return c.kern;
}

bool enabled() {
  static const bool on = [] {
    const char* e = getenv("AFG_NEST_JIT");
    return !(e && atoi(e) == 0);
  }();
  return on;
}

}  // namespace jit
}  // namespace

VmType vm_type(ElementType t) {
  switch (t) {
    case ElementType::F16: return VT_F16;
    case ElementType::BF16: return VT_BF16;
    case ElementType::I8: return VT_I8;
    case ElementType::I32: return VT_I32;
    default: return VT_F32;
  }
}

int vm_type_bytes(VmType t) {
  return t == VT_I8 ? 1 : (t == VT_F16 || t == VT_BF16) ? 2 : t == VT_F64 ? 8 : 4;
}

Linear linearize(const IndexExpr& e, const std::vector<std::string>& operands) {
  std::vector<Linear> st;
  const auto& c = e.code;
  for (size_t k = 0; k < c.size();) {
    const int64_t op = c[k++];
    switch (op) {
      case IndexExpr::Const: {
        Linear l;
        l.c = c[k++];
        st.push_back(l);
        break;
      }
      case IndexExpr::Dim: {
        Linear l;
        const int64_t d = c[k++];
        l.coef[d >= 0 && d < static_cast<int64_t>(operands.size()) ? operands[d] : "?"] = 1;
        st.push_back(l);
        break;
      }
      case IndexExpr::Add: {
        Linear b = st.back();
        st.pop_back();
        Linear& a = st.back();
        a.c += b.c;
        a.affine = a.affine && b.affine;
        for (const auto& [n, v] : b.coef) a.coef[n] += v;
        for (auto it = a.coef.begin(); it != a.coef.end();)
          it = it->second == 0 ? a.coef.erase(it) : std::next(it);
        break;
      }
      case IndexExpr::MulConst: {
        const int64_t f = c[k++];
        Linear& a = st.back();
        a.c *= f;
        for (auto& kv : a.coef) kv.second *= f;
        if (f == 0) a.coef.clear();
        break;
      }
      case IndexExpr::FloorDiv:
      case IndexExpr::Mod: {
        ++k;
        Linear& a = st.back();
        a.affine = false;
        break;
      }
      default: {
        Linear l;
        l.affine = false;
        return l;
      }
    }
  }
  if (st.size() != 1) {
    Linear l;
    l.affine = false;
    return l;
  }
  return st[0];
}

Runner::~Runner() {
  for (auto& kv : t_)
    if (kv.second.owned && kv.second.ptr) cudaFreeAsync(kv.second.ptr, s_);
  for (void* p : scratch_) cudaFreeAsync(p, s_);
  if (counters_) cudaFreeAsync(counters_, s_);
  if (err_) cudaFreeAsync(err_, s_);
  cudaStreamSynchronize(s_);
}

void Runner::sync(const char* what) {
  cudaError_t e = cudaStreamSynchronize(s_);
  if (e != cudaSuccess) throw InterpError(std::string("afg: ") + what + ": " + cudaGetErrorString(e));
}

DevTensor& Runner::alloc(const std::string& id, const std::vector<int64_t>& shape, ElementType et,
                         MemSpace space) {
  release(id);
  DevTensor d;
  d.type = vm_type(et);
  d.et = et;
  d.space = space;
  d.shape = shape;
  d.owned = true;
  const size_t bytes = static_cast<size_t>(std::max<int64_t>(d.numel(), 1)) * vm_type_bytes(d.type);
  cudaError_t e = cudaMallocAsync(&d.ptr, bytes + 16, s_);
  if (e != cudaSuccess)
    throw InterpError(std::string("afg: device allocation failed: ") + cudaGetErrorString(e));
  if (counters_) {
    counted_index_[id] = static_cast<int>(counted_.size());
    counted_.push_back(id);
  }
  return t_[id] = d;
}

DevTensor& Runner::bind(const std::string& id, void* ptr, const std::vector<int64_t>& shape,
                        ElementType et) {
  release(id);
  DevTensor d;
  d.ptr = ptr;
  d.type = vm_type(et);
  d.et = et;
  d.shape = shape;
  return t_[id] = d;
}

DevTensor& Runner::at(const std::string& id) {
  auto it = t_.find(id);
  if (it == t_.end()) throw InterpError("afg: tensor " + id + " not materialised");
  return it->second;
}

void Runner::release(const std::string& id) {
  auto it = t_.find(id);
  if (it == t_.end()) return;
  if (it->second.owned && it->second.ptr) cudaFreeAsync(it->second.ptr, s_);
  t_.erase(it);
}

void* Runner::scratch(size_t bytes) {
  void* p = nullptr;
  if (cudaMallocAsync(&p, bytes + 16, s_) != cudaSuccess)
    throw InterpError("afg: scratch allocation failed");
  scratch_.push_back(p);
  return p;
}

// Large pageable host <-> device copies (the graph API's inputs / outputs):
// the driver's own pageable path stages through pinned memory with one CPU
// memcpy on the calling thread (~10 GB/s). Here: two 64 MB pinned buffers per
// device; each chunk is copied by four threads on the host side and DMA'd on
// the stream, the next chunk's host copy overlapping the current DMA.
namespace {
constexpr size_t STAGE_CH = size_t(64) << 20;
struct Stage {
  char* buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
};
std::mutex g_stage_mu;  // one staged copy per process at a time
Stage g_stage[64];

Stage* stage_buffers() {
  static const bool off = [] {  // AFG_STAGED_COPY=0: the driver's pageable copies (A/B)
    const char* e = getenv("AFG_STAGED_COPY");
    return e && atoi(e) == 0;
  }();
  if (off) return nullptr;
  int dev = 0;
  cudaGetDevice(&dev);
  Stage& st = g_stage[dev & 63];
  for (int b = 0; b < 2; ++b) {
    if (!st.buf[b]) {
      if (cudaHostAlloc(reinterpret_cast<void**>(&st.buf[b]), STAGE_CH, cudaHostAllocDefault) !=
              cudaSuccess ||
          cudaEventCreateWithFlags(&st.ev[b], cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        st.buf[b] = nullptr;
        return nullptr;
      }
    }
  }
  return &st;
}

void par_memcpy(void* dst, const void* src, size_t len) {
  constexpr int T = 4;
  const size_t per = (len / T + 63) & ~size_t(63);
  std::thread th[T];
  for (int t = 0; t < T; ++t) {
    const size_t o = per * t;
    if (o >= len) break;
    const size_t l = std::min(per, len - o);
    th[t] = std::thread([=] { std::memcpy(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o, l); });
  }
  for (auto& x : th)
    if (x.joinable()) x.join();
}
}  // namespace

cudaError_t staged_h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_stage_mu);
  Stage* st = stage_buffers();
  if (!st) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s);
  size_t k = 0;
  for (size_t off = 0; off < bytes; off += STAGE_CH, ++k) {
    const int b = static_cast<int>(k & 1);
    const size_t len = std::min(STAGE_CH, bytes - off);
    cudaError_t e = cudaEventSynchronize(st->ev[b]);  // this buffer's previous DMA is done
    if (e != cudaSuccess) return e;
    par_memcpy(st->buf[b], static_cast<const char*>(src) + off, len);
    e = cudaMemcpyAsync(static_cast<char*>(dst) + off, st->buf[b], len, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaEventRecord(st->ev[b], s);
    if (e != cudaSuccess) return e;
  }
  return cudaEventSynchronize(st->ev[(k - 1) & 1]);  // the buffers are reused by the next call
}

cudaError_t staged_d2h(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_stage_mu);
  Stage* st = stage_buffers();
  if (!st) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s);
  const size_t n = (bytes + STAGE_CH - 1) / STAGE_CH;
  auto issue = [&](size_t k) {
    const size_t off = k * STAGE_CH;
    cudaError_t e = cudaMemcpyAsync(st->buf[k & 1], static_cast<const char*>(src) + off,
                                    std::min(STAGE_CH, bytes - off), cudaMemcpyDeviceToHost, s);
    return e == cudaSuccess ? cudaEventRecord(st->ev[k & 1], s) : e;
  };
  cudaError_t e = issue(0);
  for (size_t k = 0; k < n && e == cudaSuccess; ++k) {
    if (k + 1 < n) e = issue(k + 1);  // the next chunk's DMA overlaps this chunk's host copy
    if (e == cudaSuccess) e = cudaEventSynchronize(st->ev[k & 1]);
    if (e != cudaSuccess) break;
    const size_t off = k * STAGE_CH;
    par_memcpy(static_cast<char*>(dst) + off, st->buf[k & 1], std::min(STAGE_CH, bytes - off));
  }
  return e;
}

void Runner::upload(const std::string& id, const std::vector<double>& host) {
  upload(id, host.data(), static_cast<int64_t>(host.size()));
}

void Runner::upload(const std::string& id, const double* host, int64_t host_n) {
  DevTensor& d = at(id);
  const int64_t n = d.numel();
  if (host_n != n) throw InterpError("input shape mismatch for " + id);
  double* tmp = static_cast<double*>(scratch(static_cast<size_t>(n) * 8));
  const size_t bytes = static_cast<size_t>(n) * 8;
  cudaError_t e = cudaSuccess;
  if (bytes >= (size_t(32) << 20)) {
    e = staged_h2d(tmp, host, bytes, s_);
  } else {
    e = cudaMemcpyAsync(tmp, host, bytes, cudaMemcpyHostToDevice, s_);
  }
  if (e != cudaSuccess) throw InterpError(std::string("afg: upload failed: ") + cudaGetErrorString(e));
  f64_to_native_kernel<<<grid_for(n), 256, 0, s_>>>(tmp, static_cast<char*>(d.ptr), n, d.type);
  count_launch();
}

std::vector<double> Runner::download(const std::string& id) {
  DevTensor& d = at(id);
  const int64_t n = d.numel();
  double* tmp = static_cast<double*>(scratch(static_cast<size_t>(n) * 8));
  native_to_f64_kernel<<<grid_for(n), 256, 0, s_>>>(static_cast<const char*>(d.ptr), tmp, n,
                                                    d.type);
  count_launch();
  std::vector<double> h(static_cast<size_t>(n));
  const size_t bytes = static_cast<size_t>(n) * 8;
  cudaError_t e = bytes >= (size_t(32) << 20)
                      ? staged_d2h(h.data(), tmp, bytes, s_)
                      : cudaMemcpyAsync(h.data(), tmp, bytes, cudaMemcpyDeviceToHost, s_);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s_);
  if (e != cudaSuccess) throw InterpError(std::string("afg kernel failure: ") + cudaGetErrorString(e));
  return h;
}

void Runner::enable_counting(const std::vector<std::string>& order) {
  counted_ = order;
  counted_index_.clear();
  for (size_t i = 0; i < order.size(); ++i) counted_index_[order[i]] = static_cast<int>(i);
  const size_t n = C_PER_BUFFER + 4 * (order.size() + 4096);
  if (cudaMallocAsync(reinterpret_cast<void**>(&counters_), n * 8, s_) != cudaSuccess)
    throw InterpError("afg: counter allocation failed");
  cudaMemsetAsync(counters_, 0, n * 8, s_);
}

void Runner::fetch_metrics(gpu::NestMetrics* m) {
  if (!counters_ || !m) return;
  std::vector<unsigned long long> h(C_PER_BUFFER + 4 * counted_.size());
  cudaMemcpyAsync(h.data(), counters_, h.size() * 8, cudaMemcpyDeviceToHost, s_);
  sync("metrics");
  auto fill = [&](gpu::NestCounters& c, int at) {
    c.loads = static_cast<int64_t>(h[at]);
    c.stores = static_cast<int64_t>(h[at + 1]);
    c.loadBytes = static_cast<int64_t>(h[at + 2]);
    c.storeBytes = static_cast<int64_t>(h[at + 3]);
  };
  fill(m->global, C_GLOBAL);
  fill(m->shared, C_SHARED);
  fill(m->registers, C_REGISTER);
  m->flops = static_cast<int64_t>(h[C_FLOPS]);
  m->fragmentLoads = static_cast<int64_t>(h[C_FRAG_LOADS]);
  m->fragmentComputes = static_cast<int64_t>(h[C_FRAG_COMPUTES]);
  m->fragmentStores = static_cast<int64_t>(h[C_FRAG_STORES]);
  m->correctionOps = static_cast<int64_t>(h[C_CORRECTION]);
  for (size_t i = 0; i < counted_.size(); ++i)
    fill(m->perBuffer[counted_[i]], C_PER_BUFFER + 4 * static_cast<int>(i));
}

std::string Runner::run_vm(const NestOp& top, const std::map<std::string, int>& refcount) {
  // 1) candidate parallel levels: the perfectly nested constant-bound loops
  struct Level {
    std::string iv;
    int64_t lo, ext, step;
  };
  std::vector<Level> levels;
  const NestOp* cur = &top;
  while (cur->kind == NestOpKind::For || cur->kind == NestOpKind::Parallel) {
    bool ok = true;
    std::vector<Level> here;
    for (size_t i = 0; i < cur->ivs.size(); ++i) {
      int64_t lo = 0, hi = 0;
      if (!const_list(cur->lowers.at(i), true, &lo) || !const_list(cur->uppers.at(i), false, &hi)) {
        ok = false;
        break;
      }
      const int64_t st = cur->kind == NestOpKind::For ? cur->step : 1;
      here.push_back({cur->ivs[i], lo, hi > lo ? (hi - lo + st - 1) / st : 0, st});
    }
    if (!ok || levels.size() + here.size() > MAX_PAR) break;
    for (auto& l : here) levels.push_back(l);
    if (cur->body.size() == 1 &&
        (cur->body[0].kind == NestOpKind::For || cur->body[0].kind == NestOpKind::Parallel))
      cur = &cur->body[0];
    else
      break;
  }
  // 2) privatisable scratch buffers and the legal parallel prefix
  std::set<std::string> used;
  collect_buffers(top, used);
  std::set<std::string> priv;
  for (const auto& b : used) {
    auto it = t_.find(b);
    if (it == t_.end()) throw InterpError("unknown buffer " + b);
    auto rc = refcount.find(b);
    if (it->second.space != MemSpace::Global && rc != refcount.end() && rc->second <= 1)
      priv.insert(b);
  }
  std::vector<AccessRec> acc;
  collect_accesses(top, acc);
  size_t np = levels.size();
  for (; np > 0; --np) {
    std::vector<std::string> P;
    for (size_t i = 0; i < np; ++i) P.push_back(levels[i].iv);
    if (disjoint(acc, P, priv)) break;
  }
  if (np == 0) priv.clear();  // a single thread: scratch buffers are shared as declared
  // 3) encode: the per-thread program is what lies below the parallel levels
  Encoder enc;
  VmArgs a{};
  for (size_t i = 0; i < np; ++i) enc.iv_slot(levels[i].iv);
  if (np == 0) {
    enc.emit(top);
  } else {
    // find the body under the np-th level
    const NestOp* o = &top;
    size_t taken = 0;
    std::vector<const NestOp*> chain;
    while (true) {
      chain.push_back(o);
      taken += o->ivs.size();
      if (taken >= np) break;
      o = &o->body[0];
    }
    const NestOp* last = chain.back();
    if (taken == np) {
      for (const auto& c : last->body) enc.emit(c);
    } else {
      // np splits a Parallel op's ivs: emit its remaining ivs as loops
      NestOp rest = *last;
      const size_t skip = last->ivs.size() - (taken - np);
      rest.ivs.erase(rest.ivs.begin(), rest.ivs.begin() + skip);
      rest.lowers.erase(rest.lowers.begin(), rest.lowers.begin() + skip);
      rest.uppers.erase(rest.uppers.begin(), rest.uppers.begin() + skip);
      enc.emit(rest);
    }
  }
  // 4) device tables
  std::vector<VmBuf> bt;
  int64_t total = 1;
  for (size_t i = 0; i < np; ++i) {
    a.par_lo[i] = levels[i].lo;
    a.par_ext[i] = levels[i].ext;
    a.par_step[i] = levels[i].step;
    a.par_slot[i] = enc.iv.at(levels[i].iv);
    total *= levels[i].ext;
  }
  a.npar = static_cast<int32_t>(np);
  a.total = np == 0 ? 1 : total;
  std::ostringstream plan;
  plan << "nest_vm[" << (top.kindAttr().empty() ? "nest" : top.kindAttr()) << ", " << a.total
       << " threads x " << enc.code.size() << " ins]";
  if (a.total == 0) return plan.str();
  int64_t priv_bytes = 0;
  for (const auto& id : enc.bufs) {
    const DevTensor& d = at(id);
    VmBuf b{};
    b.ptr = static_cast<char*>(d.ptr);
    b.rank = static_cast<int32_t>(d.shape.size());
    if (b.rank > MAX_RANK) throw InterpError("afg nest vm: rank > 8");
    int64_t st = 1;
    for (int k = b.rank - 1; k >= 0; --k) {
      b.shape[k] = d.shape[k];
      b.stride[k] = st;
      st *= d.shape[k];
    }
    b.type = d.type;
    b.space = static_cast<int32_t>(d.space);
    auto ci = counted_index_.find(id);
    b.counter = ci == counted_index_.end() ? -1 : ci->second;
    if (priv.count(id)) {
      b.priv = d.numel();
      priv_bytes += d.numel() * vm_type_bytes(d.type);
    }
    bt.push_back(b);
  }
  // grid: enough threads to cover the points, bounded by private scratch
  int64_t threads = std::min<int64_t>(a.total, static_cast<int64_t>(num_sms()) * 8 * 128);
  if (priv_bytes > 0)
    threads = std::max<int64_t>(1, std::min<int64_t>(threads, (int64_t(256) << 20) / priv_bytes));
  const unsigned grid = static_cast<unsigned>((threads + 127) / 128);
  const int64_t thread_slots = static_cast<int64_t>(grid) * 128;
  for (size_t i = 0; i < bt.size(); ++i)
    if (bt[i].priv) {
      const DevTensor& d = at(enc.bufs[i]);
      bt[i].ptr = static_cast<char*>(
          scratch(static_cast<size_t>(thread_slots * d.numel() * vm_type_bytes(d.type))));
    }
  // one blob: code | expr | lists | consts | bufs
  auto align8 = [](size_t x) { return (x + 15) & ~size_t(15); };
  const size_t o_code = 0, n_code = enc.code.size() * sizeof(Ins);
  const size_t o_expr = align8(o_code + n_code), n_expr = enc.expr.size() * 8;
  const size_t o_list = align8(o_expr + n_expr), n_list = enc.lists.size() * 4;
  const size_t o_const = align8(o_list + n_list), n_const = enc.consts.size() * 8;
  const size_t o_buf = align8(o_const + n_const), n_buf = bt.size() * sizeof(VmBuf);
  const size_t total_bytes = align8(o_buf + n_buf) + 16;
  std::vector<char> blob(total_bytes, 0);
  std::memcpy(blob.data() + o_code, enc.code.data(), n_code);
  std::memcpy(blob.data() + o_expr, enc.expr.data(), n_expr);
  std::memcpy(blob.data() + o_list, enc.lists.data(), n_list);
  std::memcpy(blob.data() + o_const, enc.consts.data(), n_const);
  std::memcpy(blob.data() + o_buf, bt.data(), n_buf);
  char* dblob = static_cast<char*>(scratch(total_bytes));
  cudaError_t e = cudaMemcpyAsync(dblob, blob.data(), total_bytes, cudaMemcpyHostToDevice, s_);
  if (e != cudaSuccess) throw InterpError("afg nest vm: program upload failed");
  if (!err_) {
    if (cudaMallocAsync(reinterpret_cast<void**>(&err_), kErrBytes, s_) != cudaSuccess)
      throw InterpError("afg nest vm: allocation failed");
  }
  cudaMemsetAsync(err_, 0, kErrBytes, s_);
  a.code = reinterpret_cast<const Ins*>(dblob + o_code);
  a.expr = reinterpret_cast<const int64_t*>(dblob + o_expr);
  a.lists = reinterpret_cast<const int32_t*>(dblob + o_list);
  a.consts = reinterpret_cast<const double*>(dblob + o_const);
  a.bufs = reinterpret_cast<const VmBuf*>(dblob + o_buf);
  a.ncode = static_cast<int32_t>(enc.code.size());
  a.nbufs = static_cast<int32_t>(bt.size());
  a.counters = counters_;
  a.err = err_;
  const size_t nregs = enc.reg.size() + 1, nfrag = enc.frag.size();
  bool jitted = false;
  // big nests are compiled (NVRTC, cached): same semantics, no interpretation
  if (!counters_ && nfrag == 0 && bt.size() <= static_cast<size_t>(jit::MAX_BUFS) &&
      static_cast<double>(a.total) * static_cast<double>(enc.code.size()) >= kJitWork &&
      jit::enabled()) {
    const std::string src = jit::source(enc, bt, a);
    cudaKernel_t k = src.empty() ? nullptr : jit::get(src);
    if (k) {
      jit::JitArgs ja{};
      for (size_t i = 0; i < bt.size(); ++i) ja.ptr[i] = bt[i].ptr;
      ja.err = err_;
      ja.total = a.total;
      void* args[] = {&ja};
      e = cudaLaunchKernel(reinterpret_cast<const void*>(k), dim3(grid), dim3(128), args, 0, s_);
      count_launch();
      if (e != cudaSuccess) throw InterpError(std::string("afg nest jit launch: ") + cudaGetErrorString(e));
      jitted = true;
      plan << " jit";
    }
  }
  if (nfrag > 4) throw InterpError("afg nest vm: more than 4 live fragments");
  if (nfrag > 0 && nregs > 128) throw InterpError("afg nest vm: too many values with fragments");
  if (jitted) {
  } else if (nfrag > 0) {
    e = launch_vm<128, 4>(a, grid, s_);
  } else if (nregs <= 32) {
    e = launch_vm<32, 0>(a, grid, s_);
  } else if (nregs <= 128) {
    e = launch_vm<128, 0>(a, grid, s_);
  } else if (nregs <= 512) {
    e = launch_vm<512, 0>(a, grid, s_);
  } else {
    throw InterpError("afg nest vm: more than 512 live values in one nest");
  }
  if (!jitted) count_launch();
  if (e != cudaSuccess) throw InterpError(std::string("afg nest vm launch: ") + cudaGetErrorString(e));
  std::vector<int> herr(kErrBytes / 4, 0);
  e = cudaMemcpyAsync(herr.data(), err_, kErrBytes, cudaMemcpyDeviceToHost, s_);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s_);
  if (e != cudaSuccess) throw InterpError(std::string("afg kernel failure: ") + cudaGetErrorString(e));
  if (herr[0] != 0) {
    // "<what> [ivs: %i=3 ...]" like the interpreter's fail() (interp.cpp:258-266)
    const int64_t* t = reinterpret_cast<const int64_t*>(herr.data() + 2);
    std::map<std::string, int64_t> bound;
    for (const auto& [name, slot] : enc.iv)
      if (t[0] >> slot & 1) bound[name] = t[1 + slot];
    std::ostringstream msg;
    if (herr[0] == 1) msg << "out-of-bounds access to " << enc.bufs.at(herr[1]);
    else if (herr[0] == 2) msg << "rank mismatch on access to " << enc.bufs.at(herr[1]);
    else msg << "afg nest vm: bad instruction";
    msg << " [ivs:";
    for (const auto& [k, v] : bound) msg << " " << k << "=" << v;
    msg << "]";
    throw InterpError(msg.str());
  }
  plan << " over " << np << " parallel level(s)";
  return plan.str();
}

}  // namespace vm
}  // namespace afg
