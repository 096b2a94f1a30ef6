// nestexec.cpp - run_program: the B200 drop-in for af::interpret on a lowered
// program (interp.h:97-100; interp.cpp:164-236 for the buffer / input /
// output contract). Top-level nests are dispatched by their `kind` attribute
// and structure (classifyNestKind, analysis.cpp:1418; the conv.* attributes,
// frontend.cpp:952-968):
//   * kind=matmul nests with the lowering's exact shape (frame over C, init
//     store 0, k loop of load a / load b / load c / fma / store c; frontend.cpp
//     :679-733) run on the GEMM kernels: the fp32 SIMT kernel reproduces the
//     interpreter's sequential per-step f32 rounding; with tensor cores
//     enabled and operand values that are exactly bf16 / f16, on tcgen05;
//   * loop-form conv nests (conv.* attributes, not transposed) run on the
//     direct NCHW kernel, whose (ic, ky, kx) order and tap skipping are the
//     nest's;
//   * everything else (pointwise, broadcast, stencil, reductions, softmax's
//     four nests, fused nests with private buffers, orchestrated tiles with
//     fragments) runs on the nest VM (nestvm.cu).
// Metrics: VM nests count on the device like the interpreter; dispatched
// nests add the counts of the loop nest they replace, computed in closed form
// (the nest's trip counts are static), so InterpResult.metrics keeps its
// meaning on the fast paths.
#include <cuda_runtime.h>

#include <algorithm>
#include <set>
#include <sstream>

#include "../../include/afg.h"
#include "../../include/afg_nest.h"
#include "afg_internal.h"
#include "nestvm.h"

namespace afg {
namespace gpu {
namespace {

using vm::Linear;
using vm::linearize;

afg_dtype kdt(ElementType t) {
  return t == ElementType::F16 ? AFG_F16 : t == ElementType::BF16 ? AFG_BF16 : AFG_F32;
}
int width(ElementType t) {
  switch (t) {
    case ElementType::I8: return 1;
    case ElementType::F16:
    case ElementType::BF16: return 2;
    default: return 4;
  }
}

bool const_range(const NestOp& loop, int64_t* lo, int64_t* hi) {
  if (loop.kind != NestOpKind::For || loop.step != 1 || loop.lowers.size() != 1 ||
      loop.uppers.size() != 1 || loop.lowers[0].size() != 1 || loop.uppers[0].size() != 1)
    return false;
  const Linear l = linearize(loop.lowers[0][0], loop.boundOperands);
  const Linear u = linearize(loop.uppers[0][0], loop.boundOperands);
  if (!l.affine || !u.affine || !l.coef.empty() || !u.coef.empty()) return false;
  *lo = l.c;
  *hi = u.c;
  return true;
}

class ProgramRunner {
 public:
  ProgramRunner(const NestProgram& p, const NestRunOptions& o, NestMetrics* m, NestRunStats* st)
      : p_(p), opt_(o), m_(m), st_(st), R_(static_cast<cudaStream_t>(o.stream)) {}

  std::map<std::string, TensorValue> run(const std::map<std::string, TensorValue>& inputs) {
    if (afg_device_count() == 0)
      throw InterpError("afg: no sm_100 device visible (no CPU fallback)");
    std::vector<std::string> order;
    for (const auto& b : p_.buffers) order.push_back(b.id);
    if (m_) R_.enable_counting(order);
    for (const auto& b : p_.buffers) {
      auto& d = R_.alloc(b.id, b.shape, b.dtype, b.space);
      // the interpreter zero-initialises every buffer (interp.cpp:177-180)
      cudaMemsetAsync(d.ptr, 0, static_cast<size_t>(std::max<int64_t>(d.numel(), 1)) *
                                    vm::vm_type_bytes(d.type), R_.stream());
      decl_[b.id] = &b;
    }
    for (const auto& b : p_.buffers) {  // interp.cpp:202-213
      if (!b.isInput) continue;
      auto it = inputs.find(b.id);
      if (it == inputs.end()) throw InterpError("missing input for buffer " + b.id);
      if (it->second.shape != b.shape) throw InterpError("input shape mismatch for buffer " + b.id);
      R_.upload(b.id, it->second.values(), it->second.view ? it->second.numElements()
                                                            : static_cast<int64_t>(it->second.data.size()));
    }
    std::map<std::string, int> refs;
    for (const auto& top : p_.body) {
      std::set<std::string> used;
      collect(top, used);
      for (const auto& u : used) ++refs[u];
      if (top.kind == NestOpKind::For || top.kind == NestOpKind::Parallel) ++nests_;
    }
    // top-level straight-line code (e.g. mma_load / mma_compute / mma_store
    // at function scope) runs as one single-thread launch, so its SSA values
    // flow from op to op as in the interpreter
    NestOp seq;
    auto flush_seq = [&] {
      if (seq.body.empty()) return;
      seq.kind = NestOpKind::For;
      seq.ivs = {"$seq"};
      seq.lowers = {{IndexExpr::constant(0)}};
      seq.uppers = {{IndexExpr::constant(1)}};
      const std::string line = R_.run_vm(seq, refs);
      if (st_) st_->plan.push_back(line + " (function-scope ops)");
      seq = NestOp{};
    };
    for (const auto& top : p_.body) {
      if (top.kind != NestOpKind::For && top.kind != NestOpKind::Parallel) {
        seq.body.push_back(top);
        continue;
      }
      flush_seq();
      if (opt_.dispatch && (dispatch_matmul(top) || dispatch_conv(top))) continue;
      const std::string line = R_.run_vm(top, refs);
      if (st_) st_->plan.push_back(line);
    }
    flush_seq();
    std::map<std::string, TensorValue> out;
    for (const auto& b : p_.buffers) {
      if (!b.isOutput) continue;
      TensorValue v;
      v.shape = b.shape;
      v.type = b.dtype;
      v.data = R_.download(b.id);
      out.emplace(b.id, std::move(v));
    }
    if (m_) {
      R_.fetch_metrics(m_);
      for (const auto& b : p_.buffers) m_->perBufferSpace[b.id] = b.space;
      add_analytic();
      m_->nestCount = nests_;
    }
    R_.sync("program execution");
    return out;
  }

 private:
  const NestProgram& p_;
  NestRunOptions opt_;
  NestMetrics* m_;
  NestRunStats* st_;
  vm::Runner R_;
  std::map<std::string, const NestBuffer*> decl_;
  int64_t nests_ = 0;
  // closed-form counts of dispatched nests
  struct Analytic {
    std::string buf;
    int64_t loads = 0, stores = 0;
  };
  std::vector<Analytic> an_;
  int64_t an_flops_ = 0;

  static void collect(const NestOp& op, std::set<std::string>& used) {
    if (!op.buffer.empty()) used.insert(op.buffer);
    if (!op.srcBuffer.empty()) used.insert(op.srcBuffer);
    for (const auto& c : op.body) collect(c, used);
  }
  static void ok(afg_status st) {
    if (st != AFG_OK) throw InterpError(std::string("afg: ") + afg_last_error());
  }
  void plan(const std::string& s) {
    if (st_) st_->plan.push_back(s);
  }
  void add_analytic() {
    for (const auto& a : an_) {
      const NestBuffer& b = *decl_.at(a.buf);
      const int w = width(b.dtype);
      NestCounters& sp = b.space == MemSpace::Global ? m_->global
                         : b.space == MemSpace::Shared ? m_->shared
                                                       : m_->registers;
      NestCounters& pb = m_->perBuffer[a.buf];
      for (NestCounters* c : {&sp, &pb}) {
        c->loads += a.loads;
        c->stores += a.stores;
        c->loadBytes += a.loads * w;
        c->storeBytes += a.stores * w;
      }
    }
    m_->flops += an_flops_;
    an_.clear();
    an_flops_ = 0;
  }

  // The perfectly nested frame loops of a top-level nest: ivs and extents.
  struct Frame {
    std::vector<std::string> ivs;
    std::vector<int64_t> ext;
    const std::vector<NestOp>* body = nullptr;
  };
  static bool frame_of(const NestOp& top, Frame& f) {
    const NestOp* cur = &top;
    while (true) {
      int64_t lo, hi;
      if (!const_range(*cur, &lo, &hi) || lo != 0) return false;
      f.ivs.push_back(cur->ivs[0]);
      f.ext.push_back(hi);
      if (cur->body.size() == 1 && cur->body[0].kind == NestOpKind::For &&
          !cur->body[0].body.empty() && cur->body[0].body[0].kind == NestOpKind::For) {
        // descend only while the next level is still a frame loop (the k loop
        // of a matmul sits next to the init store, never alone)
        cur = &cur->body[0];
        continue;
      }
      if (cur->body.size() == 1 && cur->body[0].kind == NestOpKind::For) {
        cur = &cur->body[0];
        continue;
      }
      f.body = &cur->body;
      return true;
    }
  }

  // the iv (or constant 0) a result of an access must be
  static bool is_index(const Linear& l, const std::string& iv) {
    return iv.empty() ? l.is_const(0) : l.is_iv(iv);
  }

  // kind=matmul nests with the lowering's structure
  bool dispatch_matmul(const NestOp& top) {
    if (top.kindAttr() != "matmul" || top.attrs.count("conv.out")) return false;
    Frame f;
    if (!frame_of(top, f) || f.body->size() != 2) return false;
    const NestOp& init = (*f.body)[0];
    const NestOp& kl = (*f.body)[1];
    int64_t k0, K;
    if (init.kind != NestOpKind::Store || !init.operands.at(0).isImm ||
        init.operands[0].imm != 0.0 || !const_range(kl, &k0, &K) || k0 != 0 || kl.body.size() != 5)
      return false;
    const NestOp &la = kl.body[0], &lb = kl.body[1], &lc = kl.body[2], &fm = kl.body[3],
                 &sc = kl.body[4];
    if (la.kind != NestOpKind::Load || lb.kind != NestOpKind::Load || lc.kind != NestOpKind::Load ||
        fm.kind != NestOpKind::Arith || fm.arith != ArithOp::Fma || sc.kind != NestOpKind::Store)
      return false;
    if (fm.operands.size() != 3 || fm.operands[0].value != la.result ||
        fm.operands[1].value != lb.result || fm.operands[2].value != lc.result ||
        sc.operands.at(0).isImm || sc.operands[0].value != fm.result)
      return false;
    const std::string &A = la.buffer, &B = lb.buffer, &C = init.buffer;
    if (lc.buffer != C || sc.buffer != C || A == C || B == C) return false;
    if (!decl_.count(A) || !decl_.count(B) || !decl_.count(C)) return false;
    const NestBuffer *ad = decl_.at(A), *bd = decl_.at(B), *cd = decl_.at(C);
    const size_t r = cd->shape.size();
    if (r < 2 || ad->shape.size() != r || bd->shape.size() != r) return false;
    if (ad->space != MemSpace::Global || bd->space != MemSpace::Global ||
        cd->space != MemSpace::Global)
      return false;
    // C's index per dim: the frame iv of that dim (or 0 for extent 1)
    std::vector<std::string> civ(r);
    auto lin = [](const NestOp& o) {
      std::vector<Linear> v;
      for (const auto& e : o.access) v.push_back(linearize(e, o.accessOperands));
      return v;
    };
    const auto ci = lin(init), li = lin(lc), si = lin(sc), ai = lin(la), bi = lin(lb);
    if (ci.size() != r || li.size() != r || si.size() != r || ai.size() != r || bi.size() != r)
      return false;
    for (size_t d = 0; d < r; ++d) {
      if (ci[d].is_const(0) && cd->shape[d] == 1) continue;
      if (!ci[d].affine || ci[d].c != 0 || ci[d].coef.size() != 1 || ci[d].coef.begin()->second != 1)
        return false;
      civ[d] = ci[d].coef.begin()->first;
      if (std::find(f.ivs.begin(), f.ivs.end(), civ[d]) == f.ivs.end()) return false;
    }
    const std::string& kiv = kl.ivs[0];
    for (size_t d = 0; d < r; ++d) {
      if (!is_index(li[d], civ[d]) || !is_index(si[d], civ[d])) return false;
      if (d + 2 < r && (!is_index(ai[d], civ[d]) || !is_index(bi[d], civ[d]))) return false;
    }
    if (!is_index(ai[r - 2], civ[r - 2]) || !ai[r - 1].is_iv(kiv) || !bi[r - 2].is_iv(kiv) ||
        !is_index(bi[r - 1], civ[r - 1]))
      return false;
    const int64_t M = cd->shape[r - 2], N = cd->shape[r - 1];
    if (ad->shape[r - 1] != K || bd->shape[r - 2] != K) return false;
    int64_t batch = 1;
    for (size_t d = 0; d + 2 < r; ++d) batch *= cd->shape[d];
    // kernels: float operands of one type, f32 result (the SIMT kernel's
    // fmaf per k is the interpreter's round_f32(a*b + c))
    const bool fl = ad->dtype == bd->dtype &&
                    (ad->dtype == ElementType::F32 || ad->dtype == ElementType::F16 ||
                     ad->dtype == ElementType::BF16);
    if (!fl || cd->dtype != ElementType::F32) return false;
    const vm::DevTensor &Ad = R_.at(A), &Bd = R_.at(B), &Cd = R_.at(C);
    ok(afg_gemm_batched(Ad.ptr, Bd.ptr, Cd.ptr, batch, M, N, K, kdt(ad->dtype), AFG_F32,
                        R_.stream()));
    plan("afg_gemm_batched[gemm_simt " + std::to_string(batch) + "x" + std::to_string(M) + "x" +
         std::to_string(N) + "x" + std::to_string(K) + "] <- kind=matmul nest " + C);
    // the nest's counts: per (b, i, j): 1 init store, K x (3 loads, 1 store, fma)
    const int64_t pts = batch * M * N, fmas = pts * K;
    an_.push_back({A, fmas, 0});
    an_.push_back({B, fmas, 0});
    an_.push_back({C, fmas, pts + fmas});
    an_flops_ += 2 * fmas;
    return true;
  }

  // frame loops (constant, perfectly nested) whose body is exactly
  // [store 0 -> y, for ic { for ky { for kx { load x, load w, load y, fma, store y }}}]
  static bool lowered_conv_shape(const NestOp& top, const std::string& x, const std::string& w,
                                 const std::string& y) {
    const NestOp* cur = &top;
    while (cur->kind == NestOpKind::For && cur->body.size() == 1 &&
           cur->body[0].kind == NestOpKind::For)
      cur = &cur->body[0];
    if (cur->kind != NestOpKind::For || cur->body.size() != 2) return false;
    const NestOp& init = cur->body[0];
    if (init.kind != NestOpKind::Store || init.buffer != y || !init.operands.at(0).isImm) return false;
    const NestOp* l = &cur->body[1];
    for (int depth = 0; depth < 3; ++depth) {
      if (l->kind != NestOpKind::For || l->body.empty()) return false;
      if (depth < 2) {
        if (l->body.size() != 1) return false;
        l = &l->body[0];
      }
    }
    const auto& b = l->body;
    return b.size() == 5 && b[0].kind == NestOpKind::Load && b[0].buffer == x &&
           b[1].kind == NestOpKind::Load && b[1].buffer == w && b[2].kind == NestOpKind::Load &&
           b[2].buffer == y && b[3].kind == NestOpKind::Arith && b[3].arith == ArithOp::Fma &&
           b[4].kind == NestOpKind::Store && b[4].buffer == y;
  }

  // loop-form conv nests (conv.* attributes), not transposed, f32 result
  bool dispatch_conv(const NestOp& top) {
    auto attr = [&](const char* k) -> const NestAttr* {
      auto it = top.attrs.find(k);
      return it == top.attrs.end() ? nullptr : &it->second;
    };
    const NestAttr *in = attr("conv.in"), *w = attr("conv.w"), *out = attr("conv.out");
    if (!in || !w || !out || attr("conv.wflip") || attr("conv.wlayout")) return false;
    auto num = [&](const char* k) { const NestAttr* a = attr(k); return a ? a->i : -1; };
    const int64_t sy = num("conv.sy"), sx = num("conv.sx"), dy = num("conv.dy"),
                  dx = num("conv.dx"), py = num("conv.py"), px = num("conv.px"),
                  kh = num("conv.kh"), kw = num("conv.kw");
    if (std::min({sy, sx, dy, dx, kh, kw}) <= 0 || py < 0 || px < 0) return false;
    // the attributes survive later passes (tiling, fusion): only the lowering's
    // own loop form is dispatched -- frame loops over the output, then the
    // init store and the ic / ky / kx loops of load x, load w, load y, fma,
    // store y (frontend.cpp:905-950) -- with every buffer still declared
    auto dc = [&](const std::string& id) -> const NestBuffer* {
      auto it = decl_.find(id);
      return it == decl_.end() ? nullptr : it->second;
    };
    const NestBuffer *xd = dc(in->s), *wd = dc(w->s), *od = dc(out->s);
    if (!xd || !wd || !od || !lowered_conv_shape(top, in->s, w->s, out->s)) return false;
    if (xd->shape.size() != 4 || wd->shape.size() != 4 || od->shape.size() != 4) return false;
    const int64_t B = xd->shape[0], C = xd->shape[1], H = xd->shape[2], W = xd->shape[3];
    const int64_t OC = od->shape[1], OH = od->shape[2], OW = od->shape[3];
    // the unrolled (expression) form rounds once; only the loop form is the kernel's
    const bool loop_form = py > 0 || px > 0 || C * kh * kw > 8;
    const bool fl = xd->dtype == wd->dtype &&
                    (xd->dtype == ElementType::F32 || xd->dtype == ElementType::F16 ||
                     xd->dtype == ElementType::BF16);
    if (!loop_form || !fl || od->dtype != ElementType::F32 || wd->shape[0] != OC ||
        wd->shape[1] != C || wd->shape[2] != kh || wd->shape[3] != kw)
      return false;
    ok(afg_conv2d_nchw(R_.at(in->s).ptr, R_.at(w->s).ptr, R_.at(out->s).ptr, B, C, H, W, OC, kh,
                       kw, sy, sx, dy, dx, py, px, 0, OH, OW, kdt(xd->dtype), AFG_F32,
                       R_.stream()));
    plan("afg_conv2d_nchw[direct " + std::to_string(B) + "x" + std::to_string(C) + "x" +
         std::to_string(H) + "x" + std::to_string(W) + " k" + std::to_string(kh) + "x" +
         std::to_string(kw) + "] <- conv nest " + out->s);
    // counts: valid taps per output are separable in y and x
    auto valid = [](int64_t O, int64_t S, int64_t K, int64_t D, int64_t P, int64_t In) {
      int64_t t = 0;
      for (int64_t o = 0; o < O; ++o)
        for (int64_t k = 0; k < K; ++k) {
          const int64_t i = o * S + k * D - P;
          t += i >= 0 && i < In;
        }
      return t;
    };
    const int64_t taps = valid(OH, sy, kh, dy, py, H) * valid(OW, sx, kw, dx, px, W);
    const int64_t fmas = B * OC * C * taps, pts = B * OC * OH * OW;
    an_.push_back({in->s, fmas, 0});
    an_.push_back({w->s, fmas, 0});
    an_.push_back({out->s, fmas, pts + fmas});
    an_flops_ += 2 * fmas;
    return true;
  }
};

}  // namespace

std::map<std::string, TensorValue> run_program(const NestProgram& p,
                                               const std::map<std::string, TensorValue>& inputs,
                                               const NestRunOptions& opt, NestMetrics* metrics,
                                               NestRunStats* stats) {
  NestRunOptions o = opt;
  if (o.count_metrics && !metrics) o.count_metrics = false;
  ProgramRunner r(p, o, o.count_metrics ? metrics : nullptr, stats);
  auto out = r.run(inputs);
  return out;
}

}  // namespace gpu
}  // namespace afg
