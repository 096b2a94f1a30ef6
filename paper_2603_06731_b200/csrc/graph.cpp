// graph.cpp - the tensor-graph executor behind include/afg_graph.h: the B200
// drop-in for the reference's graph -> lowerGraphToAffine -> interpret path
// (frontend.cpp:975-979, interp.cpp:690-696).
//
// Pipeline
//  1. read: a small JSON reader builds the afg::gpu::TensorGraph mirror.
//  2. validate: one table of operator rules (arity + result-shape rule per
//     op) gives the reference's error behaviour: GraphError "unsupported-op",
//     "shape-mismatch", unknown / duplicate / use-before-produce tensors.
//  3. plan: a def-use DAG of the graph is matched against the fused patterns
//     the BASELINE configs are written in, independent of
//     op order in the JSON, checking on the DEVICE that the constant inputs
//     really are the constants the pattern assumes (zeros, GELU
//     coefficients, the [1, 0] softmax-selector mask, the causal -inf bias,
//     a uniform scale) and routing f32-declared tensors whose values are
//     exactly bf16 / f16 to the tensor cores:
//       matmul -> +bias [-> max(.,0) | -> tanh-GELU composite]  => K1 gemm_tc
//       transpose(k) -> batch_matmul -> [*scale] [+bias|causal] -> softmax ->
//         batch_matmul                                          => K3 attn_fwd
//       transpose(NHWC->NCHW) -> conv2d [-> +bias [-> max(.,0)]] ->
//         transpose(NCHW->NHWC)                                 => K2 conv_tc
//       dequantize x2 -> matmul [-> quantize]                   => K1c gemm_i8
//       i8 conv2d -> i32                                        => K1c conv
//  4. everything else runs on the nest VM (nestvm.cu) as fused regions: each
//     tensor that must exist in HBM (a graph output, or an input of a kernel
//     group) is one launch that recomputes its producer chain of pointwise /
//     broadcast / transpose / reshape / short-axis reduce and softmax ops in
//     registers, with the interpreter's arithmetic and rounding to every
//     intermediate's declared type (so a region is bit-exact to the unfused
//     interpretation). Large matmul / conv / softmax ops that are not part of
//     a pattern run on their dedicated kernels (float outputs) or on VM nests
//     that mirror the interpreter's per-step rounding (integer / half outputs).
// Device tensors live in their declared element type (i8 as int8, i32 as
// int32, f16, bf16, f32), so every stored value is the interpreter's value.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <functional>
#include <memory>
#include <set>
#include <sstream>
#include <unordered_map>

#include "../../include/afg.h"
#include "../../include/afg_graph.h"
#include "../../include/afg_multi.h"
#include "afg_internal.h"
#include "nestvm.h"

namespace afg {
namespace gpu {

// =============================================================== JSON ====
namespace json {

struct Value {
  enum Kind { Null, Bool, Number, String, Array, Object } kind = Null;
  bool b = false;
  double num = 0;
  std::string str;
  std::vector<Value> arr;
  std::vector<std::pair<std::string, Value>> obj;
  const Value* get(const std::string& k) const {
    for (const auto& kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
};

class Reader {
 public:
  explicit Reader(const std::string& s) : s_(s) {}
  Value document() {
    Value v = value();
    skip();
    if (p_ != s_.size()) bad("trailing characters");
    return v;
  }

 private:
  const std::string& s_;
  size_t p_ = 0;
  [[noreturn]] void bad(const char* what) {
    throw GraphError(std::string("graph json parse error: ") + what + " at offset " +
                     std::to_string(p_));
  }
  void skip() {
    while (p_ < s_.size() && std::isspace(static_cast<unsigned char>(s_[p_]))) ++p_;
  }
  bool take(char c) {
    skip();
    if (p_ < s_.size() && s_[p_] == c) {
      ++p_;
      return true;
    }
    return false;
  }
  std::string string_body() {
    std::string out;
    while (p_ < s_.size() && s_[p_] != '"') {
      char c = s_[p_++];
      if (c == '\\') {
        if (p_ >= s_.size()) bad("bad escape");
        const char e = s_[p_++];
        c = e == 'n' ? '\n' : e == 't' ? '\t' : e;
      }
      out += c;
    }
    if (p_ >= s_.size()) bad("unterminated string");
    ++p_;
    return out;
  }
  Value value() {
    skip();
    if (p_ >= s_.size()) bad("unexpected end");
    Value v;
    switch (s_[p_]) {
      case '{':
        ++p_;
        v.kind = Value::Object;
        if (take('}')) return v;
        do {
          skip();
          if (p_ >= s_.size() || s_[p_] != '"') bad("object key");
          ++p_;
          std::string key = string_body();
          if (!take(':')) bad("expected ':'");
          v.obj.emplace_back(std::move(key), value());
        } while (take(','));
        if (!take('}')) bad("expected '}'");
        return v;
      case '[':
        ++p_;
        v.kind = Value::Array;
        if (take(']')) return v;
        do v.arr.push_back(value());
        while (take(','));
        if (!take(']')) bad("expected ']'");
        return v;
      case '"':
        ++p_;
        v.kind = Value::String;
        v.str = string_body();
        return v;
      default: break;
    }
    static const struct {
      const char* word;
      Value::Kind kind;
      bool b;
    } kWords[] = {{"true", Value::Bool, true}, {"false", Value::Bool, false},
                  {"null", Value::Null, false}};
    for (const auto& w : kWords)
      if (s_.compare(p_, std::strlen(w.word), w.word) == 0) {
        p_ += std::strlen(w.word);
        v.kind = w.kind;
        v.b = w.b;
        return v;
      }
    const char* begin = s_.c_str() + p_;
    char* end = nullptr;
    v.num = std::strtod(begin, &end);
    if (end == begin) bad("unexpected character");
    p_ += static_cast<size_t>(end - begin);
    v.kind = Value::Number;
    return v;
  }
};

}  // namespace json

// ============================================================ graph API ===

// Lookups over the graph's tensor table and def-use sets.
namespace {
struct DefUse {
  std::set<std::string> produced, consumed;
  explicit DefUse(const TensorGraph& g) {
    for (const auto& op : g.ops) {
      produced.insert(op.output);
      consumed.insert(op.inputs.begin(), op.inputs.end());
    }
  }
};
}  // namespace

const TensorDesc* TensorGraph::find(const std::string& id) const {
  auto it = std::find_if(tensors.begin(), tensors.end(),
                         [&](const TensorDesc& t) { return t.id == id; });
  return it == tensors.end() ? nullptr : &*it;
}

std::vector<std::string> TensorGraph::inputIds() const {  // never produced by an op
  const DefUse du(*this);
  std::vector<std::string> ids;
  for (const auto& t : tensors)
    if (!du.produced.count(t.id)) ids.push_back(t.id);
  return ids;
}

std::vector<std::string> TensorGraph::outputIds() const {  // declared, else graph sinks
  if (!outputs.empty()) return outputs;
  const DefUse du(*this);
  std::vector<std::string> ids;
  for (const auto& t : tensors)
    if (du.produced.count(t.id) && !du.consumed.count(t.id)) ids.push_back(t.id);
  return ids;
}

namespace {

const std::map<std::string, ElementType>& dtype_names() {
  static const std::map<std::string, ElementType> m = {
      {"f32", ElementType::F32}, {"f16", ElementType::F16}, {"i8", ElementType::I8},
      {"i32", ElementType::I32}, {"bf16", ElementType::BF16}};
  return m;
}

std::vector<int64_t> ints_of(const json::Value& v, const char* what) {
  if (v.kind != json::Value::Array) throw GraphError(std::string("expected array for ") + what);
  std::vector<int64_t> out;
  out.reserve(v.arr.size());
  for (const auto& e : v.arr) {
    if (e.kind != json::Value::Number) throw GraphError(std::string("expected ints in ") + what);
    out.push_back(static_cast<int64_t>(e.num));
  }
  return out;
}

// "stride": 2 or [2, 1] -> (y, x)
void read_pair(const json::Value* v, int64_t& y, int64_t& x) {
  if (!v) return;
  if (v->kind == json::Value::Array && v->arr.size() >= 2) {
    y = static_cast<int64_t>(v->arr[0].num);
    x = static_cast<int64_t>(v->arr[1].num);
  } else {
    y = x = static_cast<int64_t>(v->num);
  }
}

const json::Value& field(const json::Value& o, const char* k) {
  const json::Value* v = o.get(k);
  if (!v) throw GraphError(std::string("graph json: missing key \"") + k + "\"");
  return *v;
}

}  // namespace

TensorGraph parseGraphJson(const std::string& text) {
  const json::Value doc = json::Reader(text).document();
  if (doc.kind != json::Value::Object || !doc.get("tensors") || !doc.get("ops"))
    throw GraphError("graph json must contain \"tensors\" and \"ops\"");
  TensorGraph g;
  for (const auto& t : doc.get("tensors")->arr) {
    TensorDesc d;
    d.id = field(t, "id").str;
    d.shape = ints_of(field(t, "shape"), "shape");
    const json::Value* dt = t.get("dtype");
    auto it = dtype_names().find(dt ? dt->str : "f32");
    if (it == dtype_names().end()) throw GraphError("unknown dtype for tensor " + d.id);
    d.dtype = it->second;
    g.tensors.push_back(std::move(d));
  }
  for (const auto& n : doc.get("ops")->arr) {
    TensorOpNode node;
    node.op = field(n, "op").str;
    for (const auto& in : field(n, "inputs").arr) node.inputs.push_back(in.str);
    node.output = field(n, "output").str;
    if (const json::Value* a = n.get("attrs")) {
      for (const auto& [key, v] : a->obj) {
        if (key == "perm") node.perm = ints_of(v, "perm");
        else if (key == "dims") node.dims = ints_of(v, "dims");
        else if (key == "stride") read_pair(&v, node.strideY, node.strideX);
        else if (key == "dilation") read_pair(&v, node.dilY, node.dilX);
        else if (key == "padding") node.samePadding = v.str == "same";
        else if (key == "transposed") node.transposed = v.b;
        else if (key == "op") node.reduceOp = v.str;
        else if (key == "axis") node.axis = static_cast<int64_t>(v.num);
        else if (key == "scale") node.scale = v.num;
      }
    }
    g.ops.push_back(std::move(node));
  }
  if (const json::Value* o = doc.get("outputs"))
    for (const auto& e : o->arr) g.outputs.push_back(e.str);
  return g;
}

namespace {

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// One spatial dimension of a conv: output extent and the begin pad. The
// window of one output spans (k-1)*dil+1 input positions; "same" keeps
// ceil(in/stride) outputs and puts the smaller half of the missing span in
// front (frontend.cpp:115-149 semantics); transposed convs invert the
// relation through the stride-stuffed input.
struct Window {
  int64_t out, pad;
};
Window conv_window(int64_t in, int64_t k, int64_t stride, int64_t dil, bool same,
                   bool transposed) {
  const int64_t span = (k - 1) * dil + 1;
  if (transposed) {
    if (!same) return {(in - 1) * stride + span, 0};
    const int64_t missing = span - stride;
    if (missing < 0)
      throw GraphError(
          "unsupported-op: transposed same-padding with stride exceeding the kernel span");
    return {in * stride, missing / 2};
  }
  if (!same) return {(in - span) / stride + 1, 0};
  const int64_t out = ceil_div(in, stride);
  return {out, std::max<int64_t>(0, (out - 1) * stride + span - in) / 2};
}

// ---- operator rules: arity and the shape of the result ----
struct RuleCtx {
  const TensorGraph& g;
  const TensorOpNode& n;
  const TensorDesc& in(size_t i) const {
    const TensorDesc* t = g.find(n.inputs.at(i));
    if (!t) throw GraphError("unknown tensor " + n.inputs.at(i));
    return *t;
  }
  const TensorDesc& out() const {
    const TensorDesc* t = g.find(n.output);
    if (!t) throw GraphError("unknown tensor " + n.output);
    return *t;
  }
  [[noreturn]] void mismatch(const std::string& why) const {
    throw GraphError("shape-mismatch: " + why + " (" + n.op + " -> " + n.output + ")");
  }
};
using ShapeRule = std::vector<int64_t> (*)(const RuleCtx&);
struct OpRule {
  int arity;
  ShapeRule shape;
};

std::vector<int64_t> same_shapes(const RuleCtx& c) {
  if (c.in(0).shape != c.in(1).shape) c.mismatch("elementwise operands differ");
  return c.in(0).shape;
}
std::vector<int64_t> like_input(const RuleCtx& c) { return c.in(0).shape; }
std::vector<int64_t> permuted(const RuleCtx& c) {
  const auto& s = c.in(0).shape;
  if (c.n.perm.size() != s.size()) c.mismatch("transpose perm rank");
  std::vector<int64_t> out;
  for (int64_t p : c.n.perm) {
    if (p < 0 || p >= static_cast<int64_t>(s.size())) c.mismatch("transpose perm entry");
    out.push_back(s[p]);
  }
  return out;
}
std::vector<int64_t> broadcast(const RuleCtx& c) {
  const auto& s = c.in(0).shape;
  const auto& o = c.out().shape;
  if (c.n.dims.size() != s.size()) c.mismatch("broadcast_in_dim dims rank");
  for (size_t d = 0; d < s.size(); ++d) {
    const int64_t to = c.n.dims[d];
    if (to < 0 || to >= static_cast<int64_t>(o.size()) || o[to] != s[d])
      c.mismatch("broadcast_in_dim extents");
  }
  return o;
}
std::vector<int64_t> reshaped(const RuleCtx& c) {
  auto count = [](const std::vector<int64_t>& s) {
    int64_t n = 1;
    for (int64_t d : s) n *= d;
    return n;
  };
  if (count(c.in(0).shape) != count(c.out().shape)) c.mismatch("reshape element count");
  return c.out().shape;
}
std::vector<int64_t> reduced(const RuleCtx& c) {
  const auto& s = c.in(0).shape;
  const int64_t r = static_cast<int64_t>(s.size());
  const int64_t axis = c.n.axis < 0 ? c.n.axis + r : c.n.axis;
  if (axis < 0 || axis >= r) c.mismatch("reduce axis out of range");
  std::vector<int64_t> out;
  for (int64_t d = 0; d < r; ++d)
    if (d != axis) out.push_back(s[d]);
  if (out.empty()) out.push_back(1);
  return out;
}
std::vector<int64_t> matmul2d(const RuleCtx& c) {
  const auto& a = c.in(0).shape;
  const auto& b = c.in(1).shape;
  if (a.size() != 2 || b.size() != 2 || a[1] != b[0]) c.mismatch("matmul operands");
  return {a[0], b[1]};
}
std::vector<int64_t> matmul_batched(const RuleCtx& c) {
  const auto& a = c.in(0).shape;
  const auto& b = c.in(1).shape;
  if (a.size() != b.size() || a.size() < 2) c.mismatch("batch_matmul rank");
  if (!std::equal(a.begin(), a.end() - 2, b.begin())) c.mismatch("batch_matmul batch dims");
  if (a.back() != b[b.size() - 2]) c.mismatch("batch_matmul contraction");
  std::vector<int64_t> out(a.begin(), a.end() - 1);
  out.push_back(b.back());
  return out;
}
std::vector<int64_t> conv_out(const RuleCtx& c) {
  const auto& x = c.in(0).shape;
  const auto& w = c.in(1).shape;
  if (x.size() != 4 || w.size() != 4) c.mismatch("conv2d operands must be rank 4");
  // weights OIHW, or IOHW when transposed
  const int64_t w_in = c.n.transposed ? w[0] : w[1], w_out = c.n.transposed ? w[1] : w[0];
  if (x[1] != w_in) c.mismatch("conv2d channel count");
  const Window wy = conv_window(x[2], w[2], c.n.strideY, c.n.dilY, c.n.samePadding, c.n.transposed);
  const Window wx = conv_window(x[3], w[3], c.n.strideX, c.n.dilX, c.n.samePadding, c.n.transposed);
  if (wy.out <= 0 || wx.out <= 0) c.mismatch("conv2d spatial dims not positive");
  return {x[0], w_out, wy.out, wx.out};
}

const std::map<std::string, OpRule>& op_rules() {
  static const std::map<std::string, OpRule> rules = {
      {"add", {2, same_shapes}},        {"sub", {2, same_shapes}},
      {"mul", {2, same_shapes}},        {"max", {2, same_shapes}},
      {"exp", {1, like_input}},         {"softmax", {1, like_input}},
      {"quantize", {1, like_input}},    {"dequantize", {1, like_input}},
      {"transpose", {1, permuted}},     {"broadcast_in_dim", {1, broadcast}},
      {"reshape", {1, reshaped}},       {"reduce", {1, reduced}},
      {"matmul", {2, matmul2d}},        {"batch_matmul", {2, matmul_batched}},
      {"conv2d", {2, conv_out}}};
  return rules;
}

}  // namespace

void validateGraph(const TensorGraph& g) {
  std::set<std::string> ids;
  for (const auto& t : g.tensors) {
    if (!ids.insert(t.id).second) throw GraphError("duplicate tensor id " + t.id);
    if (std::any_of(t.shape.begin(), t.shape.end(), [](int64_t d) { return d <= 0; }))
      throw GraphError("non-positive extent in tensor " + t.id);
  }
  const auto inputs = g.inputIds();
  std::set<std::string> ready(inputs.begin(), inputs.end());
  for (const auto& n : g.ops) {
    auto rule = op_rules().find(n.op);
    if (rule == op_rules().end()) throw GraphError("unsupported-op: " + n.op);
    if (static_cast<int>(n.inputs.size()) < rule->second.arity)
      throw GraphError("shape-mismatch: " + n.op + " needs " +
                       std::to_string(rule->second.arity) + " inputs");
    for (const auto& in : n.inputs) {
      if (!g.find(in)) throw GraphError("unknown tensor " + in);
      if (!ready.count(in)) throw GraphError("tensor " + in + " used before being produced");
    }
    const RuleCtx ctx{g, n};
    if (rule->second.shape(ctx) != ctx.out().shape)
      throw GraphError("shape-mismatch: " + n.output + " declared shape does not match op result");
    ready.insert(n.output);
  }
}

// ============================================================ executor ====
namespace {

using vm::DevTensor;

// ---- device probes of constant inputs ----
struct ProbeOut {
  int all_zero, all_bf16, all_f16, all_equal;
  double first;
};

template <typename T>
__device__ __forceinline__ float probe_ld(const T* p) {
  return static_cast<float>(*p);
}
template <>
__device__ __forceinline__ float probe_ld<__half>(const __half* p) {
  return __half2float(*p);
}
template <>
__device__ __forceinline__ float probe_ld<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(*p);
}

template <typename T>
__global__ void probe_kernel(const T* __restrict__ x, int64_t n, int* __restrict__ flags) {
  const float first = probe_ld(x);
  int zero = 1, bf = 1, hf = 1, eq = 1;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float v = probe_ld(x + i);
    uint32_t u;
    memcpy(&u, &v, 4);
    zero &= v == 0.0f;
    bf &= (u & 0xffffu) == 0u;
    hf &= __half2float(__float2half_rn(v)) == v;
    eq &= v == first;
  }
  zero = __syncthreads_and(zero);
  bf = __syncthreads_and(bf);
  hf = __syncthreads_and(hf);
  eq = __syncthreads_and(eq);
  if (threadIdx.x == 0) {
    if (!zero) atomicAnd(flags + 0, 0);
    if (!bf) atomicAnd(flags + 1, 0);
    if (!hf) atomicAnd(flags + 2, 0);
    if (!eq) atomicAnd(flags + 3, 0);
  }
}

// bias[b,h,i,j] == (j > i ? -inf : 0) over [BH, N, N]
__global__ void causal_probe_kernel(const float* __restrict__ x, int64_t bh, int64_t nq,
                                    int64_t nk, int* __restrict__ flag) {
  int ok = 1;
  const int64_t n = bh * nq * nk;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = i % nk, r = (i / nk) % nq;
    const float v = x[i];
    ok &= j > r ? (isinf(v) && v < 0.0f) : v == 0.0f;
  }
  ok = __syncthreads_and(ok);
  if (threadIdx.x == 0 && !ok) atomicAnd(flag, 0);
}

// mask[..., 2] == [1, 0]
__global__ void selector_probe_kernel(const float* __restrict__ x, int64_t pairs,
                                      int* __restrict__ flag) {
  int ok = 1;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < pairs;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    ok &= x[2 * i] == 1.0f && x[2 * i + 1] == 0.0f;
  ok = __syncthreads_and(ok);
  if (threadIdx.x == 0 && !ok) atomicAnd(flag, 0);
}

unsigned probe_grid(int64_t n) {
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8)));
}

afg_dtype kernel_dtype(ElementType t) {
  return t == ElementType::F16 ? AFG_F16 : t == ElementType::BF16 ? AFG_BF16 : AFG_F32;
}
bool is_float(ElementType t) {
  return t == ElementType::F32 || t == ElementType::F16 || t == ElementType::BF16;
}


std::string dims_str(const std::vector<int64_t>& s) {
  std::string r;
  for (size_t i = 0; i < s.size(); ++i) r += (i ? "x" : "") + std::to_string(s[i]);
  return r;
}

// A fused kernel group found by the planner.
struct Group {
  enum Kind { Gemm, Attention, ConvNHWC, QuantGemm, ConvI8 } kind;
  std::vector<int> ops;        // member op indices
  std::string out;             // the tensor the group materialises
  // GEMM / conv
  std::string a, b, bias, zeros, c1, c2, mask1, mask2;
  afg_epilogue epi = AFG_EPI_NONE;
  // attention
  std::string q, k, v, scale_t, bias_t;
  // quant
  double sa = 1, sb = 1, sc = 1;
  bool requant = false;
};

class Planner {
 public:
  Planner(const TensorGraph& g, const GpuOptions& o, ExecStats* st)
      : g_(g), opt_(o), stats_(st), R_(static_cast<cudaStream_t>(o.stream)) {}

  std::map<std::string, TensorValue> run(const std::map<std::string, TensorValue>& inputs) {
    // AFG_GRAPH_TIMING=1: host-side phase times on stderr (upload / plan +
    // launch / download), for the host-clock graph API measurements
    static const bool timing = [] {
      const char* e = getenv("AFG_GRAPH_TIMING");
      return e && atoi(e) != 0;
    }();
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    const auto t0 = now();
    validateGraph(g_);
    if (afg_device_count() == 0)
      throw InterpError("afg: no sm_100 device visible (no CPU fallback)");
    index();
    for (const auto& id : g_.inputIds()) {  // interp.cpp:202-213
      auto it = inputs.find("%" + id);
      if (it == inputs.end()) it = inputs.find(id);
      if (it == inputs.end()) throw InterpError("missing input %" + id);
      const TensorDesc* d = g_.find(id);
      if (it->second.shape != d->shape) throw InterpError("input shape mismatch for %" + id);
      R_.alloc(id, d->shape, d->dtype);
      R_.upload(id, it->second.values(), it->second.view ? it->second.numElements()
                                                          : static_cast<int64_t>(it->second.data.size()));
    }
    if (timing) R_.sync("upload");
    const auto t1 = now();
    if (opt_.fuse) find_groups();
    decide_inlining();
    for (size_t i = 0; i < g_.ops.size(); ++i) {
      const int gi = group_of_[i];
      if (gi >= 0) {
        if (static_cast<int>(i) == groups_[gi].ops.back()) run_group(groups_[gi]);
        continue;
      }
      if (!inline_[i]) materialise(static_cast<int>(i));
    }
    if (timing) R_.sync("graph execution");
    const auto t2 = now();
    std::map<std::string, TensorValue> out;
    for (const auto& id : g_.outputIds()) {
      const TensorDesc* d = g_.find(id);
      TensorValue v;
      v.shape = d->shape;
      v.type = d->dtype;
      v.data = R_.download(id);
      out["%" + id] = std::move(v);
    }
    R_.sync("graph execution");
    if (timing)
      fprintf(stderr, "afg graph timing: upload %.1f ms, plan+run %.1f ms, download %.1f ms\n",
              ms(t0, t1), ms(t1, t2), ms(t2, now()));
    return out;
  }

 private:
  const TensorGraph& g_;
  GpuOptions opt_;
  ExecStats* stats_;
  vm::Runner R_;
  std::map<std::string, int> producer_;
  std::map<std::string, std::vector<int>> consumers_;
  std::set<std::string> outputs_;
  std::vector<int> group_of_;
  std::vector<Group> groups_;
  std::vector<bool> inline_;
  std::map<std::string, ProbeOut> probes_;

  void plan(const std::string& line) {
    if (stats_) stats_->plan.push_back(line);
  }
  static void ok(afg_status st) {
    if (st != AFG_OK) throw InterpError(std::string("afg: ") + afg_last_error());
  }
  const TensorDesc& desc(const std::string& id) const { return *g_.find(id); }
  const TensorOpNode& op(int i) const { return g_.ops[i]; }

  void index() {
    for (size_t i = 0; i < g_.ops.size(); ++i) {
      producer_[g_.ops[i].output] = static_cast<int>(i);
      for (const auto& in : g_.ops[i].inputs) {
        auto& c = consumers_[in];
        if (c.empty() || c.back() != static_cast<int>(i)) c.push_back(static_cast<int>(i));
      }
    }
    for (const auto& id : g_.outputIds()) outputs_.insert(id);
    group_of_.assign(g_.ops.size(), -1);
    inline_.assign(g_.ops.size(), false);
  }

  // ---------------------------------------------------------- probes -----
  const ProbeOut& probe(const std::string& id) {
    auto it = probes_.find(id);
    if (it != probes_.end()) return it->second;
    DevTensor& d = R_.at(id);
    int* flags = static_cast<int*>(R_.scratch(16));
    const int ones[4] = {1, 1, 1, 1};
    cudaMemcpyAsync(flags, ones, 16, cudaMemcpyHostToDevice, R_.stream());
    const int64_t n = d.numel();
    ProbeOut p{0, 0, 0, 0, 0.0};
    if (is_float(d.et)) {
      if (d.type == vm::VT_F32)
        probe_kernel<float><<<probe_grid(n), 256, 0, R_.stream()>>>(
            static_cast<const float*>(d.ptr), n, flags);
      else if (d.type == vm::VT_F16)
        probe_kernel<__half><<<probe_grid(n), 256, 0, R_.stream()>>>(
            static_cast<const __half*>(d.ptr), n, flags);
      else
        probe_kernel<__nv_bfloat16><<<probe_grid(n), 256, 0, R_.stream()>>>(
            static_cast<const __nv_bfloat16*>(d.ptr), n, flags);
      count_launch();
      int h[4];
      float first = 0.0f;
      cudaMemcpyAsync(h, flags, 16, cudaMemcpyDeviceToHost, R_.stream());
      if (d.type == vm::VT_F32) cudaMemcpyAsync(&first, d.ptr, 4, cudaMemcpyDeviceToHost, R_.stream());
      R_.sync("probe");
      p = ProbeOut{h[0], h[1], h[2], h[3], first};
      if (d.type != vm::VT_F32) p.first = std::nan("");
    }
    return probes_[id] = p;
  }
  bool is_zero(const std::string& id) { return R_.has(id) && probe(id).all_zero; }
  // a uniform f32 tensor holding (float)value
  bool is_const(const std::string& id, double value, double* got = nullptr) {
    if (!R_.has(id) || desc(id).dtype != ElementType::F32) return false;
    const ProbeOut& p = probe(id);
    if (!p.all_equal) return false;
    if (got) *got = p.first;
    return std::isnan(value) || p.first == static_cast<float>(value);
  }
  bool flag_kernel(const std::function<void(int*)>& launch) {
    int* flag = static_cast<int*>(R_.scratch(4));
    const int one = 1;
    cudaMemcpyAsync(flag, &one, 4, cudaMemcpyHostToDevice, R_.stream());
    launch(flag);
    count_launch();
    int h = 0;
    cudaMemcpyAsync(&h, flag, 4, cudaMemcpyDeviceToHost, R_.stream());
    R_.sync("probe");
    return h != 0;
  }
  bool is_causal_bias(const std::string& id) {
    const TensorDesc& d = desc(id);
    if (d.dtype != ElementType::F32 || d.shape.size() != 4 || !R_.has(id)) return false;
    const int64_t bh = d.shape[0] * d.shape[1], nq = d.shape[2], nk = d.shape[3];
    if (nq != nk) return false;
    const float* x = static_cast<const float*>(R_.at(id).ptr);
    return flag_kernel([&](int* f) {
      causal_probe_kernel<<<probe_grid(bh * nq * nk), 256, 0, R_.stream()>>>(x, bh, nq, nk, f);
    });
  }
  bool is_selector(const std::string& id) {
    const TensorDesc& d = desc(id);
    if (d.dtype != ElementType::F32 || d.shape.empty() || d.shape.back() != 2 || !R_.has(id))
      return false;
    const float* x = static_cast<const float*>(R_.at(id).ptr);
    const int64_t pairs = R_.at(id).numel() / 2;
    return flag_kernel([&](int* f) {
      selector_probe_kernel<<<probe_grid(pairs), 256, 0, R_.stream()>>>(x, pairs, f);
    });
  }
  // device copy of an f32 tensor as bf16 / f16 (exact when the probe says so)
  void* narrowed(const std::string& id, afg_dtype to) {
    DevTensor& d = R_.at(id);
    void* p = R_.scratch(static_cast<size_t>(d.numel()) * 2);
    ok(afg_convert(d.ptr, p, d.numel(), AFG_F32, to, R_.stream()));
    return p;
  }
  // the tensor-core element type for a pair of f32 / f16 / bf16 operands, or F32
  afg_dtype tc_type(const std::vector<std::string>& ids) {
    if (!opt_.tensor_cores) return AFG_F32;
    ElementType t = desc(ids[0]).dtype;
    for (const auto& id : ids)
      if (desc(id).dtype != t) return AFG_F32;
    if (t == ElementType::F16) return AFG_F16;
    if (t == ElementType::BF16) return AFG_BF16;
    if (t != ElementType::F32) return AFG_F32;
    bool bf = true, hf = true;
    for (const auto& id : ids) {
      if (!R_.has(id)) return AFG_F32;
      const ProbeOut& p = probe(id);
      bf = bf && p.all_bf16;
      hf = hf && p.all_f16;
    }
    return bf ? AFG_BF16 : hf ? AFG_F16 : AFG_F32;
  }

  // ------------------------------------------------------- matching -----
  // the single consumer op of `id` (which must not be a graph output)
  int sole_use(const std::string& id) const {
    if (outputs_.count(id)) return -1;
    auto it = consumers_.find(id);
    if (it == consumers_.end() || it->second.size() != 1) return -1;
    return it->second[0];
  }
  bool internal_to(const std::string& id, const std::set<int>& members) const {
    if (outputs_.count(id)) return false;
    auto it = consumers_.find(id);
    if (it == consumers_.end()) return false;
    for (int c : it->second)
      if (!members.count(c)) return false;
    return true;
  }
  // the other operand of binary op i given one operand
  std::string other(int i, const std::string& x) const {
    const auto& in = op(i).inputs;
    if (in[0] == x) return in[1];
    if (in[1] == x) return in[0];
    return "";
  }
  bool f32(const std::string& id) const { return desc(id).dtype == ElementType::F32; }
  bool external(const std::string& id, int before) const {  // produced before op `before`
    auto it = producer_.find(id);
    return it == producer_.end() || it->second < before;
  }
  int find_consumer(const std::string& id, const char* opname,
                    const std::function<bool(int)>& pred = nullptr) const {
    auto it = consumers_.find(id);
    if (it == consumers_.end()) return -1;
    for (int c : it->second)
      if (op(c).op == opname && group_of_[c] < 0 && (!pred || pred(c))) return c;
    return -1;
  }

  void add_group(Group gr) {
    std::sort(gr.ops.begin(), gr.ops.end());
    const int gi = static_cast<int>(groups_.size());
    for (int i : gr.ops) group_of_[i] = gi;
    groups_.push_back(std::move(gr));
  }

  void find_groups() {
    for (size_t i = 0; i < g_.ops.size(); ++i) {
      if (group_of_[i] >= 0) continue;
      const std::string& o = op(static_cast<int>(i)).op;
      if (o == "matmul") match_quant_gemm(static_cast<int>(i)) || match_gemm(static_cast<int>(i));
      else if (o == "transpose") match_attention(static_cast<int>(i)) || match_nhwc_conv(static_cast<int>(i));
      else if (o == "conv2d") match_conv_i8(static_cast<int>(i));
    }
  }

  // matmul(a,b)->c ; broadcast_in_dim(bias,dims=[1])->bb ; add(c,bb)->cb ;
  // [max(cb, zeros)->y | tanh-GELU composite of cb -> y]
  bool match_gemm(int mm) {
    const TensorOpNode& m = op(mm);
    const std::string a = m.inputs[0], b = m.inputs[1], c = m.output;
    if (!is_float(desc(a).dtype) || desc(a).dtype != desc(b).dtype || !f32(c)) return false;
    Group gr;
    gr.kind = Group::Gemm;
    gr.a = a;
    gr.b = b;
    gr.ops = {mm};
    gr.out = c;
    const int ad = sole_use(c);
    if (ad >= 0 && op(ad).op == "add") {
      const std::string bb = other(ad, c);
      auto pb = producer_.find(bb);
      if (!bb.empty() && pb != producer_.end() && op(pb->second).op == "broadcast_in_dim" &&
          op(pb->second).dims == std::vector<int64_t>{1} && sole_use(bb) == ad &&
          group_of_[pb->second] < 0) {
        const std::string bias = op(pb->second).inputs[0];
        if (f32(bias) && f32(bb) && f32(op(ad).output) && external(bias, mm + 1)) {
          gr.bias = bias;
          gr.ops.push_back(pb->second);
          gr.ops.push_back(ad);
          gr.out = op(ad).output;
          gr.epi = AFG_EPI_BIAS;
          const std::string cb = gr.out;
          const int mx = sole_use(cb);
          if (mx >= 0 && op(mx).op == "max" && f32(op(mx).output)) {
            const std::string z = other(mx, cb);
            if (!z.empty() && z != cb && external(z, mm + 1) && is_zero(z)) {
              gr.zeros = z;
              gr.ops.push_back(mx);
              gr.out = op(mx).output;
              gr.epi = AFG_EPI_BIAS_RELU;
            }
          } else {
            match_gelu(cb, mm, gr);
          }
        }
      }
    }
    add_group(std::move(gr));
    return true;
  }

  // The tanh-GELU composite of SURVEY.md App. B on x = cb:
  //  x2 = x*x ; x3 = x2*x ; t = x3*c1 ; s = x + t ; u2 = s*c2 ;
  //  bu = broadcast(u2, [..., 2], dims [0, 1]) ; m = bu*mask ; sm = softmax(m, -1) ;
  //  sel = sm*mask ; sg = reduce_sum(sel, axis -1) ; y = x*sg
  // with c1 == 0.044715, c2 == 2 sqrt(2/pi) and mask == [1, 0]: y = x sigmoid(2u).
  void match_gelu(const std::string& x, int first, Group& gr) {
    auto bin = [&](const char* name, const std::string& p, const std::string& q) -> int {
      return find_consumer(p, name, [&](int c) { return other(c, p) == q; });
    };
    std::vector<int> ops;
    const int x2 = bin("mul", x, x);
    if (x2 < 0) return;
    const int x3 = bin("mul", op(x2).output, x);
    if (x3 < 0) return;
    const int t = find_consumer(op(x3).output, "mul");
    if (t < 0) return;
    const std::string c1 = other(t, op(x3).output);
    const int s = bin("add", x, op(t).output);
    if (s < 0) return;
    const int u2 = find_consumer(op(s).output, "mul");
    if (u2 < 0) return;
    const std::string c2 = other(u2, op(s).output);
    const int bu = find_consumer(op(u2).output, "broadcast_in_dim");
    if (bu < 0) return;
    const auto& xs = desc(x).shape;
    std::vector<int64_t> want_shape = xs;
    want_shape.push_back(2);
    std::vector<int64_t> want_dims;
    for (size_t d = 0; d < xs.size(); ++d) want_dims.push_back(static_cast<int64_t>(d));
    if (desc(op(bu).output).shape != want_shape || op(bu).dims != want_dims) return;
    const int mk = find_consumer(op(bu).output, "mul");
    if (mk < 0) return;
    const std::string mask1 = other(mk, op(bu).output);
    const int sm = find_consumer(op(mk).output, "softmax");
    const int64_t last = static_cast<int64_t>(want_shape.size()) - 1;
    if (sm < 0 || !(op(sm).axis == -1 || op(sm).axis == last)) return;
    const int sel = find_consumer(op(sm).output, "mul");
    if (sel < 0) return;
    const std::string mask2 = other(sel, op(sm).output);
    const int sg = find_consumer(op(sel).output, "reduce");
    if (sg < 0 || op(sg).reduceOp != "sum" || !(op(sg).axis == -1 || op(sg).axis == last)) return;
    const int y = bin("mul", x, op(sg).output);
    if (y < 0) return;
    ops = {x2, x3, t, s, u2, bu, mk, sm, sel, sg, y};
    std::set<int> members(gr.ops.begin(), gr.ops.end());
    members.insert(ops.begin(), ops.end());
    for (int i : ops) {
      if (!f32(op(i).output)) return;
      if (i != y && !internal_to(op(i).output, members)) return;
    }
    if (!internal_to(x, members)) return;
    for (const std::string& k : {c1, c2, mask1, mask2})
      if (k.empty() || !external(k, first + 1)) return;
    if (!is_const(c1, 0.044715) || !is_const(c2, 2.0 * std::sqrt(2.0 / M_PI)) ||
        !is_selector(mask1) || (mask2 != mask1 && !is_selector(mask2)))
      return;
    gr.ops.insert(gr.ops.end(), ops.begin(), ops.end());
    gr.c1 = c1;
    gr.c2 = c2;
    gr.mask1 = mask1;
    gr.mask2 = mask2;
    gr.out = op(y).output;
    gr.epi = AFG_EPI_BIAS_GELU_TANH;
  }

  // dequantize(qa)->a ; dequantize(qb)->b ; matmul(a,b)->c [; quantize(c)->q]
  bool match_quant_gemm(int mm) {
    const TensorOpNode& m = op(mm);
    auto dq = [&](const std::string& t) -> int {
      auto it = producer_.find(t);
      if (it == producer_.end() || op(it->second).op != "dequantize") return -1;
      if (desc(op(it->second).inputs[0]).dtype != ElementType::I8 || sole_use(t) != mm) return -1;
      return it->second;
    };
    const int da = dq(m.inputs[0]), db = dq(m.inputs[1]);
    if (da < 0 || db < 0 || !f32(m.output) || !f32(m.inputs[0]) || !f32(m.inputs[1])) return false;
    const int64_t K = desc(m.inputs[0]).shape[1];
    if (K >= 131072) return false;
    Group gr;
    gr.kind = Group::QuantGemm;
    gr.a = op(da).inputs[0];
    gr.b = op(db).inputs[0];
    gr.sa = op(da).scale;
    gr.sb = op(db).scale;
    gr.ops = {da, db, mm};
    gr.out = m.output;
    const int qz = sole_use(m.output);
    if (qz >= 0 && op(qz).op == "quantize" && desc(op(qz).output).dtype == ElementType::I8) {
      gr.sc = op(qz).scale;
      gr.requant = true;
      gr.ops.push_back(qz);
      gr.out = op(qz).output;
    }
    add_group(std::move(gr));
    return true;
  }

  // conv2d(i8, i8) -> i32 (the repositioned integer conv)
  bool match_conv_i8(int cv) {
    const TensorOpNode& n = op(cv);
    if (desc(n.inputs[0]).dtype != ElementType::I8 || desc(n.inputs[1]).dtype != ElementType::I8 ||
        desc(n.output).dtype != ElementType::I32 || n.transposed)
      return false;
    const int64_t C = desc(n.inputs[0]).shape[1];
    if (C % 16 != 0) return false;
    Group gr;
    gr.kind = Group::ConvI8;
    gr.a = n.inputs[0];
    gr.b = n.inputs[1];
    gr.ops = {cv};
    gr.out = n.output;
    add_group(std::move(gr));
    return true;
  }

  // transpose(k,[0,1,3,2])->kt ; batch_matmul(q,kt)->qk ; [mul(qk,S)->qs] ;
  // [add(.,bias)->qkb] ; softmax(.,-1)->soft ; batch_matmul(soft,v)->out
  bool match_attention(int tr) {
    const TensorOpNode& t = op(tr);
    const std::string k = t.inputs[0];
    if (desc(k).shape.size() != 4 || t.perm != std::vector<int64_t>{0, 1, 3, 2}) return false;
    const int qk = sole_use(t.output);
    if (qk < 0 || op(qk).op != "batch_matmul" || op(qk).inputs[1] != t.output ||
        op(qk).inputs[0] == t.output)
      return false;
    Group gr;
    gr.kind = Group::Attention;
    gr.q = op(qk).inputs[0];
    gr.k = k;
    gr.ops = {tr, qk};
    std::string s = op(qk).output;
    if (!f32(s)) return false;
    int nx = sole_use(s);
    if (nx >= 0 && op(nx).op == "mul") {
      const std::string sc = other(nx, s);
      if (sc.empty() || sc == s || !f32(op(nx).output) || !is_const(sc, std::nan(""))) return false;
      gr.scale_t = sc;
      gr.ops.push_back(nx);
      s = op(nx).output;
      nx = sole_use(s);
    }
    if (nx >= 0 && op(nx).op == "add") {
      const std::string bias = other(nx, s);
      if (bias.empty() || bias == s || !f32(bias) || !f32(op(nx).output)) return false;
      gr.bias_t = bias;
      gr.ops.push_back(nx);
      s = op(nx).output;
      nx = sole_use(s);
    }
    if (nx < 0 || op(nx).op != "softmax" || !(op(nx).axis == -1 || op(nx).axis == 3) ||
        !f32(op(nx).output))
      return false;
    gr.ops.push_back(nx);
    const int pv = sole_use(op(nx).output);
    if (pv < 0 || op(pv).op != "batch_matmul" || op(pv).inputs[0] != op(nx).output) return false;
    gr.ops.push_back(pv);
    gr.v = op(pv).inputs[1];
    gr.out = op(pv).output;
    const auto& qs = desc(gr.q).shape;
    const auto& vs = desc(gr.v).shape;
    if (desc(gr.q).dtype != desc(k).dtype || desc(gr.v).dtype != desc(k).dtype ||
        !is_float(desc(k).dtype) || qs.size() != 4 || vs[3] != qs[3] ||
        !is_float(desc(gr.out).dtype))
      return false;
    // every operand from outside the group must exist when the group runs
    const int last = *std::max_element(gr.ops.begin(), gr.ops.end());
    for (const std::string& x : {gr.q, gr.k, gr.v, gr.scale_t, gr.bias_t})
      if (!x.empty() && !external(x, last)) return false;
    (void)last;
    add_group(std::move(gr));
    return true;
  }

  // transpose(x,[0,3,1,2])->xt ; conv2d(xt,w)->c ; [broadcast(bias,dims[1])->bb ;
  // add(c,bb)->cb ; [max(cb,z)->r]] ; transpose(.,[0,2,3,1])->y
  bool match_nhwc_conv(int tr) {
    const TensorOpNode& t = op(tr);
    if (t.perm != std::vector<int64_t>{0, 3, 1, 2} || desc(t.inputs[0]).shape.size() != 4)
      return false;
    const int cv = sole_use(t.output);
    if (cv < 0 || op(cv).op != "conv2d" || op(cv).inputs[0] != t.output || op(cv).transposed)
      return false;
    Group gr;
    gr.kind = Group::ConvNHWC;
    gr.a = t.inputs[0];
    gr.b = op(cv).inputs[1];
    gr.ops = {tr, cv};
    std::string s = op(cv).output;
    if (!f32(s) || !f32(gr.a) || !f32(gr.b) || !f32(t.output)) return false;
    int nx = sole_use(s);
    if (nx >= 0 && op(nx).op == "add") {
      const std::string bb = other(nx, s);
      auto pb = producer_.find(bb);
      if (bb.empty() || pb == producer_.end() || op(pb->second).op != "broadcast_in_dim" ||
          op(pb->second).dims != std::vector<int64_t>{1} || sole_use(bb) != nx ||
          !f32(op(pb->second).inputs[0]) || !f32(bb) || !f32(op(nx).output))
        return false;
      gr.bias = op(pb->second).inputs[0];
      gr.ops.push_back(pb->second);
      gr.ops.push_back(nx);
      gr.epi = AFG_EPI_BIAS;
      s = op(nx).output;
      nx = sole_use(s);
      if (nx >= 0 && op(nx).op == "max" && f32(op(nx).output)) {
        const std::string z = other(nx, s);
        if (z.empty() || z == s || !R_.has(z) || !is_zero(z)) return false;
        gr.zeros = z;
        gr.ops.push_back(nx);
        gr.epi = AFG_EPI_BIAS_RELU;
        s = op(nx).output;
        nx = sole_use(s);
      }
    }
    if (nx < 0 || op(nx).op != "transpose" || op(nx).perm != std::vector<int64_t>{0, 2, 3, 1} ||
        !f32(op(nx).output))
      return false;
    gr.ops.push_back(nx);
    gr.out = op(nx).output;
    const int64_t C = desc(gr.a).shape[3];
    if (C % 64 != 0 || !R_.has(gr.a) || !R_.has(gr.b)) return false;
    if (!gr.bias.empty() && !R_.has(gr.bias)) return false;
    if (tc_type({gr.a, gr.b}) == AFG_F32) return false;  // exact f32 path: unfused ops
    add_group(std::move(gr));
    return true;
  }

  // ---------------------------------------------------- kernel groups -----
  void run_group(const Group& gr) {
    switch (gr.kind) {
      case Group::Gemm: run_gemm(gr); break;
      case Group::Attention: run_attention(gr); break;
      case Group::ConvNHWC: run_nhwc_conv(gr); break;
      case Group::QuantGemm: run_quant_gemm(gr); break;
      case Group::ConvI8: run_conv_i8(gr); break;
    }
    if (stats_) ++stats_->fused;
  }

  static const char* epi_name(afg_epilogue e) {
    switch (e) {
      case AFG_EPI_BIAS: return " +bias epilogue";
      case AFG_EPI_BIAS_RELU: return " +bias+relu epilogue";
      case AFG_EPI_BIAS_GELU_TANH: return " +bias+gelu(tanh) epilogue";
      case AFG_EPI_BIAS_GELU_ERF: return " +bias+gelu(erf) epilogue";
      default: return "";
    }
  }

  void run_gemm(const Group& gr) {
    const auto& as = desc(gr.a).shape;
    const int64_t M = as[0], K = as[1], N = desc(gr.b).shape[1];
    DevTensor& C = R_.alloc(gr.out, desc(gr.out).shape, ElementType::F32);
    const float* bias = gr.bias.empty() ? nullptr : static_cast<const float*>(R_.at(gr.bias).ptr);
    afg_dtype t = tc_type({gr.a, gr.b});
    const bool aligned = K % 8 == 0 && N % 8 == 0;
    std::string path = "simt f32";
    if (t != AFG_F32 && aligned) {
      const void* A = desc(gr.a).dtype == ElementType::F32 ? narrowed(gr.a, t) : R_.at(gr.a).ptr;
      const void* B = desc(gr.b).dtype == ElementType::F32 ? narrowed(gr.b, t) : R_.at(gr.b).ptr;
      ok(afg_gemm(A, K, B, N, bias, nullptr, C.ptr, N, M, N, K, t, AFG_F32, AFG_B_KN, gr.epi,
                  R_.stream()));
      path = t == AFG_BF16 ? "gemm_tc bf16" : "gemm_tc f16";
    } else {
      const afg_dtype ab = kernel_dtype(desc(gr.a).dtype);
      ok(afg_gemm(R_.at(gr.a).ptr, K, R_.at(gr.b).ptr, N, bias, nullptr, C.ptr, N, M, N, K, ab,
                  AFG_F32, AFG_B_KN, gr.epi, R_.stream()));
      path = ab == AFG_F32 ? "gemm_simt f32" : "gemm_simt";
    }
    plan("afg_gemm[" + path + " " + std::to_string(M) + "x" + std::to_string(N) + "x" +
         std::to_string(K) + "]" + epi_name(gr.epi) + " <- " + std::to_string(gr.ops.size()) +
         " ops -> " + gr.out);
  }

  void run_attention(const Group& gr) {
    const auto& qs = desc(gr.q).shape;
    const int64_t B = qs[0], H = qs[1], Nq = qs[2], D = qs[3], Nk = desc(gr.k).shape[2];
    float scale = 1.0f;
    std::string note;
    std::vector<std::string> pending;  // ops the kernel does not absorb
    if (!gr.scale_t.empty()) {
      double s = 0;
      if (!is_const(gr.scale_t, std::nan(""), &s))
        throw InterpError("afg: attention scale tensor is not uniform");  // planner guarantees
      scale = static_cast<float>(s);
      note += " scale";
    }
    int causal = 0;
    const float* bias = nullptr;
    if (!gr.bias_t.empty()) {
      if (is_causal_bias(gr.bias_t)) {
        causal = 1;
        note += " causal";
      } else if (!is_zero(gr.bias_t)) {
        bias = static_cast<const float*>(R_.at(gr.bias_t).ptr);
        note += " +bias";
      }
    }
    const ElementType et = desc(gr.q).dtype;
    afg_dtype t = kernel_dtype(et);
    const void *Q = R_.at(gr.q).ptr, *K = R_.at(gr.k).ptr, *V = R_.at(gr.v).ptr;
    if (et == ElementType::F32 && (D == 64 || D == 128)) {
      const afg_dtype n = tc_type({gr.q, gr.k, gr.v});
      if (n != AFG_F32) {
        Q = narrowed(gr.q, n);
        K = narrowed(gr.k, n);
        V = narrowed(gr.v, n);
        t = n;
      }
    }
    DevTensor& O = R_.alloc(gr.out, desc(gr.out).shape, desc(gr.out).dtype);
    ok(afg_attention_fwd(Q, K, V, bias, O.ptr, B, H, Nq, Nk, D, scale, causal, t,
                         kernel_dtype(desc(gr.out).dtype), R_.stream()));
    const bool tc = t != AFG_F32 && (D == 64 || D == 128);
    plan(std::string("afg_attention_fwd[") + (tc ? "attn_fwd tcgen05 " : "attn_simt ") +
         dims_str(qs) + "]" + note + " <- " + std::to_string(gr.ops.size()) + " ops -> " + gr.out);
  }

  void run_nhwc_conv(const Group& gr) {
    const auto& xs = desc(gr.a).shape;  // NHWC
    const auto& ws = desc(gr.b).shape;  // OIHW
    const TensorOpNode& cv = op(gr.ops[1]);
    const int64_t B = xs[0], H = xs[1], W = xs[2], C = xs[3], OC = ws[0], KH = ws[2], KW = ws[3];
    const Window wy = conv_window(H, KH, cv.strideY, cv.dilY, cv.samePadding, false);
    const Window wx = conv_window(W, KW, cv.strideX, cv.dilX, cv.samePadding, false);
    const afg_dtype t = tc_type({gr.a, gr.b});
    void* x = narrowed(gr.a, t);
    void* w_oihw = narrowed(gr.b, t);
    void* w = R_.scratch(static_cast<size_t>(OC * C * KH * KW) * 2);
    ok(afg_conv_pack_filter(w_oihw, w, OC, C, KH, KW, t, R_.stream()));
    DevTensor& Y = R_.alloc(gr.out, desc(gr.out).shape, ElementType::F32);
    const float* bias = gr.bias.empty() ? nullptr : static_cast<const float*>(R_.at(gr.bias).ptr);
    ok(afg_conv2d_nhwc_ex(x, w, bias, Y.ptr, B, H, W, C, OC, KH, KW, cv.strideY, cv.strideX,
                          wy.pad, wx.pad, cv.dilY, cv.dilX, wy.out, wx.out, t, AFG_F32, gr.epi,
                          R_.stream()));
    plan("afg_conv2d_nhwc[conv_tc " + std::string(t == AFG_BF16 ? "bf16 " : "f16 ") +
         dims_str(xs) + " k" + std::to_string(KH) + "x" + std::to_string(KW) + " s" +
         std::to_string(cv.strideY) + "]" + epi_name(gr.epi) + " <- " +
         std::to_string(gr.ops.size()) + " ops -> " + gr.out);
  }

  void run_quant_gemm(const Group& gr) {
    const auto& as = desc(gr.a).shape;
    const int64_t M = as[0], K = as[1], N = desc(gr.b).shape[1];
    const int64_t Kp = (K + 15) / 16 * 16;
    // operands: A [M, Kp] and B^T [N, Kp] int8 (zero-padded K), via the VM
    int8_t* a8 = static_cast<int8_t*>(R_.scratch(static_cast<size_t>(M * Kp)));
    int8_t* b8 = static_cast<int8_t*>(R_.scratch(static_cast<size_t>(N * Kp)));
    pack_i8(gr.a, a8, M, K, Kp, false);
    pack_i8(gr.b, b8, K, N, Kp, true);
    const ElementType ot = desc(gr.out).dtype;
    DevTensor& C = R_.alloc(gr.out, desc(gr.out).shape, ot);
    const double scale = gr.sa * gr.sb / (gr.requant ? gr.sc : 1.0);
    ok(afg_gemm_i8(a8, Kp, b8, Kp, C.ptr, N, M, N, Kp, gr.requant ? 1 : 2,
                   static_cast<float>(scale), R_.stream()));
    plan("afg_gemm_i8[" + std::to_string(M) + "x" + std::to_string(N) + "x" + std::to_string(K) +
         (gr.requant ? "] dequant.matmul.quant repositioned" : "] dequant.matmul repositioned") +
         " <- " + std::to_string(gr.ops.size()) + " ops -> " + gr.out);
  }

  void run_conv_i8(const Group& gr) {
    const TensorOpNode& cv = op(gr.ops[0]);
    const auto& xs = desc(gr.a).shape;  // NCHW
    const auto& ws = desc(gr.b).shape;  // OIHW
    const int64_t B = xs[0], C = xs[1], H = xs[2], W = xs[3], OC = ws[0], KH = ws[2], KW = ws[3];
    const Window wy = conv_window(H, KH, cv.strideY, cv.dilY, cv.samePadding, false);
    const Window wx = conv_window(W, KW, cv.strideX, cv.dilX, cv.samePadding, false);
    // NCHW -> NHWC, OIHW -> OHWI (int8), through the VM's exact copies
    int8_t* x = static_cast<int8_t*>(R_.scratch(static_cast<size_t>(B * H * W * C)));
    int8_t* w = static_cast<int8_t*>(R_.scratch(static_cast<size_t>(OC * KH * KW * C)));
    permute_into(gr.a, x, {0, 2, 3, 1});
    permute_into(gr.b, w, {0, 2, 3, 1});
    int32_t* y = static_cast<int32_t*>(R_.scratch(static_cast<size_t>(B * wy.out * wx.out * OC) * 4));
    ok(afg_conv2d_nhwc_i8(x, w, y, B, H, W, C, OC, KH, KW, cv.strideY, cv.strideX, wy.pad, wx.pad,
                          cv.dilY, cv.dilX, wy.out, wx.out, 0, 1.0f, R_.stream()));
    // NHWC i32 -> NCHW output tensor
    R_.bind("$conv_i8_nhwc", y, {B, wy.out, wx.out, OC}, ElementType::I32);
    R_.alloc(gr.out, desc(gr.out).shape, ElementType::I32);
    run_copy_permuted("$conv_i8_nhwc", gr.out, {0, 3, 1, 2});
    R_.release("$conv_i8_nhwc");
    plan("afg_conv2d_nhwc_i8[" + dims_str(xs) + " k" + std::to_string(KH) + "x" +
         std::to_string(KW) + "] i8 conv on K1c -> " + gr.out);
  }

  // copies src (graph tensor) into an int8 scratch [rows, Kp] (or its
  // transpose), zero-filling the K padding, on the VM
  void pack_i8(const std::string& src, int8_t* dst, int64_t rows, int64_t cols, int64_t Kp,
               bool transpose) {
    const std::string id = "$pack_" + src;
    if (!transpose) {
      R_.bind(id, dst, {rows, Kp}, ElementType::I8);
      cudaMemsetAsync(dst, 0, static_cast<size_t>(rows * Kp), R_.stream());
      NestBuilder nb(*this);
      nb.frame({rows, cols});
      const std::string v = nb.load(src, {nb.iv(0), nb.iv(1)});
      nb.store(id, v, {nb.iv(0), nb.iv(1)});
      R_.run_vm(nb.finish(), {});
    } else {  // src [K = rows, N = cols] -> dst [N, Kp]
      R_.bind(id, dst, {cols, Kp}, ElementType::I8);
      cudaMemsetAsync(dst, 0, static_cast<size_t>(cols * Kp), R_.stream());
      NestBuilder nb(*this);
      nb.frame({cols, rows});
      const std::string v = nb.load(src, {nb.iv(1), nb.iv(0)});
      nb.store(id, v, {nb.iv(0), nb.iv(1)});
      R_.run_vm(nb.finish(), {});
    }
    R_.release(id);
  }
  void permute_into(const std::string& src, void* dst, const std::vector<int64_t>& perm) {
    const auto& s = R_.at(src).shape;
    std::vector<int64_t> os;
    for (int64_t p : perm) os.push_back(s[p]);
    const std::string id = "$perm_" + src;
    R_.bind(id, dst, os, R_.at(src).et);
    run_copy_permuted(src, id, perm);
    R_.release(id);
  }
  // dst[d...] = src[...] with dst dim d = src dim perm[d]
  void run_copy_permuted(const std::string& src, const std::string& dst,
                         const std::vector<int64_t>& perm) {
    NestBuilder nb(*this);
    nb.frame(R_.at(dst).shape);
    std::vector<gpu::IndexExpr> in(perm.size());
    for (size_t d = 0; d < perm.size(); ++d) in[perm[d]] = nb.iv(static_cast<int>(d));
    const std::string v = nb.load(src, in);
    std::vector<gpu::IndexExpr> out;
    for (size_t d = 0; d < perm.size(); ++d) out.push_back(nb.iv(static_cast<int>(d)));
    nb.store(dst, v, out);
    R_.run_vm(nb.finish(), {});
  }

  // ------------------------------------------------------ VM regions -----
  // Builds one top-level nest: frame loops over a shape, then a body.
  class NestBuilder {
   public:
    explicit NestBuilder(Planner& p) : p_(p) {}
    void frame(const std::vector<int64_t>& shape) {
      shape_ = shape;
      if (shape_.empty()) {  // rank-0 tensor: one point, accesses have no results
        shape_ = {1};
        scalar_ = true;
      }
      for (size_t d = 0; d < shape.size(); ++d) ivs_.push_back("$p" + std::to_string(d));
      scopes_.emplace_back();
    }
    gpu::IndexExpr iv(int d) const { return gpu::IndexExpr::dim(d); }
    bool scalar_ = false;
    std::string fresh() { return "$v" + std::to_string(n_++); }
    std::vector<gpu::NestOp>& cur() { return stack_.empty() ? body_ : stack_.back().body; }
    std::string load(const std::string& buf, const std::vector<gpu::IndexExpr>& at) {
      gpu::NestOp o;
      o.kind = gpu::NestOpKind::Load;
      o.buffer = buf;
      o.access = at;
      o.accessOperands = ivs_;
      o.result = fresh();
      cur().push_back(o);
      return o.result;
    }
    void store(const std::string& buf, const std::string& v, const std::vector<gpu::IndexExpr>& at) {
      gpu::NestOp o;
      o.kind = gpu::NestOpKind::Store;
      o.buffer = buf;
      o.access = at;
      o.accessOperands = ivs_;
      o.operands = {gpu::NestOperand::val(v)};
      cur().push_back(o);
    }
    std::string arith(gpu::ArithOp k, std::vector<gpu::NestOperand> ops, double scale = 1.0,
                      ElementType cast = ElementType::F32, const std::string& into = "") {
      gpu::NestOp o;
      o.kind = gpu::NestOpKind::Arith;
      o.arith = k;
      o.operands = std::move(ops);
      o.scale = scale;
      o.castType = cast;
      o.result = into.empty() ? fresh() : into;
      cur().push_back(o);
      return o.result;
    }
    std::string round(const std::string& v, ElementType t, const std::string& into = "") {
      return arith(gpu::ArithOp::Round, {gpu::NestOperand::val(v)}, 1.0, t, into);
    }
    // opens `for r in [0, extent)`; returns the iv's operand position
    int open_loop(int64_t extent) {
      gpu::NestOp o;
      o.kind = gpu::NestOpKind::For;
      const std::string name = "$r" + std::to_string(n_++);
      o.ivs = {name};
      o.lowers = {{gpu::IndexExpr::constant(0)}};
      o.uppers = {{gpu::IndexExpr::constant(extent)}};
      stack_.push_back(o);
      ivs_.push_back(name);
      scopes_.emplace_back();
      return static_cast<int>(ivs_.size()) - 1;
    }
    void close_loop() {
      gpu::NestOp o = std::move(stack_.back());
      stack_.pop_back();
      scopes_.pop_back();
      cur().push_back(std::move(o));
    }
    // value memo per loop scope (a value computed inside a loop is only
    // valid in that iteration)
    const std::string* memo(const std::string& key) const {
      for (auto it = scopes_.rbegin(); it != scopes_.rend(); ++it) {
        auto f = it->find(key);
        if (f != it->end()) return &f->second;
      }
      return nullptr;
    }
    void remember(const std::string& key, const std::string& v) { scopes_.back()[key] = v; }
    gpu::NestOp finish() {
      // wrap the body in the frame loops, outermost first
      std::vector<gpu::NestOp> inner = std::move(body_);
      for (int d = static_cast<int>(shape_.size()) - 1; d >= 0; --d) {
        gpu::NestOp f;
        f.kind = gpu::NestOpKind::For;
        f.ivs = {"$p" + std::to_string(d)};
        f.lowers = {{gpu::IndexExpr::constant(0)}};
        f.uppers = {{gpu::IndexExpr::constant(shape_[d])}};
        f.body = std::move(inner);
        inner.clear();
        inner.push_back(std::move(f));
      }
      return std::move(inner[0]);
    }
    size_t depth() const { return ivs_.size(); }

   private:
    Planner& p_;
    std::vector<int64_t> shape_;
    std::vector<std::string> ivs_;
    std::vector<gpu::NestOp> body_;
    std::vector<gpu::NestOp> stack_;
    std::vector<std::map<std::string, std::string>> scopes_;
    int n_ = 0;
  };

  static std::string key_of(const std::string& id, const std::vector<gpu::IndexExpr>& at) {
    std::ostringstream k;
    k << id;
    for (const auto& e : at) {
      k << '|';
      for (int64_t w : e.code) k << w << ',';
    }
    return k.str();
  }
  static gpu::IndexExpr add(const gpu::IndexExpr& a, const gpu::IndexExpr& b) {
    gpu::IndexExpr r = a;
    r.code.insert(r.code.end(), b.code.begin(), b.code.end());
    r.code.push_back(gpu::IndexExpr::Add);
    return r;
  }
  static gpu::IndexExpr mulc(const gpu::IndexExpr& a, int64_t c) {
    gpu::IndexExpr r = a;
    r.code.push_back(gpu::IndexExpr::MulConst);
    r.code.push_back(c);
    return r;
  }
  static gpu::IndexExpr divmod(const gpu::IndexExpr& a, int64_t c, bool mod) {
    gpu::IndexExpr r = a;
    r.code.push_back(mod ? gpu::IndexExpr::Mod : gpu::IndexExpr::FloorDiv);
    r.code.push_back(c);
    return r;
  }

  // extent limit for reductions recomputed inside a consumer
  static constexpr int64_t kInlineAxis = 16;

  bool inlinable_kind(int i) const {
    const std::string& o = op(i).op;
    if (o == "add" || o == "sub" || o == "mul" || o == "max" || o == "exp" || o == "quantize" ||
        o == "dequantize" || o == "transpose" || o == "broadcast_in_dim" || o == "reshape")
      return true;
    if (o == "reduce" || o == "softmax") {
      const auto& s = desc(op(i).inputs[0]).shape;
      const int64_t r = static_cast<int64_t>(s.size());
      const int64_t ax = op(i).axis < 0 ? op(i).axis + r : op(i).axis;
      return ax >= 0 && ax < r && s[ax] <= kInlineAxis;
    }
    return false;
  }

  // An op's result is computed inside its consumers' launches when it is a
  // cheap index-local op, not a graph output, and every consumer is itself a
  // VM-region op (kernel groups need their inputs in HBM).
  void decide_inlining() {
    if (!opt_.fuse) return;
    for (int i = static_cast<int>(g_.ops.size()) - 1; i >= 0; --i) {
      if (group_of_[i] >= 0 || !inlinable_kind(i) || outputs_.count(op(i).output)) continue;
      auto it = consumers_.find(op(i).output);
      if (it == consumers_.end()) continue;
      bool all_vm = true;
      for (int c : it->second)
        if (group_of_[c] >= 0 || is_heavy(c)) all_vm = false;
      inline_[i] = all_vm;
    }
  }
  bool is_heavy(int i) const {
    const std::string& o = op(i).op;
    return o == "matmul" || o == "batch_matmul" || o == "conv2d" ||
           ((o == "softmax" || o == "reduce") && !inlinable_kind(i));
  }

  // value of tensor `id` at coordinates `at`, recomputing inlined producers
  std::string value_at(NestBuilder& nb, const std::string& id,
                       const std::vector<gpu::IndexExpr>& at) {
    const std::string key = key_of(id, at);
    if (const std::string* m = nb.memo(key)) return *m;
    std::string v;
    auto pi = producer_.find(id);
    if (R_.has(id) || pi == producer_.end() || !inline_[pi->second]) {
      v = nb.load(id, at);
    } else {
      v = compute_at(nb, pi->second, at);
    }
    nb.remember(key, v);
    return v;
  }

  // emits the computation of op i's result at `at`, rounded to its type
  std::string compute_at(NestBuilder& nb, int i, const std::vector<gpu::IndexExpr>& at) {
    using gpu::ArithOp;
    using gpu::NestOperand;
    const TensorOpNode& n = op(i);
    const ElementType ot = desc(n.output).dtype;
    const std::string& o = n.op;
    auto V = [](const std::string& s) { return NestOperand::val(s); };
    if (o == "add" || o == "sub" || o == "mul" || o == "max") {
      const std::string a = value_at(nb, n.inputs[0], at);
      const std::string b = value_at(nb, n.inputs[1], at);
      const ArithOp k = o == "add" ? ArithOp::Add : o == "sub" ? ArithOp::Sub
                        : o == "mul" ? ArithOp::Mul : ArithOp::Max;
      return nb.round(nb.arith(k, {V(a), V(b)}), ot);
    }
    if (o == "exp" || o == "quantize" || o == "dequantize") {
      const std::string a = value_at(nb, n.inputs[0], at);
      const ArithOp k = o == "exp" ? ArithOp::Exp : o == "quantize" ? ArithOp::Quant
                                                                    : ArithOp::Dequant;
      return nb.round(nb.arith(k, {V(a)}, n.scale), ot);
    }
    if (o == "transpose") {
      std::vector<gpu::IndexExpr> in(n.perm.size());
      for (size_t d = 0; d < n.perm.size(); ++d) in[n.perm[d]] = at[d];
      return nb.round(value_at(nb, n.inputs[0], in), ot);
    }
    if (o == "broadcast_in_dim") {
      std::vector<gpu::IndexExpr> in;
      for (int64_t d : n.dims) in.push_back(at[d]);
      return nb.round(value_at(nb, n.inputs[0], in), ot);
    }
    if (o == "reshape") {
      const auto& is = desc(n.inputs[0]).shape;
      const auto& os = desc(n.output).shape;
      std::vector<int64_t> is1, os1;
      for (int64_t d : is)
        if (d != 1) is1.push_back(d);
      for (int64_t d : os)
        if (d != 1) os1.push_back(d);
      std::vector<gpu::IndexExpr> in;
      if (is1 == os1) {  // only unit dims move: a direct dim correspondence
        size_t k = 0;
        for (int64_t d : is) {
          if (d == 1) {
            in.push_back(gpu::IndexExpr::constant(0));
            continue;
          }
          while (k < os.size() && os[k] == 1) ++k;
          in.push_back(at[k++]);
        }
      } else {  // through the flat row-major index
        gpu::IndexExpr flat = gpu::IndexExpr::constant(0);
        int64_t st = 1;
        for (int d = static_cast<int>(os.size()) - 1; d >= 0; --d) {
          flat = add(flat, mulc(at[d], st));
          st *= os[d];
        }
        std::vector<int64_t> ist(is.size(), 1);
        for (int d = static_cast<int>(is.size()) - 2; d >= 0; --d) ist[d] = ist[d + 1] * is[d + 1];
        for (size_t d = 0; d < is.size(); ++d) {
          gpu::IndexExpr e = divmod(flat, ist[d], false);
          if (d > 0) e = divmod(e, is[d], true);
          in.push_back(e);
        }
      }
      return nb.round(value_at(nb, n.inputs[0], in), ot);
    }
    if (o == "reduce") {
      const auto& is = desc(n.inputs[0]).shape;
      const int64_t r = static_cast<int64_t>(is.size());
      const int64_t ax = n.axis < 0 ? n.axis + r : n.axis;
      const bool mx = n.reduceOp == "max";
      // init store (-3e38 / 0 rounded to the output type), then acc = op(acc, x) per step
      const std::string acc = nb.round(
          nb.arith(ArithOp::Add, {NestOperand::immF(mx ? -3.0e38 : 0.0), NestOperand::immF(0.0)}),
          ot);
      const int pos = nb.open_loop(is[ax]);
      std::vector<gpu::IndexExpr> in;
      size_t k = 0;
      for (int64_t d = 0; d < r; ++d)
        in.push_back(d == ax ? gpu::IndexExpr::dim(pos) : at[k++]);
      const std::string x = value_at(nb, n.inputs[0], in);
      nb.round(nb.arith(mx ? ArithOp::Max : ArithOp::Add, {V(acc), V(x)}), ot, acc);
      nb.close_loop();
      return acc;
    }
    if (o == "softmax") {
      // the four nests of the lowering (frontend.cpp:564-625): row max, shifted
      // exp, row sum, divide; intermediates in the input's type
      const TensorDesc& in = desc(n.inputs[0]);
      const int64_t r = static_cast<int64_t>(in.shape.size());
      const int64_t ax = n.axis < 0 ? n.axis + r : n.axis;
      const ElementType it = in.dtype;
      auto along = [&](int pos) {
        std::vector<gpu::IndexExpr> c = at;
        c[ax] = gpu::IndexExpr::dim(pos);
        return c;
      };
      const std::string m = nb.round(
          nb.arith(ArithOp::Add, {NestOperand::immF(-3.0e38), NestOperand::immF(0.0)}), it);
      int pos = nb.open_loop(in.shape[ax]);
      nb.round(nb.arith(ArithOp::Max, {V(m), V(value_at(nb, n.inputs[0], along(pos)))}), it, m);
      nb.close_loop();
      const std::string s = nb.round(
          nb.arith(ArithOp::Add, {NestOperand::immF(0.0), NestOperand::immF(0.0)}), it);
      pos = nb.open_loop(in.shape[ax]);
      {
        const std::string x = value_at(nb, n.inputs[0], along(pos));
        const std::string e = nb.round(nb.arith(ArithOp::Exp, {V(nb.arith(ArithOp::Sub, {V(x), V(m)}))}), it);
        nb.round(nb.arith(ArithOp::Add, {V(s), V(e)}), it, s);
      }
      nb.close_loop();
      const std::string x = value_at(nb, n.inputs[0], at);
      const std::string e = nb.round(nb.arith(ArithOp::Exp, {V(nb.arith(ArithOp::Sub, {V(x), V(m)}))}), it);
      return nb.round(nb.arith(ArithOp::Div, {V(e), V(s)}), ot);
    }
    throw InterpError("afg: op " + o + " cannot be computed in a fused region");
  }

  // the refcounts of buffers referenced by other launches (none are private)
  const std::map<std::string, int>& no_priv() const {
    static const std::map<std::string, int> m;
    return m;
  }

  // one launch producing op i's output
  void materialise(int i) {
    const TensorOpNode& n = op(i);
    const TensorDesc& od = desc(n.output);
    const std::string& o = n.op;
    if (o == "matmul" || o == "batch_matmul") return run_matmul(i);
    if (o == "conv2d") return run_conv(i);
    if (o == "softmax" && is_float(od.dtype) && is_float(desc(n.inputs[0]).dtype) &&
        !inlinable_kind(i) && opt_.tensor_cores) {
      const auto& s = desc(n.inputs[0]).shape;
      const int64_t r = static_cast<int64_t>(s.size());
      const int64_t ax = n.axis < 0 ? n.axis + r : n.axis;
      if (ax == r - 1 && s.back() >= 32) {
        const DevTensor& x = R_.at(n.inputs[0]);
        DevTensor& y = R_.alloc(n.output, od.shape, od.dtype);
        ok(afg_softmax_lastdim(x.ptr, y.ptr, x.numel() / s.back(), s.back(),
                               kernel_dtype(x.et), kernel_dtype(od.dtype), R_.stream()));
        plan("afg_softmax_lastdim[K4 " + dims_str(s) + "] -> " + n.output);
        return;
      }
    }
    R_.alloc(n.output, od.shape, od.dtype);
    NestBuilder nb(*this);
    nb.frame(od.shape);
    std::vector<gpu::IndexExpr> at;
    for (size_t d = 0; d < od.shape.size(); ++d) at.push_back(nb.iv(static_cast<int>(d)));
    const std::string v = compute_at(nb, i, at);
    nb.store(n.output, v, at);
    const std::string line = R_.run_vm(nb.finish(), no_priv());
    plan(line + " fused region -> " + n.output);
  }

  // matmul / batch_matmul outside a pattern
  void run_matmul(int i) {
    const TensorOpNode& n = op(i);
    const TensorDesc& ad = desc(n.inputs[0]);
    const TensorDesc& bd = desc(n.inputs[1]);
    const TensorDesc& od = desc(n.output);
    const int64_t rank = static_cast<int64_t>(ad.shape.size());
    const int64_t M = ad.shape[rank - 2], K = ad.shape[rank - 1], N = bd.shape[rank - 1];
    int64_t batch = 1;
    for (int64_t d = 0; d + 2 < rank; ++d) batch *= ad.shape[d];
    // i8 x i8 -> i32: exact on K1c (no partial sum of K < 2^17 steps saturates)
    if (n.op == "matmul" && ad.dtype == ElementType::I8 && bd.dtype == ElementType::I8 &&
        od.dtype == ElementType::I32 && K < 131072) {
      const int64_t Kp = (K + 15) / 16 * 16;
      int8_t* a8 = static_cast<int8_t*>(R_.scratch(static_cast<size_t>(M * Kp)));
      int8_t* b8 = static_cast<int8_t*>(R_.scratch(static_cast<size_t>(N * Kp)));
      pack_i8(n.inputs[0], a8, M, K, Kp, false);
      pack_i8(n.inputs[1], b8, K, N, Kp, true);
      DevTensor& C = R_.alloc(n.output, od.shape, ElementType::I32);
      ok(afg_gemm_i8(a8, Kp, b8, Kp, C.ptr, N, M, N, Kp, 0, 1.0f, R_.stream()));
      plan("afg_gemm_i8[" + std::to_string(M) + "x" + std::to_string(N) + "x" +
           std::to_string(K) + "] -> " + n.output);
      return;
    }
    // float operands, f32 result: the GEMM kernels (fp32 SIMT is the
    // interpreter's sequential per-step f32 rounding, bit-exact)
    if (is_float(ad.dtype) && ad.dtype == bd.dtype && od.dtype == ElementType::F32) {
      DevTensor& C = R_.alloc(n.output, od.shape, ElementType::F32);
      afg_dtype t = tc_type({n.inputs[0], n.inputs[1]});
      if (t != AFG_F32 && K % 8 == 0 && N % 8 == 0) {
        const void* A = ad.dtype == ElementType::F32 ? narrowed(n.inputs[0], t) : R_.at(n.inputs[0]).ptr;
        const void* B = bd.dtype == ElementType::F32 ? narrowed(n.inputs[1], t) : R_.at(n.inputs[1]).ptr;
        const int64_t e = 2;
        for (int64_t b = 0; b < batch; ++b)
          ok(afg_gemm(static_cast<const char*>(A) + b * M * K * e, K,
                      static_cast<const char*>(B) + b * K * N * e, N, nullptr, nullptr,
                      static_cast<char*>(C.ptr) + b * M * N * 4, N, M, N, K, t, AFG_F32, AFG_B_KN,
                      AFG_EPI_NONE, R_.stream()));
        plan(std::string("afg_gemm[gemm_tc ") + (t == AFG_BF16 ? "bf16 " : "f16 ") +
             std::to_string(batch) + "x" + std::to_string(M) + "x" + std::to_string(N) + "x" +
             std::to_string(K) + "] -> " + n.output);
        return;
      }
      ok(afg_gemm_batched(R_.at(n.inputs[0]).ptr, R_.at(n.inputs[1]).ptr, C.ptr, batch, M, N, K,
                          kernel_dtype(ad.dtype), AFG_F32, R_.stream()));
      plan("afg_gemm[gemm_simt " + std::to_string(batch) + "x" + std::to_string(M) + "x" +
           std::to_string(N) + "x" + std::to_string(K) + "] -> " + n.output);
      return;
    }
    // anything else (integer / half results): the interpreter's nest on the VM
    // (C = 0; for k: C = round(a*b + C) -- every partial sum rounded / saturated)
    R_.alloc(n.output, od.shape, od.dtype);
    NestBuilder nb(*this);
    nb.frame(od.shape);
    std::vector<gpu::IndexExpr> c;
    for (int64_t d = 0; d < rank; ++d) c.push_back(nb.iv(static_cast<int>(d)));
    const std::string acc = nb.round(nb.arith(gpu::ArithOp::Add, {gpu::NestOperand::immF(0.0),
                                                                 gpu::NestOperand::immF(0.0)}),
                                     od.dtype);
    const int k = nb.open_loop(K);
    std::vector<gpu::IndexExpr> ai(c.begin(), c.end() - 1), bi(c.begin(), c.end() - 2);
    ai.push_back(gpu::IndexExpr::dim(k));
    bi.push_back(gpu::IndexExpr::dim(k));
    bi.push_back(c.back());
    const std::string a = nb.load(n.inputs[0], ai);
    const std::string b = nb.load(n.inputs[1], bi);
    nb.round(nb.arith(gpu::ArithOp::Fma, {gpu::NestOperand::val(a), gpu::NestOperand::val(b),
                                          gpu::NestOperand::val(acc)}),
             od.dtype, acc);
    nb.close_loop();
    nb.store(n.output, acc, c);
    plan(R_.run_vm(nb.finish(), no_priv()) + " matmul (per-step rounding) -> " + n.output);
  }

  // conv2d outside a pattern
  void run_conv(int i) {
    const TensorOpNode& n = op(i);
    const TensorDesc& xd = desc(n.inputs[0]);
    const TensorDesc& wd = desc(n.inputs[1]);
    const TensorDesc& od = desc(n.output);
    const int64_t B = xd.shape[0], C = xd.shape[1], H = xd.shape[2], W = xd.shape[3];
    const int64_t KH = wd.shape[2], KW = wd.shape[3], OC = od.shape[1];
    const Window wy = conv_window(H, KH, n.strideY, n.dilY, n.samePadding, n.transposed);
    const Window wx = conv_window(W, KW, n.strideX, n.dilX, n.samePadding, n.transposed);
    if (is_float(xd.dtype) && xd.dtype == wd.dtype && od.dtype == ElementType::F32 &&
        C % 64 == 0 && R_.has(n.inputs[0]) && R_.has(n.inputs[1])) {
      const afg_dtype t = tc_type({n.inputs[0], n.inputs[1]});
      if (t != AFG_F32) return run_conv_tc(i, wy, wx, t);
    }
    if (is_float(xd.dtype) && xd.dtype == wd.dtype && od.dtype == ElementType::F32) {
      DevTensor& Y = R_.alloc(n.output, od.shape, ElementType::F32);
      // the direct kernel takes the interpreter's begin pads; transposed convs
      // invert through the stuffed input (pad = span - 1 - same pad)
      ok(afg_conv2d_nchw(R_.at(n.inputs[0]).ptr, R_.at(n.inputs[1]).ptr, Y.ptr, B, C, H, W, OC,
                         KH, KW, n.strideY, n.strideX, n.dilY, n.dilX, wy.pad, wx.pad,
                         n.transposed ? 1 : 0, wy.out, wx.out, kernel_dtype(xd.dtype), AFG_F32,
                         R_.stream()));
      plan("afg_conv2d_nchw[direct " + dims_str(xd.shape) + "] -> " + n.output);
      return;
    }
    run_conv_vm(i, wy, wx);
  }

  // conv2d in the reference's NCHW / OIHW (IOHW transposed) layout on the
  // implicit-GEMM tensor-core kernel, for bf16 / f16-valued operands: the
  // input is re-laid out NHWC in the 16-bit type (exact), the filter packed
  // OHWI (flipped and transposed for a transposed conv), the fp32 result
  // permuted back to NCHW. Every conv variant of frontend.cpp:752-970 maps
  // onto the kernel's explicit geometry: stride / dilation / begin pads
  // (the far pads follow from OH, OW); a transposed conv is a stride-1 conv
  // over the zero-stuffed input (frontend.cpp:764-803) whose begin pad is
  // (K-1)*dil minus the dropped half of the same-pad.
  void run_conv_tc(int i, const Window& wy, const Window& wx, afg_dtype t) {
    const TensorOpNode& n = op(i);
    const TensorDesc& xd = desc(n.inputs[0]);
    const TensorDesc& wd = desc(n.inputs[1]);
    const TensorDesc& od = desc(n.output);
    const int64_t B = xd.shape[0], C = xd.shape[1], H = xd.shape[2], W = xd.shape[3];
    const int64_t KH = wd.shape[2], KW = wd.shape[3], OC = od.shape[1];
    const ElementType et = t == AFG_BF16 ? ElementType::BF16 : ElementType::F16;
    const int64_t sy = n.transposed ? n.strideY : 1, sx = n.transposed ? n.strideX : 1;
    // NHWC input (zero-stuffed when transposed)
    const int64_t IH = (H - 1) * sy + 1, IW = (W - 1) * sx + 1;
    const std::string X = "$tcx_" + n.output, Wt = "$tcw_" + n.output, Y = "$tcy_" + n.output;
    DevTensor& xt = R_.alloc(X, {B, IH, IW, C}, et);
    if (n.transposed)
      cudaMemsetAsync(xt.ptr, 0, static_cast<size_t>(xt.numel()) * 2, R_.stream());
    {
      NestBuilder nb(*this);
      nb.frame(xd.shape);  // b, c, y, x
      const std::string v = nb.load(n.inputs[0], {nb.iv(0), nb.iv(1), nb.iv(2), nb.iv(3)});
      nb.store(X, v, {nb.iv(0), mulc(nb.iv(2), sy), mulc(nb.iv(3), sx), nb.iv(1)});
      R_.run_vm(nb.finish(), no_priv());
    }
    // filter [OC, KH, KW, C] in the 16-bit type
    R_.alloc(Wt, {OC, KH, KW, C}, et);
    {
      NestBuilder nb(*this);
      nb.frame({OC, KH, KW, C});  // oc, ky, kx, c
      std::string v;
      if (!n.transposed) {
        v = nb.load(n.inputs[1], {nb.iv(0), nb.iv(3), nb.iv(1), nb.iv(2)});
      } else {  // IOHW, flipped taps
        v = nb.load(n.inputs[1], {nb.iv(3), nb.iv(0),
                                  add(mulc(nb.iv(1), -1), gpu::IndexExpr::constant(KH - 1)),
                                  add(mulc(nb.iv(2), -1), gpu::IndexExpr::constant(KW - 1))});
      }
      nb.store(Wt, v, {nb.iv(0), nb.iv(1), nb.iv(2), nb.iv(3)});
      R_.run_vm(nb.finish(), no_priv());
    }
    const int64_t pt = n.transposed ? (KH - 1) * n.dilY - wy.pad : wy.pad;
    const int64_t pl = n.transposed ? (KW - 1) * n.dilX - wx.pad : wx.pad;
    DevTensor& yt = R_.alloc(Y, {B, wy.out, wx.out, OC}, ElementType::F32);
    ok(afg_conv2d_nhwc_ex(R_.at(X).ptr, R_.at(Wt).ptr, nullptr, yt.ptr, B, IH, IW, C, OC, KH, KW,
                          n.transposed ? 1 : n.strideY, n.transposed ? 1 : n.strideX, pt, pl,
                          n.dilY, n.dilX, wy.out, wx.out, t, AFG_F32, AFG_EPI_NONE,
                          R_.stream()));
    R_.alloc(n.output, od.shape, ElementType::F32);
    run_copy_permuted(Y, n.output, {0, 3, 1, 2});
    R_.release(X);
    R_.release(Wt);
    R_.release(Y);
    plan(std::string("afg_conv2d_nhwc[conv_tc ") + (t == AFG_BF16 ? "bf16 " : "f16 ") +
         dims_str(xd.shape) + " k" + std::to_string(KH) + "x" + std::to_string(KW) + " s" +
         std::to_string(n.strideY) + " d" + std::to_string(n.dilY) +
         (n.samePadding ? " same" : " valid") + (n.transposed ? " transposed" : "") +
         "] NCHW conv2d -> " + n.output);
  }

  // The interpreter's conv nest (frontend.cpp:752-970 semantics) on the VM,
  // for integer / half outputs where every stored partial sum is rounded: the
  // loop form (padded or > 8 taps) rounds after every tap, the unrolled form
  // once at the end; taps outside the input are skipped.
  void run_conv_vm(int i, const Window& wy, const Window& wx) {
    using gpu::ArithOp;
    using gpu::NestOperand;
    const TensorOpNode& n = op(i);
    const TensorDesc& xd = desc(n.inputs[0]);
    const TensorDesc& wd = desc(n.inputs[1]);
    const TensorDesc& od = desc(n.output);
    const int64_t C = xd.shape[1], H = xd.shape[2], W = xd.shape[3], KH = wd.shape[2],
                  KW = wd.shape[3];
    // the reference unrolls unpadded reductions of <= 8 taps (one rounding);
    // a transposed conv is an unpadded conv over its stride-stuffed input
    const bool unrolled = (n.transposed || (wy.pad == 0 && wx.pad == 0)) && C * KH * KW <= 8;
    R_.alloc(n.output, od.shape, od.dtype);
    // Taps outside the input are skipped by the interpreter; a zero tap adds
    // exactly 0 to the running sum, so the nest reads a zero-bordered copy P
    // of the input (stride-stuffed for transposed convs) and never branches.
    const int64_t pad_y = (KH - 1) * n.dilY, pad_x = (KW - 1) * n.dilX;
    const int64_t sy_in = n.transposed ? n.strideY : 1, sx_in = n.transposed ? n.strideX : 1;
    const int64_t PH = (H - 1) * sy_in + 1 + 2 * pad_y;
    const int64_t PW = (W - 1) * sx_in + 1 + 2 * pad_x;
    const std::string P = "$convpad_" + n.output;
    DevTensor& pt = R_.alloc(P, {xd.shape[0], C, PH, PW}, xd.dtype);
    cudaMemsetAsync(pt.ptr, 0, static_cast<size_t>(pt.numel()) * vm::vm_type_bytes(pt.type),
                    R_.stream());
    {
      NestBuilder nb(*this);
      nb.frame(xd.shape);
      const std::string v = nb.load(n.inputs[0], {nb.iv(0), nb.iv(1), nb.iv(2), nb.iv(3)});
      nb.store(P, v, {nb.iv(0), nb.iv(1),
                      add(mulc(nb.iv(2), sy_in), gpu::IndexExpr::constant(pad_y)),
                      add(mulc(nb.iv(3), sx_in), gpu::IndexExpr::constant(pad_x))});
      R_.run_vm(nb.finish(), no_priv());
    }
    // effective valid conv over P: stride 1 + flipped IOHW weights when transposed
    const int64_t sy = n.transposed ? 1 : n.strideY, sx = n.transposed ? 1 : n.strideX;
    // P row of output oy, tap ky: oy*s + ky*d - pad + pad_y (direct); the
    // stuffed-input row oy + ky*d shifted by the dropped half of the same-pad
    // (transposed)
    const int64_t off_y = n.transposed ? wy.pad : pad_y - wy.pad;
    const int64_t off_x = n.transposed ? wx.pad : pad_x - wx.pad;
    NestBuilder nb(*this);
    nb.frame(od.shape);
    const std::vector<gpu::IndexExpr> o = {nb.iv(0), nb.iv(1), nb.iv(2), nb.iv(3)};
    std::string acc;
    bool first = true;
    auto tap = [&](const gpu::IndexExpr& ic, const gpu::IndexExpr& ky, const gpu::IndexExpr& kx) {
      const gpu::IndexExpr iy =
          add(add(mulc(o[2], sy), mulc(ky, n.dilY)), gpu::IndexExpr::constant(off_y));
      const gpu::IndexExpr ix =
          add(add(mulc(o[3], sx), mulc(kx, n.dilX)), gpu::IndexExpr::constant(off_x));
      const std::string xv = nb.load(P, {o[0], ic, iy, ix});
      gpu::IndexExpr wky = ky, wkx = kx;
      if (n.transposed) {  // flipped taps, IOHW layout
        wky = add(mulc(ky, -1), gpu::IndexExpr::constant(KH - 1));
        wkx = add(mulc(kx, -1), gpu::IndexExpr::constant(KW - 1));
      }
      const std::string wv = n.transposed ? nb.load(n.inputs[1], {ic, o[1], wky, wkx})
                                          : nb.load(n.inputs[1], {o[1], ic, wky, wkx});
      if (unrolled) {
        acc = first ? nb.arith(ArithOp::Mul, {NestOperand::val(xv), NestOperand::val(wv)})
                    : nb.arith(ArithOp::Fma, {NestOperand::val(xv), NestOperand::val(wv),
                                              NestOperand::val(acc)});
      } else {
        nb.round(nb.arith(ArithOp::Fma, {NestOperand::val(xv), NestOperand::val(wv),
                                         NestOperand::val(acc)}),
                 od.dtype, acc);
      }
      first = false;
    };
    if (unrolled) {
      for (int64_t c = 0; c < C; ++c)
        for (int64_t ky = 0; ky < KH; ++ky)
          for (int64_t kx = 0; kx < KW; ++kx)
            tap(gpu::IndexExpr::constant(c), gpu::IndexExpr::constant(ky),
                gpu::IndexExpr::constant(kx));
      acc = nb.round(acc, od.dtype);
    } else {
      acc = nb.round(nb.arith(ArithOp::Add, {NestOperand::immF(0.0), NestOperand::immF(0.0)}),
                     od.dtype);
      const int ic = nb.open_loop(C);
      const int ky = nb.open_loop(KH);
      const int kx = nb.open_loop(KW);
      tap(gpu::IndexExpr::dim(ic), gpu::IndexExpr::dim(ky), gpu::IndexExpr::dim(kx));
      nb.close_loop();
      nb.close_loop();
      nb.close_loop();
    }
    nb.store(n.output, acc, o);
    plan(R_.run_vm(nb.finish(), no_priv()) + " conv2d (" +
         (unrolled ? "unrolled, one rounding" : "per-tap rounding") + ") -> " + n.output);
    R_.release(P);
  }
};

}  // namespace

namespace {

// Which tensors carry the shard dimension (dim 0 split over the shards)?
// Propagates from the graph inputs whose leading extent is B; throws a
// GraphError when an op would mix rows of different shards.
std::set<std::string> shard_plan(const TensorGraph& g, int64_t B) {
  std::set<std::string> sh;
  auto lead = [&](const std::string& id) {
    const TensorDesc* d = g.find(id);
    return d && !d->shape.empty() ? d->shape[0] : -1;
  };
  // graph inputs with leading extent B are split, except operands that must
  // stay whole (a matmul's B, a conv filter) whose extent matches by accident
  std::set<std::string> whole;
  for (const auto& n : g.ops)
    if (n.op == "matmul" || n.op == "conv2d") whole.insert(n.inputs.at(1));
  for (const auto& id : g.inputIds())
    if (lead(id) == B && !whole.count(id)) sh.insert(id);
  auto no = [&](const TensorOpNode& n, const std::string& why) {
    throw GraphError("graph not shardable along dim 0 at " + n.op + " -> " + n.output + ": " + why);
  };
  for (const auto& n : g.ops) {
    const std::string& o = n.op;
    std::vector<bool> in;
    for (const auto& x : n.inputs) in.push_back(sh.count(x) != 0);
    const bool any = std::find(in.begin(), in.end(), true) != in.end();
    const bool all = std::find(in.begin(), in.end(), false) == in.end();
    bool out = false;
    if (o == "add" || o == "sub" || o == "mul" || o == "max" || o == "exp" || o == "quantize" ||
        o == "dequantize") {
      if (any && !all) no(n, "a sharded and a replicated operand");
      out = any;
    } else if (o == "matmul") {
      if (in[1]) no(n, "the B operand is sharded");
      out = in[0];
    } else if (o == "batch_matmul" || o == "conv2d") {
      if (o == "conv2d" && in[1]) no(n, "the filter is sharded");
      if (o == "batch_matmul" && in[0] != in[1]) no(n, "one operand sharded");
      out = in[0];
    } else if (o == "transpose") {
      if (in[0] && n.perm.at(0) != 0) no(n, "dim 0 moves");
      out = in[0];
    } else if (o == "broadcast_in_dim") {
      const bool maps0 = std::find(n.dims.begin(), n.dims.end(), 0) != n.dims.end();
      if (in[0]) {
        if (n.dims.at(0) != 0) no(n, "dim 0 moves");
        out = true;
      } else {
        // a replicated value broadcast into a [B, ...] result: each shard
        // computes its own slice
        out = !maps0 && lead(n.output) == B;
      }
    } else if (o == "reshape") {
      if (in[0] && !(lead(n.inputs[0]) == B && lead(n.output) == B)) no(n, "dim 0 changes");
      out = in[0];
    } else if (o == "reduce" || o == "softmax") {
      const int64_t r = static_cast<int64_t>(g.find(n.inputs[0])->shape.size());
      const int64_t ax = n.axis < 0 ? n.axis + r : n.axis;
      if (in[0] && ax == 0) no(n, "reduces over dim 0");
      out = in[0];
    }
    if (out) sh.insert(n.output);
  }
  return sh;
}

}  // namespace

std::map<std::string, TensorValue> execute(const TensorGraph& g,
                                           const std::map<std::string, TensorValue>& inputs,
                                           const GpuOptions& opt, ExecStats* stats) {
  if (opt.devices.size() <= 1) {
    GpuOptions o = opt;
    int prev = -1;
    if (opt.devices.size() == 1) {
      cudaGetDevice(&prev);
      cudaSetDevice(opt.devices[0]);
    }
    Planner p(g, o, stats);
    auto out = p.run(inputs);
    if (prev >= 0) cudaSetDevice(prev);
    return out;
  }
  // ---- thread-per-device sharded execution ----
  validateGraph(g);
  const auto ins = g.inputIds();
  int64_t B = opt.shard_extent;
  if (B <= 0) {
    const TensorDesc* d = ins.empty() ? nullptr : g.find(ins[0]);
    if (!d || d->shape.empty()) throw GraphError("graph not shardable: no leading extent");
    B = d->shape[0];
  }
  const int P = static_cast<int>(opt.devices.size());
  if (B < P) throw GraphError("graph not shardable: leading extent below the device count");
  const std::set<std::string> sh = shard_plan(g, B);
  // contiguous blocks of the leading extent, remainder spread (shard.py)
  std::vector<std::pair<int64_t, int64_t>> blocks;
  for (int r = 0; r < P; ++r) {
    const int64_t base = B / P, rem = B % P;
    const int64_t b0 = r * base + std::min<int64_t>(r, rem);
    blocks.push_back({b0, b0 + base + (r < rem ? 1 : 0)});
  }
  std::vector<TensorGraph> graphs(P, g);
  std::vector<std::map<std::string, TensorValue>> shard_in(P);
  for (int r = 0; r < P; ++r) {
    const int64_t rows = blocks[r].second - blocks[r].first;
    for (auto& t : graphs[r].tensors)
      if (sh.count(t.id)) t.shape[0] = rows;
    for (const auto& id : ins) {
      auto it = inputs.find("%" + id);
      if (it == inputs.end()) it = inputs.find(id);
      if (it == inputs.end()) throw InterpError("missing input %" + id);
      if (!it->second.view && static_cast<int64_t>(it->second.data.size()) != it->second.numElements())
        throw InterpError("input shape mismatch for %" + id);
      TensorValue v;  // a view of the caller's values: the shard's rows, or all of them
      v.shape = it->second.shape;
      v.type = it->second.type;
      v.view = it->second.values();
      if (sh.count(id)) {
        const int64_t inner = v.numElements() / v.shape[0];
        v.shape[0] = rows;
        v.view += blocks[r].first * inner;
      }
      shard_in[r]["%" + id] = std::move(v);
    }
  }
  std::vector<std::map<std::string, TensorValue>> shard_out(P);
  std::vector<std::string> errors(P);
  std::vector<ExecStats> shard_stats(P);
  DeviceGroup group(opt.devices, /*with_comms=*/false);  // shards exchange nothing
  group.run([&](int r, int, void* stream, void*) {
    try {
      GpuOptions o = opt;
      o.devices.clear();
      o.stream = stream;
      Planner p(graphs[r], o, &shard_stats[r]);
      shard_out[r] = p.run(shard_in[r]);
    } catch (const std::exception& e) {
      errors[r] = e.what();
    }
  });
  for (int r = 0; r < P; ++r)
    if (!errors[r].empty()) throw InterpError("shard " + std::to_string(r) + ": " + errors[r]);
  std::map<std::string, TensorValue> out;
  for (const auto& [key, v0] : shard_out[0]) {
    const std::string id = key.substr(1);
    if (!sh.count(id)) {  // replicated: every shard computed the same value
      out[key] = v0;
      continue;
    }
    TensorValue v = v0;
    v.shape[0] = B;
    v.data.clear();
    for (int r = 0; r < P; ++r) {
      const auto& part = shard_out[r].at(key).data;
      v.data.insert(v.data.end(), part.begin(), part.end());
    }
    out[key] = std::move(v);
  }
  if (stats)
    for (int r = 0; r < P; ++r) {
      for (const auto& l : shard_stats[r].plan)
        stats->plan.push_back("[shard " + std::to_string(r) + " on device " +
                              std::to_string(opt.devices[r]) + "] " + l);
      stats->fused += shard_stats[r].fused;
    }
  return out;
}

}  // namespace gpu
}  // namespace afg

// ============================================================== C ABI ====

struct afg_graph_result {
  std::vector<std::string> names;
  std::vector<afg::gpu::TensorValue> values;
  std::string plan;
};

extern "C" {

AFG_API afg_status afg_graph_run(const char* graph_json, int n_inputs, const char* const* names,
                                 const double* const* data, const int64_t* numel, int flags,
                                 void* stream, afg_graph_result** out) {
  using namespace afg::gpu;
  if (!graph_json || !out || (n_inputs > 0 && (!names || !data || !numel)))
    return afg::set_error(AFG_ERR_INVALID_ARG, "afg_graph_run: null argument");
  *out = nullptr;
  try {
    TensorGraph g = parseGraphJson(graph_json);
    std::map<std::string, TensorValue> inputs;
    for (int i = 0; i < n_inputs; ++i) {
      std::string id = names[i];
      if (!id.empty() && id[0] == '%') id.erase(0, 1);
      const TensorDesc* d = g.find(id);
      if (!d) throw InterpError("unknown input " + id);
      TensorValue v;
      v.shape = d->shape;
      v.type = d->dtype;
      if (v.numElements() != numel[i]) throw InterpError("input shape mismatch for %" + id);
      v.view = data[i];  // the caller's buffer, read once on upload (no host copy)
      inputs["%" + id] = std::move(v);
    }
    GpuOptions opt;
    opt.stream = stream;
    opt.fuse = (flags & AFG_GRAPH_FUSE) != 0;
    opt.tensor_cores = (flags & AFG_GRAPH_EXACT) == 0;
    ExecStats stats;
    auto res = execute(g, inputs, opt, &stats);
    auto* r = new afg_graph_result;
    for (auto& kv : res) {
      r->names.push_back(kv.first);
      r->values.push_back(std::move(kv.second));
    }
    for (const auto& l : stats.plan) r->plan += l + "\n";
    *out = r;
    return AFG_OK;
  } catch (const GraphError& e) {
    return afg::set_error(AFG_ERR_INVALID_ARG, "GraphError: %s", e.what());
  } catch (const InterpError& e) {
    return afg::set_error(AFG_ERR_CUDA, "InterpError: %s", e.what());
  } catch (const std::exception& e) {
    return afg::set_error(AFG_ERR_INTERNAL, "%s", e.what());
  }
}

AFG_API afg_status afg_graph_run_sharded(const char* graph_json, int n_inputs,
                                         const char* const* names, const double* const* data,
                                         const int64_t* numel, int flags, int ndev,
                                         const int* devices, int64_t shard_extent,
                                         afg_graph_result** out) {
  using namespace afg::gpu;
  if (!graph_json || !out || ndev < 1 || !devices || (n_inputs > 0 && (!names || !data || !numel)))
    return afg::set_error(AFG_ERR_INVALID_ARG, "afg_graph_run_sharded: bad argument");
  *out = nullptr;
  try {
    TensorGraph g = parseGraphJson(graph_json);
    std::map<std::string, TensorValue> inputs;
    for (int i = 0; i < n_inputs; ++i) {
      std::string id = names[i];
      if (!id.empty() && id[0] == '%') id.erase(0, 1);
      const TensorDesc* d = g.find(id);
      if (!d) throw InterpError("unknown input " + id);
      TensorValue v;
      v.shape = d->shape;
      v.type = d->dtype;
      if (v.numElements() != numel[i]) throw InterpError("input shape mismatch for %" + id);
      v.view = data[i];  // the caller's buffer, read once on upload (no host copy)
      inputs["%" + id] = std::move(v);
    }
    GpuOptions opt;
    opt.fuse = (flags & AFG_GRAPH_FUSE) != 0;
    opt.tensor_cores = (flags & AFG_GRAPH_EXACT) == 0;
    opt.devices.assign(devices, devices + ndev);
    opt.shard_extent = shard_extent;
    ExecStats stats;
    auto res = execute(g, inputs, opt, &stats);
    auto* r = new afg_graph_result;
    for (auto& kv : res) {
      r->names.push_back(kv.first);
      r->values.push_back(std::move(kv.second));
    }
    for (const auto& l : stats.plan) r->plan += l + "\n";
    *out = r;
    return AFG_OK;
  } catch (const GraphError& e) {
    return afg::set_error(AFG_ERR_INVALID_ARG, "GraphError: %s", e.what());
  } catch (const InterpError& e) {
    return afg::set_error(AFG_ERR_CUDA, "InterpError: %s", e.what());
  } catch (const std::exception& e) {
    return afg::set_error(AFG_ERR_INTERNAL, "%s", e.what());
  }
}

AFG_API int afg_graph_result_count(const afg_graph_result* r) {
  return r ? static_cast<int>(r->names.size()) : 0;
}
AFG_API const char* afg_graph_result_name(const afg_graph_result* r, int i) {
  return r->names.at(i).c_str();
}
AFG_API int afg_graph_result_rank(const afg_graph_result* r, int i) {
  return static_cast<int>(r->values.at(i).shape.size());
}
AFG_API int64_t afg_graph_result_dim(const afg_graph_result* r, int i, int d) {
  return r->values.at(i).shape.at(d);
}
AFG_API int64_t afg_graph_result_numel(const afg_graph_result* r, int i) {
  return r->values.at(i).numElements();
}
AFG_API const double* afg_graph_result_data(const afg_graph_result* r, int i) {
  return r->values.at(i).data.data();
}
AFG_API const char* afg_graph_result_plan(const afg_graph_result* r) { return r->plan.c_str(); }
AFG_API void afg_graph_result_free(afg_graph_result* r) { delete r; }

AFG_API afg_status afg_graph_check_json(const char* graph_json) {
  try {
    afg::gpu::validateGraph(afg::gpu::parseGraphJson(graph_json ? graph_json : ""));
    return AFG_OK;
  } catch (const std::exception& e) {
    return afg::set_error(AFG_ERR_INVALID_ARG, "GraphError: %s", e.what());
  }
}

}  // extern "C"
