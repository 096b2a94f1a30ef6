// graph.cpp - the C++ host executor behind include/afg_graph.h: the drop-in
// for the reference's graph -> interpret path (frontend.cpp:57-294, :975;
// interp.cpp:164-696).
//
//  * parseGraphJson / checkGraph / convGeometry restate the reference's
//    frontend rules (same schema, same GraphError texts "unsupported-op",
//    "shape-mismatch", ...), with a self-contained JSON reader.
//  * execute() keeps every tensor resident on the device in its declared
//    element type (so each op's result is rounded to the declared type at its
//    store, the interpreter's convention, interp.cpp:335-347), plans the
//    graph into kernel launches and returns the outputs keyed "%id":
//      - matmul -> broadcast_in_dim(bias) -> add [-> max(., zeros)]
//          => ONE afg_gemm with the BIAS / BIAS_RELU epilogue;
//      - transpose(k) -> batch_matmul(q, kt) [-> add(bias)] -> softmax ->
//        batch_matmul(., v)  => ONE afg_attention_fwd (the reduce-reduce +
//          matmul-outlining + register fusion of SPEC.md:454-529);
//      - every other op => its own afg kernel (no CPU execution anywhere).
//  * afg_graph_run (extern "C") exposes the same to non-C++ callers.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <set>
#include <sstream>

#include "../../include/afg.h"
#include "../../include/afg_graph.h"
#include "afg_internal.h"

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

class Parser {
 public:
  explicit Parser(const std::string& s) : s_(s) {}
  Value parse() {
    Value v = value();
    ws();
    if (i_ != s_.size()) fail("trailing characters");
    return v;
  }

 private:
  const std::string& s_;
  size_t i_ = 0;
  [[noreturn]] void fail(const char* what) {
    throw GraphError(std::string("graph json parse error: ") + what + " at offset " +
                     std::to_string(i_));
  }
  void ws() {
    while (i_ < s_.size() && std::isspace(static_cast<unsigned char>(s_[i_]))) ++i_;
  }
  bool eat(char c) {
    ws();
    if (i_ < s_.size() && s_[i_] == c) {
      ++i_;
      return true;
    }
    return false;
  }
  Value value() {
    ws();
    if (i_ >= s_.size()) fail("unexpected end");
    const char c = s_[i_];
    Value v;
    if (c == '{') {
      ++i_;
      v.kind = Value::Object;
      if (eat('}')) return v;
      do {
        ws();
        Value k = value();
        if (k.kind != Value::String) fail("object key");
        if (!eat(':')) fail("expected ':'");
        v.obj.emplace_back(k.str, value());
      } while (eat(','));
      if (!eat('}')) fail("expected '}'");
    } else if (c == '[') {
      ++i_;
      v.kind = Value::Array;
      if (eat(']')) return v;
      do v.arr.push_back(value());
      while (eat(','));
      if (!eat(']')) fail("expected ']'");
    } else if (c == '"') {
      ++i_;
      v.kind = Value::String;
      while (i_ < s_.size() && s_[i_] != '"') {
        if (s_[i_] == '\\') {
          ++i_;
          if (i_ >= s_.size()) fail("bad escape");
          const char e = s_[i_];
          v.str += e == 'n' ? '\n' : e == 't' ? '\t' : e;
        } else {
          v.str += s_[i_];
        }
        ++i_;
      }
      if (i_ >= s_.size()) fail("unterminated string");
      ++i_;
    } else if (s_.compare(i_, 4, "true") == 0) {
      i_ += 4;
      v.kind = Value::Bool;
      v.b = true;
    } else if (s_.compare(i_, 5, "false") == 0) {
      i_ += 5;
      v.kind = Value::Bool;
    } else if (s_.compare(i_, 4, "null") == 0) {
      i_ += 4;
    } else {
      size_t end = i_;
      while (end < s_.size() && (std::isdigit(static_cast<unsigned char>(s_[end])) ||
                                 s_[end] == '-' || s_[end] == '+' || s_[end] == '.' ||
                                 s_[end] == 'e' || s_[end] == 'E'))
        ++end;
      if (end == i_) fail("unexpected character");
      v.kind = Value::Number;
      v.num = std::strtod(s_.substr(i_, end - i_).c_str(), nullptr);
      i_ = end;
    }
    return v;
  }
};

}  // namespace json

// ================================================= graph API (frontend) ====

const TensorDesc* TensorGraph::find(const std::string& id) const {
  for (const auto& t : tensors)
    if (t.id == id) return &t;
  return nullptr;
}

std::vector<std::string> TensorGraph::inputIds() const {
  std::set<std::string> produced;
  for (const auto& op : ops) produced.insert(op.output);
  std::vector<std::string> out;
  for (const auto& t : tensors)
    if (!produced.count(t.id)) out.push_back(t.id);
  return out;
}

std::vector<std::string> TensorGraph::outputIds() const {
  if (!outputs.empty()) return outputs;
  std::set<std::string> consumed, produced;
  for (const auto& op : ops) {
    for (const auto& in : op.inputs) consumed.insert(in);
    produced.insert(op.output);
  }
  std::vector<std::string> out;
  for (const auto& t : tensors)
    if (produced.count(t.id) && !consumed.count(t.id)) out.push_back(t.id);
  return out;
}

namespace {

std::vector<int64_t> int_list(const json::Value& v, const char* what) {
  if (v.kind != json::Value::Array) throw GraphError(std::string("expected array for ") + what);
  std::vector<int64_t> out;
  for (const auto& e : v.arr) {
    if (e.kind != json::Value::Number) throw GraphError(std::string("expected ints in ") + what);
    out.push_back(static_cast<int64_t>(e.num));
  }
  return out;
}

const json::Value& need(const json::Value& o, const char* k) {
  const json::Value* v = o.get(k);
  if (!v) throw GraphError(std::string("graph json: missing key \"") + k + "\"");
  return *v;
}

bool parse_dtype(const std::string& s, ElementType& t) {
  if (s == "f32") t = ElementType::F32;
  else if (s == "f16") t = ElementType::F16;
  else if (s == "i8") t = ElementType::I8;
  else if (s == "i32") t = ElementType::I32;
  else if (s == "bf16") t = ElementType::BF16;  // extension
  else return false;
  return true;
}

}  // namespace

TensorGraph parseGraphJson(const std::string& text) {
  json::Value g = json::Parser(text).parse();
  if (g.kind != json::Value::Object || !g.get("tensors") || !g.get("ops"))
    throw GraphError("graph json must contain \"tensors\" and \"ops\"");
  TensorGraph graph;
  for (const auto& t : g.get("tensors")->arr) {
    TensorDesc d;
    d.id = need(t, "id").str;
    d.shape = int_list(need(t, "shape"), "shape");
    const json::Value* dt = t.get("dtype");
    if (!parse_dtype(dt ? dt->str : "f32", d.dtype))
      throw GraphError("unknown dtype for tensor " + d.id);
    graph.tensors.push_back(std::move(d));
  }
  for (const auto& n : g.get("ops")->arr) {
    TensorOpNode node;
    node.op = need(n, "op").str;
    for (const auto& in : need(n, "inputs").arr) node.inputs.push_back(in.str);
    node.output = need(n, "output").str;
    if (const json::Value* a = n.get("attrs")) {
      if (const json::Value* v = a->get("perm")) node.perm = int_list(*v, "perm");
      if (const json::Value* v = a->get("dims")) node.dims = int_list(*v, "dims");
      auto pair = [&](const char* key, int64_t& y, int64_t& x) {
        const json::Value* v = a->get(key);
        if (!v) return;
        if (v->kind == json::Value::Array) {
          y = static_cast<int64_t>(v->arr.at(0).num);
          x = static_cast<int64_t>(v->arr.at(1).num);
        } else {
          y = x = static_cast<int64_t>(v->num);
        }
      };
      pair("stride", node.strideY, node.strideX);
      pair("dilation", node.dilY, node.dilX);
      if (const json::Value* v = a->get("padding")) node.samePadding = v->str == "same";
      if (const json::Value* v = a->get("transposed")) node.transposed = v->b;
      if (const json::Value* v = a->get("op")) node.reduceOp = v->str;
      if (const json::Value* v = a->get("axis")) node.axis = static_cast<int64_t>(v->num);
      if (const json::Value* v = a->get("scale")) node.scale = v->num;
    }
    graph.ops.push_back(std::move(node));
  }
  if (const json::Value* o = g.get("outputs"))
    for (const auto& e : o->arr) graph.outputs.push_back(e.str);
  return graph;
}

ConvGeometry convGeometry(int64_t inH, int64_t inW, int64_t kH, int64_t kW,
                          const TensorOpNode& node) {
  ConvGeometry d{};
  if (!node.transposed) {
    if (node.samePadding) {
      d.outH = (inH + node.strideY - 1) / node.strideY;
      d.outW = (inW + node.strideX - 1) / node.strideX;
      const int64_t ty =
          std::max<int64_t>(0, (d.outH - 1) * node.strideY + (kH - 1) * node.dilY + 1 - inH);
      const int64_t tx =
          std::max<int64_t>(0, (d.outW - 1) * node.strideX + (kW - 1) * node.dilX + 1 - inW);
      d.padY = ty / 2;
      d.padX = tx / 2;
    } else {
      d.outH = (inH - (kH - 1) * node.dilY - 1) / node.strideY + 1;
      d.outW = (inW - (kW - 1) * node.dilX - 1) / node.strideX + 1;
    }
  } else {
    if (node.samePadding) {
      d.outH = inH * node.strideY;
      d.outW = inW * node.strideX;
      const int64_t ty = (kH - 1) * node.dilY + 1 - node.strideY;
      const int64_t tx = (kW - 1) * node.dilX + 1 - node.strideX;
      if (ty < 0 || tx < 0)
        throw GraphError(
            "unsupported-op: transposed same-padding with stride exceeding the kernel span");
      d.padY = ty / 2;
      d.padX = tx / 2;
    } else {
      d.outH = (inH - 1) * node.strideY + (kH - 1) * node.dilY + 1;
      d.outW = (inW - 1) * node.strideX + (kW - 1) * node.dilX + 1;
    }
  }
  return d;
}

namespace {

const std::set<std::string> kSupportedOps = {
    "conv2d", "matmul", "batch_matmul", "transpose", "add", "mul", "sub", "exp", "max",
    "broadcast_in_dim", "reduce", "softmax", "reshape", "quantize", "dequantize"};

std::vector<int64_t> expectedShape(const TensorGraph& g, const TensorOpNode& node) {
  auto in = [&](size_t i) -> const TensorDesc& {
    const TensorDesc* t = g.find(node.inputs.at(i));
    if (!t) throw GraphError("unknown tensor " + node.inputs.at(i));
    return *t;
  };
  const std::string& op = node.op;
  if (op == "add" || op == "mul" || op == "sub" || op == "max") {
    if (in(0).shape != in(1).shape)
      throw GraphError("shape-mismatch: elementwise operands of " + node.output);
    return in(0).shape;
  }
  if (op == "exp" || op == "softmax" || op == "quantize" || op == "dequantize")
    return in(0).shape;
  if (op == "transpose") {
    const auto& s = in(0).shape;
    if (node.perm.size() != s.size()) throw GraphError("shape-mismatch: transpose perm rank");
    std::vector<int64_t> out(s.size());
    for (size_t d = 0; d < s.size(); ++d) out[d] = s.at(node.perm[d]);
    return out;
  }
  if (op == "broadcast_in_dim") {
    const TensorDesc* o = g.find(node.output);
    if (!o) throw GraphError("unknown tensor " + node.output);
    const auto& s = in(0).shape;
    if (node.dims.size() != s.size())
      throw GraphError("shape-mismatch: broadcast_in_dim dims rank");
    for (size_t d = 0; d < s.size(); ++d)
      if (o->shape.at(node.dims[d]) != s[d])
        throw GraphError("shape-mismatch: broadcast_in_dim extents");
    return o->shape;
  }
  if (op == "reshape") {
    const TensorDesc* o = g.find(node.output);
    if (!o) throw GraphError("unknown tensor " + node.output);
    int64_t a = 1, b = 1;
    for (int64_t d : in(0).shape) a *= d;
    for (int64_t d : o->shape) b *= d;
    if (a != b) throw GraphError("shape-mismatch: reshape element count");
    return o->shape;
  }
  if (op == "reduce") {
    const auto& s = in(0).shape;
    const int64_t axis = node.axis < 0 ? node.axis + static_cast<int64_t>(s.size()) : node.axis;
    if (axis < 0 || axis >= static_cast<int64_t>(s.size()))
      throw GraphError("shape-mismatch: reduce axis out of range");
    std::vector<int64_t> out;
    for (size_t d = 0; d < s.size(); ++d)
      if (static_cast<int64_t>(d) != axis) out.push_back(s[d]);
    if (out.empty()) out.push_back(1);
    return out;
  }
  if (op == "matmul") {
    const auto& a = in(0).shape;
    const auto& b = in(1).shape;
    if (a.size() != 2 || b.size() != 2 || a[1] != b[0])
      throw GraphError("shape-mismatch: matmul operands of " + node.output);
    return {a[0], b[1]};
  }
  if (op == "batch_matmul") {
    const auto& a = in(0).shape;
    const auto& b = in(1).shape;
    if (a.size() != b.size() || a.size() < 2) throw GraphError("shape-mismatch: batch_matmul rank");
    for (size_t d = 0; d + 2 < a.size(); ++d)
      if (a[d] != b[d]) throw GraphError("shape-mismatch: batch_matmul batch dims");
    if (a.back() != b[b.size() - 2]) throw GraphError("shape-mismatch: batch_matmul contraction");
    std::vector<int64_t> out(a.begin(), a.end() - 1);
    out.push_back(b.back());
    return out;
  }
  if (op == "conv2d") {
    const auto& s = in(0).shape;
    const auto& w = in(1).shape;
    if (s.size() != 4 || w.size() != 4)
      throw GraphError("shape-mismatch: conv2d operands must be rank 4");
    const int64_t ic = node.transposed ? w[0] : w[1];
    if (s[1] != ic) throw GraphError("shape-mismatch: conv2d channel count");
    const ConvGeometry geo = convGeometry(s[2], s[3], w[2], w[3], node);
    if (geo.outH <= 0 || geo.outW <= 0)
      throw GraphError("shape-mismatch: conv2d spatial dims not positive");
    return {s[0], node.transposed ? w[1] : w[0], geo.outH, geo.outW};
  }
  throw GraphError("unsupported-op: " + op);
}

}  // namespace

void checkGraph(const TensorGraph& g) {
  std::set<std::string> seen;
  for (const auto& t : g.tensors) {
    if (!seen.insert(t.id).second) throw GraphError("duplicate tensor id " + t.id);
    for (int64_t d : t.shape)
      if (d <= 0) throw GraphError("non-positive extent in tensor " + t.id);
  }
  std::set<std::string> defined;
  for (const auto& id : g.inputIds()) defined.insert(id);
  for (const auto& node : g.ops) {
    if (!kSupportedOps.count(node.op)) throw GraphError("unsupported-op: " + node.op);
    for (const auto& in : node.inputs) {
      if (!g.find(in)) throw GraphError("unknown tensor " + in);
      if (!defined.count(in)) throw GraphError("tensor " + in + " used before being produced");
    }
    const TensorDesc* out = g.find(node.output);
    if (!out) throw GraphError("unknown tensor " + node.output);
    if (expectedShape(g, node) != out->shape)
      throw GraphError("shape-mismatch: " + node.output +
                       " declared shape does not match op result");
    defined.insert(node.output);
  }
}

// ============================================================ executor ====
namespace {

// int8 matmul plumbing: graph ints live in f32 storage; K1c wants int8
// operands with 16-byte row pitches (B K-major) and returns int32 / int8.
__global__ void ints_to_i8_kernel(const float* __restrict__ x, int8_t* __restrict__ y,
                                  int64_t rows, int64_t cols, int64_t ldy, int transpose) {
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / cols, c = i % cols;
    const int8_t v = static_cast<int8_t>(x[i]);  // an i8 tensor holds exact values in [-128, 127]
    if (transpose) y[c * ldy + r] = v;  // x [rows = K, cols = N] -> y [N, K]
    else y[r * ldy + c] = v;
  }
}

__global__ void ints_to_f32_kernel(const void* __restrict__ x, float* __restrict__ y, int64_t n,
                                   int bytes) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    y[i] = bytes == 4 ? static_cast<float>(static_cast<const int32_t*>(x)[i])
                      : static_cast<float>(static_cast<const int8_t*>(x)[i]);
}

// Integer-typed matmul output other than the K1c case: the interpreter's
// nest exactly — C = 0; for k: C = store_int(fma(a, b, C)) with the I8 / I32
// store rounding nearbyint + saturate applied to every partial sum
// (frontend.cpp:679-733, interp.cpp:88-104, :502-561), one thread per output.
__global__ void int_matmul_sat_kernel(const float* __restrict__ a, const float* __restrict__ b,
                                      float* __restrict__ c, int64_t M, int64_t N, int64_t K,
                                      double lo, double hi) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < M * N;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / N, col = i % N;
    double acc = 0.0;
    for (int64_t k = 0; k < K; ++k) {
      acc = fma(static_cast<double>(a[r * K + k]), static_cast<double>(b[k * N + col]), acc);
      acc = fmin(fmax(nearbyint(acc), lo), hi);
    }
    c[i] = static_cast<float>(acc);
  }
}

unsigned elem_grid(int64_t n) {
  return static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 148 * 16));
}

// device storage type for a declared element type (ints carried exactly in f32)
afg_dtype dev_type(ElementType t) {
  switch (t) {
    case ElementType::F16: return AFG_F16;
    case ElementType::BF16: return AFG_BF16;
    default: return AFG_F32;
  }
}

uint16_t f32_to_f16_bits(float f) {  // RNE incl. subnormals (interp.cpp:25-60)
  uint32_t bits;
  std::memcpy(&bits, &f, 4);
  const uint32_t sign = (bits >> 16) & 0x8000u;
  if ((bits & 0x7f800000u) == 0x7f800000u)
    return static_cast<uint16_t>(sign | 0x7c00u | ((bits & 0x7fffffu) ? 0x200u : 0u));
  int32_t e = static_cast<int32_t>((bits >> 23) & 0xff) - 127 + 15;
  uint32_t m = bits & 0x7fffffu;
  if (e >= 31) return static_cast<uint16_t>(sign | 0x7c00u);
  if (e <= 0) {
    if (e < -10) return static_cast<uint16_t>(sign);
    m |= 0x800000u;
    const int shift = 14 - e;
    uint32_t h = m >> shift;
    const uint32_t rem = m & ((1u << shift) - 1), half = 1u << (shift - 1);
    if (rem > half || (rem == half && (h & 1))) ++h;
    return static_cast<uint16_t>(sign | h);
  }
  uint32_t h = m >> 13;
  const uint32_t rem = m & 0x1fffu;
  if (rem > 0x1000u || (rem == 0x1000u && (h & 1))) ++h;
  uint32_t c = (static_cast<uint32_t>(e) << 10) + h;
  if (c >= 0x7c00u) c = 0x7c00u;
  return static_cast<uint16_t>(sign | c);
}

double f16_bits_to_double(uint16_t h) {
  const uint32_t s = (h & 0x8000u) << 16, e = (h >> 10) & 0x1f, m = h & 0x3ffu;
  uint32_t ob;
  if (e == 0) {
    if (m == 0) {
      ob = s;
    } else {
      int k = -1;
      uint32_t mm = m;
      do {
        ++k;
        mm <<= 1;
      } while (!(mm & 0x400u));
      ob = s | (static_cast<uint32_t>(127 - 15 - k) << 23) | ((mm & 0x3ffu) << 13);
    }
  } else if (e == 31) {
    ob = s | 0x7f800000u | (m << 13);
  } else {
    ob = s | ((e - 15 + 127) << 23) | (m << 13);
  }
  float f;
  std::memcpy(&f, &ob, 4);
  return f;
}

uint16_t f32_to_bf16_bits(float f) {
  uint32_t b;
  std::memcpy(&b, &f, 4);
  if ((b & 0x7f800000u) == 0x7f800000u) return static_cast<uint16_t>(b >> 16);
  b += 0x7fffu + ((b >> 16) & 1u);
  return static_cast<uint16_t>(b >> 16);
}

double round_int(double v, double lo, double hi) {
  const double r = std::nearbyint(v);
  return r < lo ? lo : (r > hi ? hi : r);
}

struct DevBuf {
  void* ptr = nullptr;
  afg_dtype dt = AFG_F32;
  ElementType et = ElementType::F32;
  std::vector<int64_t> shape;
  int64_t n = 0;
};

class Executor {
 public:
  Executor(const TensorGraph& g, const GpuOptions& o, ExecStats* st)
      : g_(g), opt_(o), stats_(st), s_(static_cast<cudaStream_t>(o.stream)) {}
  ~Executor() {
    for (auto& kv : bufs_)
      if (kv.second.ptr) cudaFreeAsync(kv.second.ptr, s_);
    for (void* p : scratch_) cudaFreeAsync(p, s_);
    cudaStreamSynchronize(s_);
  }

  std::map<std::string, TensorValue> run(const std::map<std::string, TensorValue>& inputs) {
    checkGraph(g_);
    if (afg_device_count() == 0) throw InterpError("afg: no sm_100 device visible (no CPU fallback)");
    count_uses();
    // inputs: every graph input must be present, keyed "%id" (interp.cpp:202-210)
    for (const auto& id : g_.inputIds()) {
      auto it = inputs.find("%" + id);
      if (it == inputs.end()) it = inputs.find(id);
      if (it == inputs.end()) throw InterpError("missing input %" + id);
      const TensorDesc* d = g_.find(id);
      if (it->second.shape != d->shape) throw InterpError("input shape mismatch for %" + id);
      upload(*d, it->second);
    }
    size_t i = 0;
    while (i < g_.ops.size()) i += opt_.fuse ? try_fused(i) : run_op(i);
    std::map<std::string, TensorValue> out;
    for (const auto& id : g_.outputIds()) out["%" + id] = download(id);
    cudaError_t e = cudaStreamSynchronize(s_);
    if (e != cudaSuccess) throw InterpError(std::string("afg kernel failure: ") + cudaGetErrorString(e));
    return out;
  }

 private:
  const TensorGraph& g_;
  GpuOptions opt_;
  ExecStats* stats_;
  cudaStream_t s_;
  std::map<std::string, DevBuf> bufs_;
  std::map<std::string, int> uses_;
  std::set<std::string> outputs_;
  std::vector<void*> scratch_;

  void plan(const std::string& line) {
    if (stats_) stats_->plan.push_back(line);
  }
  static void ok(afg_status st) {
    if (st != AFG_OK) throw InterpError(std::string("afg: ") + afg_last_error());
  }
  void count_uses() {
    for (const auto& op : g_.ops)
      for (const auto& in : op.inputs) ++uses_[in];
    for (const auto& id : g_.outputIds()) outputs_.insert(id);
  }
  // intermediate that only feeds the next op of a chain and is not an output
  bool internal(const std::string& id) const {
    auto it = uses_.find(id);
    return it != uses_.end() && it->second == 1 && !outputs_.count(id);
  }

  DevBuf& alloc(const std::string& id) {
    const TensorDesc* d = g_.find(id);
    DevBuf b;
    b.et = d->dtype;
    b.dt = dev_type(d->dtype);
    b.shape = d->shape;
    b.n = 1;
    for (int64_t x : d->shape) b.n *= x;
    cudaError_t e = cudaMallocAsync(&b.ptr, std::max<int64_t>(b.n, 1) * dtype_bytes(b.dt) + 16, s_);
    if (e != cudaSuccess) throw InterpError(std::string("afg: device allocation failed: ") + cudaGetErrorString(e));
    auto& slot = bufs_[id];
    if (slot.ptr) cudaFreeAsync(slot.ptr, s_);
    slot = b;
    return slot;
  }
  void* scratch(size_t bytes) {
    void* p = nullptr;
    if (cudaMallocAsync(&p, bytes + 16, s_) != cudaSuccess) throw InterpError("afg: scratch allocation failed");
    scratch_.push_back(p);
    return p;
  }
  const DevBuf& buf(const std::string& id) {
    auto it = bufs_.find(id);
    if (it == bufs_.end()) throw InterpError("afg: tensor " + id + " not materialised");
    return it->second;
  }

  void upload(const TensorDesc& d, const TensorValue& v) {
    DevBuf& b = alloc(d.id);
    std::vector<uint8_t> host(static_cast<size_t>(b.n) * dtype_bytes(b.dt));
    for (int64_t i = 0; i < b.n; ++i) {
      double x = v.data[i];
      if (d.dtype == ElementType::I8) x = round_int(x, -128.0, 127.0);
      if (d.dtype == ElementType::I32) x = round_int(x, -2147483648.0, 2147483647.0);
      const float f = static_cast<float>(x);
      if (b.dt == AFG_F32) std::memcpy(&host[i * 4], &f, 4);
      else if (b.dt == AFG_F16) {
        const uint16_t h = f32_to_f16_bits(f);
        std::memcpy(&host[i * 2], &h, 2);
      } else {
        const uint16_t h = f32_to_bf16_bits(f);
        std::memcpy(&host[i * 2], &h, 2);
      }
    }
    cudaError_t e = cudaMemcpyAsync(b.ptr, host.data(), host.size(), cudaMemcpyHostToDevice, s_);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s_);
    if (e != cudaSuccess) throw InterpError(std::string("afg: upload failed: ") + cudaGetErrorString(e));
  }

  TensorValue download(const std::string& id) {
    const DevBuf& b = buf(id);
    std::vector<uint8_t> host(static_cast<size_t>(b.n) * dtype_bytes(b.dt));
    cudaError_t e = cudaMemcpyAsync(host.data(), b.ptr, host.size(), cudaMemcpyDeviceToHost, s_);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s_);
    if (e != cudaSuccess) throw InterpError(std::string("afg kernel failure: ") + cudaGetErrorString(e));
    TensorValue v;
    v.shape = b.shape;
    v.type = b.et;
    v.data.resize(b.n);
    for (int64_t i = 0; i < b.n; ++i) {
      if (b.dt == AFG_F32) {
        float f;
        std::memcpy(&f, &host[i * 4], 4);
        v.data[i] = f;
      } else if (b.dt == AFG_F16) {
        uint16_t h;
        std::memcpy(&h, &host[i * 2], 2);
        v.data[i] = f16_bits_to_double(h);
      } else {
        uint16_t h;
        std::memcpy(&h, &host[i * 2], 2);
        const uint32_t u = static_cast<uint32_t>(h) << 16;
        float f;
        std::memcpy(&f, &u, 4);
        v.data[i] = f;
      }
    }
    return v;
  }

  // Is the device tensor `id` identically zero (the ReLU constant)? Checked
  // on the device (reduce max|x| via max(x) and max(-x) on a small copy).
  bool is_zero_tensor(const std::string& id) {
    const DevBuf& b = buf(id);
    float* tmp = static_cast<float*>(scratch(sizeof(float)));
    ok(afg_reduce_lastdim(b.ptr, tmp, 1, b.n, AFG_REDUCE_MAXABS, b.dt, AFG_F32, s_));
    float h = 1.0f;
    cudaMemcpyAsync(&h, tmp, sizeof(h), cudaMemcpyDeviceToHost, s_);
    cudaStreamSynchronize(s_);
    return h == 0.0f;
  }

  // -------------------------------------------------------------- fusion --
  size_t try_fused(size_t i) {
    if (size_t n = fuse_matmul_epilogue(i)) return n;
    if (size_t n = fuse_attention(i)) return n;
    return run_op(i);
  }

  // matmul(a,b)->c ; broadcast_in_dim(bias,dims=[1])->bb ; add(c,bb)->cb [; max(cb,z)->y]
  size_t fuse_matmul_epilogue(size_t i) {
    const auto& ops = g_.ops;
    if (i + 2 >= ops.size() || ops[i].op != "matmul") return 0;
    const TensorOpNode& mm = ops[i];
    const TensorOpNode& bc = ops[i + 1];
    const TensorOpNode& ad = ops[i + 2];
    if (bc.op != "broadcast_in_dim" || ad.op != "add") return 0;
    const TensorDesc* c = g_.find(mm.output);
    const TensorDesc* bias = g_.find(bc.inputs[0]);
    if (bias->shape.size() != 1 || bc.dims != std::vector<int64_t>{1}) return 0;
    const bool order = (ad.inputs[0] == mm.output && ad.inputs[1] == bc.output) ||
                       (ad.inputs[1] == mm.output && ad.inputs[0] == bc.output);
    if (!order || !internal(mm.output) || !internal(bc.output)) return 0;
    const TensorDesc* a = g_.find(mm.inputs[0]);
    const TensorDesc* bm = g_.find(mm.inputs[1]);
    const TensorDesc* y = g_.find(ad.output);
    // every intermediate store must round to the same type for the fused
    // epilogue to be the graph's semantics: c, bb, cb (and y) share one type
    if (y->dtype != c->dtype || g_.find(bc.output)->dtype != c->dtype || bias->dtype != ElementType::F32 ||
        a->dtype != bm->dtype || a->dtype == ElementType::I8 || a->dtype == ElementType::I32)
      return 0;
    afg_epilogue epi = AFG_EPI_BIAS;
    size_t consumed = 3;
    std::string out_id = ad.output;
    if (i + 3 < ops.size() && ops[i + 3].op == "max" && internal(ad.output)) {
      const TensorOpNode& mx = ops[i + 3];
      const std::string other = mx.inputs[0] == ad.output ? mx.inputs[1] : mx.inputs[0];
      if ((mx.inputs[0] == ad.output || mx.inputs[1] == ad.output) && other != ad.output &&
          bufs_.count(other) && g_.find(mx.output)->dtype == c->dtype && is_zero_tensor(other)) {
        epi = AFG_EPI_BIAS_RELU;
        consumed = 4;
        out_id = mx.output;
      }
    }
    const DevBuf& A = buf(mm.inputs[0]);
    const DevBuf& B = buf(mm.inputs[1]);
    const DevBuf& Bias = buf(bc.inputs[0]);
    DevBuf& C = alloc(out_id);
    const int64_t M = a->shape[0], K = a->shape[1], N = bm->shape[1];
    ok(afg_gemm(A.ptr, K, B.ptr, N, static_cast<const float*>(Bias.ptr), nullptr, C.ptr, N, M, N,
                K, A.dt, C.dt, AFG_B_KN, epi, s_));
    plan("afg_gemm[" + std::to_string(M) + "x" + std::to_string(N) + "x" + std::to_string(K) +
         (epi == AFG_EPI_BIAS_RELU ? "] +bias+relu epilogue" : "] +bias epilogue") + " <- " +
         mm.output + "," + bc.output + "," + ad.output + (consumed == 4 ? "," + out_id : ""));
    if (stats_) ++stats_->fused;
    return consumed;
  }

  // transpose(k)->kt ; batch_matmul(q,kt)->qk ; [add(qk,bias)->qkb] ; softmax->soft ;
  // batch_matmul(soft, v)->out
  size_t fuse_attention(size_t i) {
    const auto& ops = g_.ops;
    if (i + 3 >= ops.size() || ops[i].op != "transpose") return 0;
    const TensorOpNode& tr = ops[i];
    const TensorDesc* k = g_.find(tr.inputs[0]);
    const size_t r = k->shape.size();
    if (r != 4) return 0;
    if (tr.perm != std::vector<int64_t>{0, 1, 3, 2}) return 0;
    const TensorOpNode& qk = ops[i + 1];
    if (qk.op != "batch_matmul" || qk.inputs.size() != 2 || qk.inputs[1] != tr.output) return 0;
    size_t j = i + 2;
    std::string scores = qk.output;
    const TensorOpNode* add = nullptr;
    if (ops[j].op == "add") {
      add = &ops[j];
      if (!(add->inputs[0] == scores || add->inputs[1] == scores)) return 0;
      scores = add->output;
      ++j;
    }
    if (j + 1 >= ops.size()) return 0;
    const TensorOpNode& sm = ops[j];
    const TensorOpNode& pv = ops[j + 1];
    if (sm.op != "softmax" || sm.inputs[0] != scores || (sm.axis != -1 && sm.axis != 3)) return 0;
    if (pv.op != "batch_matmul" || pv.inputs[0] != sm.output) return 0;
    if (!internal(tr.output) || !internal(qk.output) || !internal(sm.output) ||
        (add && !internal(add->output)))
      return 0;
    const TensorDesc* q = g_.find(qk.inputs[0]);
    const TensorDesc* v = g_.find(pv.inputs[1]);
    const TensorDesc* o = g_.find(pv.output);
    if (q->dtype != k->dtype || v->dtype != k->dtype || q->shape[3] != k->shape[3] ||
        v->shape[3] != q->shape[3] || q->dtype == ElementType::I8 || q->dtype == ElementType::I32)
      return 0;
    // intermediate stores (scores, probabilities) must be f32 like the paper's
    // mixed-precision graph for the fused kernel's fp32
    // softmax to be the graph's semantics
    for (const std::string& id : {qk.output, sm.output})
      if (g_.find(id)->dtype != ElementType::F32) return 0;
    const std::string bias_id = add ? (add->inputs[0] == qk.output ? add->inputs[1] : add->inputs[0]) : "";
    if (add && (g_.find(bias_id)->dtype != ElementType::F32 || g_.find(add->output)->dtype != ElementType::F32))
      return 0;
    const DevBuf& Q = buf(qk.inputs[0]);
    const DevBuf& K = buf(tr.inputs[0]);
    const DevBuf& V = buf(pv.inputs[1]);
    const float* bias = add ? static_cast<const float*>(buf(bias_id).ptr) : nullptr;
    DevBuf& O = alloc(pv.output);
    ok(afg_attention_fwd(Q.ptr, K.ptr, V.ptr, bias, O.ptr, q->shape[0], q->shape[1], q->shape[2],
                         k->shape[2], q->shape[3], 1.0f, 0, Q.dt, dev_type(o->dtype), s_));
    plan("afg_attention_fwd[" + std::to_string(q->shape[0]) + "x" + std::to_string(q->shape[1]) +
         "x" + std::to_string(q->shape[2]) + "x" + std::to_string(q->shape[3]) + "]" +
         (add ? " +bias" : "") + " <- " + std::to_string(j + 2 - i) + " ops");
    if (stats_) ++stats_->fused;
    return j + 2 - i;
  }

  // --------------------------------------------------------- single ops --
  size_t run_op(size_t i) {
    const TensorOpNode& n = g_.ops[i];
    const TensorDesc* od = g_.find(n.output);
    auto in = [&](size_t k) -> const DevBuf& { return buf(n.inputs.at(k)); };
    const std::string& op = n.op;
    if (op == "add" || op == "sub" || op == "mul" || op == "max") {
      const afg_binop bop = op == "add" ? AFG_OP_ADD : op == "sub" ? AFG_OP_SUB : op == "mul" ? AFG_OP_MUL : AFG_OP_MAX;
      const DevBuf& a = in(0);
      const DevBuf& b = in(1);
      DevBuf& y = alloc(n.output);
      ok(afg_elementwise(a.ptr, b.ptr, y.ptr, y.n, 0, bop, a.dt, b.dt, y.dt, s_));
      round_int_out(y);
      plan("afg_elementwise[" + op + "] -> " + n.output);
    } else if (op == "exp") {
      const DevBuf& a = in(0);
      DevBuf& y = alloc(n.output);
      ok(afg_elementwise(a.ptr, nullptr, y.ptr, y.n, 0, AFG_OP_EXP, a.dt, a.dt, y.dt, s_));
      round_int_out(y);
      plan("afg_elementwise[exp] -> " + n.output);
    } else if (op == "transpose") {
      const DevBuf& a = in(0);
      DevBuf& y = alloc(n.output);
      const DevBuf* src = &a;
      void* conv = nullptr;
      if (a.dt != y.dt) {
        conv = scratch(a.n * dtype_bytes(y.dt));
        ok(afg_convert(a.ptr, conv, a.n, a.dt, y.dt, s_));
      }
      ok(afg_transpose(conv ? conv : src->ptr, y.ptr, static_cast<int>(a.shape.size()), a.shape.data(),
                       n.perm.data(), y.dt, s_));
      plan("afg_transpose -> " + n.output);
    } else if (op == "broadcast_in_dim") {
      const DevBuf& a = in(0);
      DevBuf& y = alloc(n.output);
      ok(afg_broadcast_in_dim(a.ptr, y.ptr, static_cast<int>(a.shape.size()), a.shape.data(),
                              static_cast<int>(y.shape.size()), y.shape.data(), n.dims.data(),
                              a.dt, y.dt, s_));
      plan("afg_broadcast_in_dim -> " + n.output);
    } else if (op == "reshape") {
      const DevBuf& a = in(0);
      DevBuf& y = alloc(n.output);
      ok(afg_convert(a.ptr, y.ptr, a.n, a.dt, y.dt, s_));
      round_int_out(y);
      plan("afg_convert[reshape] -> " + n.output);
    } else if (op == "reduce") {
      run_reduce(n);
    } else if (op == "softmax") {
      const DevBuf& a = in(0);
      DevBuf& y = alloc(n.output);
      const int64_t rank = static_cast<int64_t>(a.shape.size());
      const int64_t axis = n.axis < 0 ? n.axis + rank : n.axis;
      if (axis != rank - 1) throw InterpError("afg: softmax over a non-last axis is not supported");
      const int64_t cols = a.shape.back();
      ok(afg_softmax_lastdim(a.ptr, y.ptr, a.n / cols, cols, a.dt, y.dt, s_));
      plan("afg_softmax_lastdim -> " + n.output);
    } else if (op == "matmul" && in(0).et == ElementType::I8 && in(1).et == ElementType::I8 &&
               g_.find(n.output) && g_.find(n.output)->dtype == ElementType::I32) {
      // i8 x i8 -> i32 (the quant path): exact integer
      // accumulation on K1c (the interpreter's per-step I32 stores never
      // saturate for K < 131072). An i8 OUTPUT is not routed here: the
      // interpreter saturates every partial sum (e.g. 100+100-100 -> 27).
      const DevBuf& a = in(0);
      const DevBuf& b = in(1);
      DevBuf& y = alloc(n.output);
      const int64_t M = a.shape[0], K = a.shape[1], N = b.shape[1];
      const int64_t Kp = (K + 15) / 16 * 16;
      int8_t* a8 = static_cast<int8_t*>(scratch(static_cast<size_t>(M * Kp)));
      int8_t* b8 = static_cast<int8_t*>(scratch(static_cast<size_t>(N * Kp)));
      ints_to_i8_kernel<<<elem_grid(M * K), 256, 0, s_>>>(static_cast<const float*>(a.ptr), a8, M,
                                                           K, Kp, 0);
      ints_to_i8_kernel<<<elem_grid(K * N), 256, 0, s_>>>(static_cast<const float*>(b.ptr), b8, K,
                                                           N, Kp, 1);
      count_launch(2);
      const bool i32 = true;
      void* c = scratch(static_cast<size_t>(M * N * (i32 ? 4 : 1)));
      ok(afg_gemm_i8(a8, Kp, b8, Kp, c, N, M, N, K, i32 ? 0 : 1, 1.0f, s_));
      ints_to_f32_kernel<<<elem_grid(M * N), 256, 0, s_>>>(c, static_cast<float*>(y.ptr), M * N,
                                                            i32 ? 4 : 1);
      count_launch();
      ok(cuda_status(cudaGetLastError(), "graph int8 matmul conversions"));
      plan("afg_gemm_i8 -> " + n.output);
    } else if (op == "matmul" && g_.find(n.output) &&
               (g_.find(n.output)->dtype == ElementType::I8 ||
                g_.find(n.output)->dtype == ElementType::I32) &&
               in(0).dt == AFG_F32 && in(1).dt == AFG_F32) {
      const DevBuf& a = in(0);
      const DevBuf& b = in(1);
      DevBuf& y = alloc(n.output);
      const int64_t M = a.shape[0], K = a.shape[1], N = b.shape[1];
      const bool i8 = y.et == ElementType::I8;
      int_matmul_sat_kernel<<<elem_grid(M * N), 256, 0, s_>>>(
          static_cast<const float*>(a.ptr), static_cast<const float*>(b.ptr),
          static_cast<float*>(y.ptr), M, N, K, i8 ? -128.0 : -2147483648.0,
          i8 ? 127.0 : 2147483647.0);
      count_launch();
      ok(cuda_status(cudaGetLastError(), "graph integer matmul"));
      plan("int_matmul_sat -> " + n.output);
    } else if (op == "matmul") {
      const DevBuf& a = in(0);
      const DevBuf& b = in(1);
      DevBuf& y = alloc(n.output);
      const int64_t M = a.shape[0], K = a.shape[1], N = b.shape[1];
      ok(afg_gemm(a.ptr, K, b.ptr, N, nullptr, nullptr, y.ptr, N, M, N, K, a.dt, y.dt, AFG_B_KN,
                  AFG_EPI_NONE, s_));
      round_int_out(y);
      plan("afg_gemm -> " + n.output);
    } else if (op == "batch_matmul") {
      const DevBuf& a = in(0);
      const DevBuf& b = in(1);
      DevBuf& y = alloc(n.output);
      const int64_t M = a.shape[a.shape.size() - 2], K = a.shape.back(), N = b.shape.back();
      ok(afg_gemm_batched(a.ptr, b.ptr, y.ptr, a.n / (M * K), M, N, K, a.dt, y.dt, s_));
      plan("afg_gemm_batched -> " + n.output);
    } else if (op == "conv2d") {
      const DevBuf& x = in(0);
      const DevBuf& w = in(1);
      DevBuf& y = alloc(n.output);
      const ConvGeometry geo = convGeometry(x.shape[2], x.shape[3], w.shape[2], w.shape[3], n);
      ok(afg_conv2d_nchw(x.ptr, w.ptr, y.ptr, x.shape[0], x.shape[1], x.shape[2], x.shape[3],
                         y.shape[1], w.shape[2], w.shape[3], n.strideY, n.strideX, n.dilY, n.dilX,
                         geo.padY, geo.padX, n.transposed ? 1 : 0, geo.outH, geo.outW, x.dt, y.dt,
                         s_));
      plan("afg_conv2d_nchw -> " + n.output);
    } else if (op == "quantize" || op == "dequantize") {
      const DevBuf& a = in(0);
      DevBuf& y = alloc(n.output);
      ok(afg_quantize(a.ptr, y.ptr, a.n, static_cast<float>(n.scale), op == "quantize" ? 0 : 1,
                      a.dt, y.dt, s_));
      round_int_out(y);
      plan("afg_quantize[" + op + "] -> " + n.output);
    } else {
      throw GraphError("unsupported-op: " + op);
    }
    return 1;
  }

  // integer-declared outputs: round + saturate like roundToType (interp.cpp:94-101)
  void round_int_out(DevBuf& y) {
    if (y.et == ElementType::I8)
      ok(afg_quantize(y.ptr, y.ptr, y.n, 1.0f, 2, y.dt, y.dt, s_));
    else if (y.et == ElementType::I32)
      ok(afg_quantize(y.ptr, y.ptr, y.n, 1.0f, 3, y.dt, y.dt, s_));
  }

  void run_reduce(const TensorOpNode& n) {
    const DevBuf& a = buf(n.inputs[0]);
    DevBuf& y = alloc(n.output);
    const int64_t rank = static_cast<int64_t>(a.shape.size());
    const int64_t axis = n.axis < 0 ? n.axis + rank : n.axis;
    const afg_reduce_kind kind = n.reduceOp == "max" ? AFG_REDUCE_MAX : AFG_REDUCE_SUM;
    const void* src = a.ptr;
    if (axis != rank - 1) {  // move the reduced axis last
      std::vector<int64_t> perm;
      for (int64_t d = 0; d < rank; ++d)
        if (d != axis) perm.push_back(d);
      perm.push_back(axis);
      void* t = scratch(a.n * dtype_bytes(a.dt));
      ok(afg_transpose(a.ptr, t, static_cast<int>(rank), a.shape.data(), perm.data(), a.dt, s_));
      src = t;
    }
    const int64_t cols = a.shape[axis];
    ok(afg_reduce_lastdim(src, y.ptr, a.n / cols, cols, kind, a.dt, y.dt, s_));
    round_int_out(y);
    plan("afg_reduce_lastdim[" + n.reduceOp + "] -> " + n.output);
  }
};

}  // namespace

std::map<std::string, TensorValue> execute(const TensorGraph& g,
                                           const std::map<std::string, TensorValue>& inputs,
                                           const GpuOptions& opt, ExecStats* stats) {
  Executor ex(g, opt, stats);
  return ex.run(inputs);
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
                                 const double* const* data, const int64_t* numel, int fuse,
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
      if (!id.empty() && id[0] == '%') id = id.substr(1);
      const TensorDesc* d = g.find(id);
      if (!d) throw InterpError("unknown input " + id);
      TensorValue v;
      v.shape = d->shape;
      v.type = d->dtype;
      if (v.numElements() != numel[i]) throw InterpError("input shape mismatch for %" + id);
      v.data.assign(data[i], data[i] + numel[i]);
      inputs["%" + id] = std::move(v);
    }
    GpuOptions opt;
    opt.stream = stream;
    opt.fuse = fuse != 0;
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
    afg::gpu::checkGraph(afg::gpu::parseGraphJson(graph_json ? graph_json : ""));
    return AFG_OK;
  } catch (const std::exception& e) {
    return afg::set_error(AFG_ERR_INVALID_ARG, "GraphError: %s", e.what());
  }
}

}  // extern "C"
