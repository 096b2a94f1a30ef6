// af_gpu.cpp - af:: <-> afg::gpu:: adapter (see af_gpu.h).
#include "af_gpu.h"

#include "../include/afg_graph.h"
#include "../include/afg_nest.h"

namespace af {
namespace gpu {

namespace {

afg::gpu::ElementType to_afg(ElementType t) {
  switch (t) {
    case ElementType::F16: return afg::gpu::ElementType::F16;
    case ElementType::I8: return afg::gpu::ElementType::I8;
    case ElementType::I32: return afg::gpu::ElementType::I32;
    default: return afg::gpu::ElementType::F32;
  }
}

ElementType to_af(afg::gpu::ElementType t) {
  switch (t) {
    case afg::gpu::ElementType::F16: return ElementType::F16;
    case afg::gpu::ElementType::I8: return ElementType::I8;
    case afg::gpu::ElementType::I32: return ElementType::I32;
    default: return ElementType::F32;
  }
}

std::map<std::string, afg::gpu::TensorValue> to_afg(const std::map<std::string, TensorValue>& in) {
  std::map<std::string, afg::gpu::TensorValue> out;
  for (const auto& [k, v] : in) {  // views of the caller's values: no host copy
    afg::gpu::TensorValue t;
    t.shape = v.shape;
    t.type = to_afg(v.type);
    t.view = v.data.data();
    if (static_cast<int64_t>(v.data.size()) != t.numElements()) t.data = v.data;  // let the executor report it
    if (!t.data.empty()) t.view = nullptr;
    out[k] = std::move(t);
  }
  return out;
}

std::map<std::string, TensorValue> to_af(std::map<std::string, afg::gpu::TensorValue>&& in) {
  std::map<std::string, TensorValue> out;
  for (auto& [k, v] : in) {
    TensorValue tv;
    tv.shape = v.shape;
    tv.type = to_af(v.type);
    tv.data = std::move(v.data);
    out[k] = std::move(tv);
  }
  return out;
}

// AffineExpr tree -> postfix index program (affine.h:21-80)
void flatten(const AffineExpr& e, std::vector<int64_t>& code) {
  using K = AffineExpr::Kind;
  using C = afg::gpu::IndexExpr;
  switch (e.kind()) {
    case K::Constant: code.insert(code.end(), {C::Const, e.value()}); break;
    case K::Dim: code.insert(code.end(), {C::Dim, static_cast<int64_t>(e.index())}); break;
    case K::Symbol: throw InterpError("afg: affine symbols are not supported");
    case K::Add:
      flatten(e.lhs(), code);
      flatten(e.rhs(), code);
      code.push_back(C::Add);
      break;
    case K::MulConst:
      flatten(e.lhs(), code);
      code.insert(code.end(), {C::MulConst, e.rhsConstant()});
      break;
    case K::FloorDiv:
      flatten(e.lhs(), code);
      code.insert(code.end(), {C::FloorDiv, e.rhsConstant()});
      break;
    case K::Mod:
      flatten(e.lhs(), code);
      code.insert(code.end(), {C::Mod, e.rhsConstant()});
      break;
  }
}

std::vector<afg::gpu::IndexExpr> results(const AffineMap& m) {
  std::vector<afg::gpu::IndexExpr> out;
  for (const auto& r : m.results) {
    afg::gpu::IndexExpr e;
    flatten(r, e.code);
    out.push_back(std::move(e));
  }
  return out;
}

afg::gpu::NestOp convert(const Op& op) {
  afg::gpu::NestOp n;
  n.kind = static_cast<afg::gpu::NestOpKind>(static_cast<int>(op.kind));
  for (const auto& [k, v] : op.attrs) {
    afg::gpu::NestAttr a;
    a.kind = static_cast<afg::gpu::NestAttr::Kind>(static_cast<int>(v.kind));
    a.i = v.i;
    a.s = v.s;
    n.attrs[k] = a;
  }
  if (op.kind == OpKind::For) {
    n.ivs = {op.iv};
    n.lowers = {results(op.lower)};
    n.uppers = {results(op.upper)};
  } else if (op.kind == OpKind::Parallel) {
    n.ivs = op.ivs;
    for (const auto& m : op.lowers) n.lowers.push_back(results(m));
    for (const auto& m : op.uppers) n.uppers.push_back(results(m));
  }
  n.boundOperands = op.mapOperands;
  n.step = op.step;
  for (const auto& c : op.body) n.body.push_back(convert(c));
  n.buffer = op.buffer;
  n.access = results(op.access);
  n.accessOperands = op.accessOperands;
  n.result = op.result;
  n.arith = static_cast<afg::gpu::ArithOp>(static_cast<int>(op.arith));
  for (const auto& o : op.operands) n.operands.push_back({o.isImm, o.value, o.imm});
  n.castType = to_afg(op.castType);
  n.scale = op.scale;
  n.mmaRole = static_cast<int>(op.mmaRole);
  n.tag = op.tag;
  n.srcBuffer = op.srcBuffer;
  return n;
}

void fill(SpaceCounters& s, const afg::gpu::NestCounters& c) {
  s.loads = c.loads;
  s.stores = c.stores;
  s.loadBytes = c.loadBytes;
  s.storeBytes = c.storeBytes;
}

}  // namespace

std::map<std::string, TensorValue> execute(const TensorGraph& g,
                                           const std::map<std::string, TensorValue>& inputs,
                                           const GpuOptions& opt) {
  checkGraph(g);  // the reference's own validation (frontend.cpp:264-294)
  afg::gpu::TensorGraph ag;
  for (const auto& t : g.tensors) ag.tensors.push_back({t.id, t.shape, to_afg(t.dtype)});
  for (const auto& n : g.ops) {
    afg::gpu::TensorOpNode m;
    m.op = n.op;
    m.inputs = n.inputs;
    m.output = n.output;
    m.perm = n.perm;
    m.dims = n.dims;
    m.strideY = n.strideY;
    m.strideX = n.strideX;
    m.dilY = n.dilY;
    m.dilX = n.dilX;
    m.samePadding = n.samePadding;
    m.transposed = n.transposed;
    m.reduceOp = n.reduceOp;
    m.axis = n.axis;
    m.scale = n.scale;
    ag.ops.push_back(std::move(m));
  }
  ag.outputs = g.outputs;
  afg::gpu::GpuOptions o;
  o.stream = opt.stream;
  o.fuse = opt.fuse;
  o.tensor_cores = opt.tensor_cores;
  try {
    return to_af(afg::gpu::execute(ag, to_afg(inputs), o));
  } catch (const afg::gpu::GraphError& e) {
    throw GraphError(e.what());
  } catch (const afg::gpu::InterpError& e) {
    throw InterpError(e.what());
  }
}

InterpResult interpret(const Program& p, const std::map<std::string, TensorValue>& inputs,
                       const InterpOptions& options, const std::string& funcName) {
  (void)options;
  const Function* fn = nullptr;  // interp.cpp:172-183
  if (funcName.empty()) {
    fn = p.findFunction("main");
    if (!fn && p.functions.size() == 1) fn = &p.functions[0];
  } else {
    fn = p.findFunction(funcName);
  }
  if (!fn) throw InterpError("no such function: " + (funcName.empty() ? "main" : funcName));
  afg::gpu::NestProgram np;
  for (const auto& b : p.buffers) {
    afg::gpu::NestBuffer nb;
    nb.id = b.id;
    nb.shape = b.shape;
    nb.dtype = to_afg(b.elementType);
    nb.space = static_cast<afg::gpu::MemSpace>(static_cast<int>(b.space));
    nb.isInput = b.isInput;
    nb.isOutput = b.isOutput;
    np.buffers.push_back(std::move(nb));
  }
  InterpResult res;
  afg::gpu::NestMetrics m;
  afg::gpu::NestRunOptions o;
  o.count_metrics = true;
  try {
    for (const auto& op : fn->body) np.body.push_back(convert(op));
    res.outputs = to_af(afg::gpu::run_program(np, to_afg(inputs), o, &m));
  } catch (const afg::gpu::InterpError& e) {
    throw InterpError(e.what());
  }
  fill(res.metrics.global, m.global);
  fill(res.metrics.shared, m.shared);
  fill(res.metrics.registers, m.registers);
  res.metrics.flops = m.flops;
  res.metrics.fragmentLoads = m.fragmentLoads;
  res.metrics.fragmentComputes = m.fragmentComputes;
  res.metrics.fragmentStores = m.fragmentStores;
  res.metrics.nestCount = m.nestCount;
  res.metrics.correctionOps = m.correctionOps;
  for (const auto& [id, c] : m.perBuffer) {
    BufferCounters bc;
    bc.loads = c.loads;
    bc.stores = c.stores;
    bc.loadBytes = c.loadBytes;
    bc.storeBytes = c.storeBytes;
    auto sp = m.perBufferSpace.find(id);
    bc.space = sp == m.perBufferSpace.end() ? MemorySpace::Global
                                            : static_cast<MemorySpace>(static_cast<int>(sp->second));
    res.metrics.perBuffer[id] = bc;
  }
  return res;
}

}  // namespace gpu
}  // namespace af
