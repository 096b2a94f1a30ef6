// af_gpu.cpp - af:: <-> afg::gpu:: adapter (see af_gpu.h).
#include "af_gpu.h"

#include "../include/afg_graph.h"

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

}  // namespace

std::map<std::string, TensorValue> execute(const TensorGraph& g,
                                           const std::map<std::string, TensorValue>& inputs,
                                           const GpuOptions& opt) {
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
  std::map<std::string, afg::gpu::TensorValue> ain;
  for (const auto& [k, v] : inputs) ain[k] = {v.shape, to_afg(v.type), v.data};
  afg::gpu::GpuOptions o;
  o.stream = opt.stream;
  o.fuse = opt.fuse;
  std::map<std::string, afg::gpu::TensorValue> aout;
  try {
    aout = afg::gpu::execute(ag, ain, o);
  } catch (const afg::gpu::GraphError& e) {
    throw GraphError(e.what());
  } catch (const afg::gpu::InterpError& e) {
    throw InterpError(e.what());
  }
  std::map<std::string, TensorValue> out;
  for (auto& [k, v] : aout) {
    TensorValue tv;
    tv.shape = v.shape;
    tv.type = to_af(v.type);
    tv.data = std::move(v.data);
    out[k] = std::move(tv);
  }
  return out;
}

}  // namespace gpu
}  // namespace af
