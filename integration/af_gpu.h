// af_gpu.h - the adapter a reference maintainer adds next to af/interp.h to
// run lowered graphs and programs on a B200 through afg. It
// is written against the reference's own types (af::TensorGraph,
// af::Program, af::TensorValue, af::InterpResult, af::GraphError,
// af::InterpError; frontend.h:24-80, ir.h:36-318, interp.h:29-125) and only
// converts to / from the afg::gpu mirrors (include/afg_graph.h,
// include/afg_nest.h).
#pragma once

#include <map>
#include <string>

#include "af/frontend.h"
#include "af/interp.h"

namespace af {
namespace gpu {

struct GpuOptions {
  void* stream = nullptr;
  bool fuse = true;          // kernel patterns + fused regions
  bool tensor_cores = true;  // bf16 / f16-valued f32 tensors on tcgen05 (stated tolerance)
};

/// Drop-in for `interpret(lowerGraphToAffine(g, cfg), inputs).outputs`:
/// same input keys ("%id"), same output keys and element-type rounding.
/// Runs the reference's own af::checkGraph first; throws af::GraphError /
/// af::InterpError like the reference.
std::map<std::string, TensorValue> execute(const TensorGraph& g,
                                           const std::map<std::string, TensorValue>& inputs,
                                           const GpuOptions& opt = {});

/// Drop-in for af::interpret (interp.h:97-100) with the same signature and
/// InterpResult: outputs keyed by buffer id, metrics counted like the
/// interpreter (global / shared / register traffic, per buffer, flops,
/// fragment and correction ops, nest count). InterpOptions::traceBuffer and
/// checkParallelConflicts are not supported on the GPU (the trace stays
/// empty; conflicting parallel writes are not diagnosed).
InterpResult interpret(const Program& p, const std::map<std::string, TensorValue>& inputs,
                       const InterpOptions& options = {}, const std::string& funcName = "");

}  // namespace gpu
}  // namespace af
