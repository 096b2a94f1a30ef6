// af_gpu.h - the adapter a reference maintainer adds next to af/interp.h to
// run lowered graphs on a B200 through afg. It is written
// against the reference's own types (af::TensorGraph, af::TensorValue,
// af::GraphError, af::InterpError, frontend.h:24-80, interp.h:29-125) and
// only forwards to afg::gpu::execute (include/afg_graph.h).
#pragma once

#include <map>
#include <string>

#include "af/frontend.h"
#include "af/interp.h"

namespace af {
namespace gpu {

struct GpuOptions {
  void* stream = nullptr;
  bool fuse = true;
};

/// Drop-in for `interpret(lowerGraphToAffine(g, cfg), inputs).outputs`:
/// same input keys ("%id"), same output keys and element-type rounding.
/// Throws af::GraphError / af::InterpError like the reference.
std::map<std::string, TensorValue> execute(const TensorGraph& g,
                                           const std::map<std::string, TensorValue>& inputs,
                                           const GpuOptions& opt = {});

}  // namespace gpu
}  // namespace af
