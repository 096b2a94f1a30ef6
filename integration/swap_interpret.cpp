// swap_interpret.cpp - TEST INFRASTRUCTURE: routes the reference suites'
// af::interpret calls to the B200 executor. The suites (and testsupport.cpp)
// are compiled with -Dinterpret=afg_swapped_interpret, which renames the
// declaration in af/interp.h and every call in those translation units; this
// file (compiled without the macro) defines the renamed function on top of
// the adapter af::gpu::interpret (integration/af_gpu.h).
#include "af_gpu.h"

namespace af {
InterpResult afg_swapped_interpret(const Program& p,
                                   const std::map<std::string, TensorValue>& inputs,
                                   const InterpOptions& options, const std::string& funcName) {
  return gpu::interpret(p, inputs, options, funcName);
}
}  // namespace af
