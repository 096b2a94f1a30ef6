// afg_graph.h - C++ host API mirroring the reference's graph/operator API
// (AffineForge, /root/reference/proj/include/af/frontend.h:24-80 and
// af/interp.h:29-125) on top of the afg C ABI (afg.h).
//
// A maintainer swaps executors in one line: where the reference test does
//     af::Program p = af::lowerGraphToAffine(g, af::TargetConfig{});
//     auto result = af::interpret(p, inputs);          // interp.h:97-100
// the B200 path is
//     auto outputs = afg::gpu::execute(g, inputs);      // same keys "%id"
// with the same input contract (a value for every graph input, keyed "%id",
// shape-checked) and the same outputs (declared outputs or produced-and-never-
// consumed tensors, keyed "%id", values rounded to the declared element
// type). Errors are the reference's: GraphError for malformed graphs /
// unsupported ops / shape mismatches, InterpError for missing or mis-shaped
// inputs and execution failures. See INTEGRATION.md for the adapter from the
// reference's own af:: types.
#pragma once

#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#if defined(__GNUC__)
#pragma GCC visibility push(default)  // exported from libafg.so (built -fvisibility=hidden)
#endif

namespace afg {
namespace gpu {

// af::ElementType order (ir.h:29) + BF16 (additive extension).
enum class ElementType { F32 = 0, F16 = 1, I8 = 2, I32 = 3, BF16 = 10 };

struct GraphError : public std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InterpError : public std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct TensorDesc {  // frontend.h:30-34
  std::string id;
  std::vector<int64_t> shape;
  ElementType dtype = ElementType::F32;
};

struct TensorOpNode {  // frontend.h:36-50
  std::string op;
  std::vector<std::string> inputs;
  std::string output;
  std::vector<int64_t> perm;
  std::vector<int64_t> dims;
  int64_t strideY = 1, strideX = 1;
  int64_t dilY = 1, dilX = 1;
  bool samePadding = false;
  bool transposed = false;
  std::string reduceOp;
  int64_t axis = -1;
  double scale = 1.0;
};

struct TensorGraph {  // frontend.h:52-60
  std::vector<TensorDesc> tensors;
  std::vector<TensorOpNode> ops;
  std::vector<std::string> outputs;
  const TensorDesc* find(const std::string& id) const;
  std::vector<std::string> inputIds() const;
  std::vector<std::string> outputIds() const;
};

struct TensorValue {  // interp.h:33-44
  std::vector<int64_t> shape;
  ElementType type = ElementType::F32;
  std::vector<double> data;
  // Optional non-owning view of numElements() doubles, read instead of `data`
  // when set (an input the caller keeps alive for the call: the C ABI and the
  // adapter pass their buffers without copying them). Outputs use `data`.
  const double* view = nullptr;
  const double* values() const { return view ? view : data.data(); }
  int64_t numElements() const {
    int64_t n = 1;
    for (int64_t d : shape) n *= d;
    return n;
  }
};

// Reads the graph JSON schema of parseGraphJson (frontend.cpp:57-113).
TensorGraph parseGraphJson(const std::string& text);
// Table-driven validation with checkGraph's error behaviour
// (frontend.cpp:159-294): GraphError "unsupported-op: ...", "shape-mismatch:
// ...", unknown / duplicate / used-before-produced tensors, non-positive
// extents. (A C++ caller holding an af::TensorGraph runs the reference's own
// af::checkGraph first, integration/af_gpu.cpp.)
void validateGraph(const TensorGraph& g);

struct GpuOptions {
  void* stream = nullptr;     // cudaStream_t; NULL = legacy default stream
  bool fuse = true;           // kernel patterns + fused VM regions (else one launch per op)
  bool tensor_cores = true;   // f32 tensors holding exact bf16 / f16 values run on
                              // tcgen05 (fp32 accumulation; stated tolerance
                              // instead of bit-exactness); false = exact paths only
  // Multi-GPU: with more than one entry the graph runs as one
  // shard per entry on a thread-per-device group (include/afg_multi.h), the
  // leading (batch / row) dimension of every graph input whose extent is
  // shard_extent split into contiguous blocks; the split is propagated through
  // the ops (elementwise, matmul rows, batch_matmul, conv batch, transposes /
  // reshapes / reductions that keep dim 0, broadcasts into it) and outputs are
  // concatenated back. A graph that mixes rows across shards is a GraphError
  // ("not shardable"). Entries may repeat a device (shards then share it).
  std::vector<int> devices;
  int64_t shard_extent = 0;  // 0: the leading extent of the first graph input
};

struct ExecStats {
  std::vector<std::string> plan;  // one line per launched kernel group
  int fused = 0;                  // number of fused chains
};

// Executes the graph on the current CUDA device. inputs keyed "%id".
std::map<std::string, TensorValue> execute(const TensorGraph& g,
                                           const std::map<std::string, TensorValue>& inputs,
                                           const GpuOptions& opt = {}, ExecStats* stats = nullptr);

}  // namespace gpu
}  // namespace afg

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
