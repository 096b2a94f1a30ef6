// nestvm.h - internal interface of the nest VM (nestvm.cu), shared by the
// program executor (af::interpret drop-in, nestexec.cpp) and the graph
// planner's fused pointwise / reduction regions (graph.cpp).
//
// A NestOp tree (include/afg_nest.h) is encoded into a flat instruction
// stream; its outermost perfectly nested loops whose iterations write
// disjoint elements become the thread grid, everything below runs per thread
// with the reference interpreter's arithmetic (interp.cpp:502-561).
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <string>
#include <vector>

#include "../../include/afg_nest.h"
#include "afg_internal.h"

namespace afg {
namespace vm {

// storage types of VM buffers (the interpreter's element types + bf16 / f64)
enum VmType : int32_t { VT_F32 = 0, VT_F16 = 1, VT_BF16 = 2, VT_I8 = 3, VT_I32 = 4, VT_F64 = 5 };

VmType vm_type(gpu::ElementType t);
int vm_type_bytes(VmType t);

// A device tensor known to the runner.
struct DevTensor {
  void* ptr = nullptr;
  VmType type = VT_F32;
  gpu::ElementType et = gpu::ElementType::F32;
  gpu::MemSpace space = gpu::MemSpace::Global;
  std::vector<int64_t> shape;
  bool owned = false;
  int64_t numel() const {
    int64_t n = 1;
    for (int64_t d : shape) n *= d;
    return n;
  }
};

// Counters laid out as NestMetrics (device array of unsigned long long).
enum CounterSlot {
  C_GLOBAL = 0, C_SHARED = 4, C_REGISTER = 8,  // loads, stores, loadBytes, storeBytes
  C_FLOPS = 12, C_FRAG_LOADS = 13, C_FRAG_COMPUTES = 14, C_FRAG_STORES = 15, C_CORRECTION = 16,
  C_PER_BUFFER = 32  // + 4 * buffer index
};

// Runs top-level nests over a table of device tensors (ids with '%').
class Runner {
 public:
  explicit Runner(cudaStream_t s) : s_(s) {}
  ~Runner();
  Runner(const Runner&) = delete;
  Runner& operator=(const Runner&) = delete;

  // Allocates (uninitialised) device storage for a tensor.
  DevTensor& alloc(const std::string& id, const std::vector<int64_t>& shape, gpu::ElementType et,
                   gpu::MemSpace space = gpu::MemSpace::Global);
  // Registers caller-owned device memory.
  DevTensor& bind(const std::string& id, void* ptr, const std::vector<int64_t>& shape,
                  gpu::ElementType et);
  bool has(const std::string& id) const { return t_.count(id) != 0; }
  DevTensor& at(const std::string& id);
  void release(const std::string& id);
  // Host doubles -> device, rounded to the tensor's type (interp.cpp:212-213).
  void upload(const std::string& id, const std::vector<double>& host);
  void upload(const std::string& id, const double* host, int64_t n);
  // Device -> host doubles (exact: every stored value is representable).
  std::vector<double> download(const std::string& id);
  // Scratch device memory freed with the runner.
  void* scratch(size_t bytes);

  // Executes one top-level op on the VM. `buffers_elsewhere` lists buffers
  // referenced by other top-level ops (they are never privatised per thread).
  // Returns a one-line plan entry.
  std::string run_vm(const gpu::NestOp& top, const std::map<std::string, int>& refcount);

  // Enables interpreter-style metrics counting (all buffers known so far and
  // later are counted); read with metrics().
  void enable_counting(const std::vector<std::string>& buffer_order);
  void fetch_metrics(gpu::NestMetrics* m);

  cudaStream_t stream() const { return s_; }
  void sync(const char* what);

 private:
  cudaStream_t s_;
  std::map<std::string, DevTensor> t_;
  std::vector<void*> scratch_;
  unsigned long long* counters_ = nullptr;
  std::vector<std::string> counted_;
  std::map<std::string, int> counted_index_;
  int* err_ = nullptr;
};

// Linear form of an index expression over named ivs (no div/mod), used by the
// dispatchers to verify nest structure.
struct Linear {
  std::map<std::string, int64_t> coef;
  int64_t c = 0;
  bool affine = true;  // false when a FloorDiv/Mod made it non-linear
  bool is_iv(const std::string& iv) const {
    return affine && c == 0 && coef.size() == 1 && coef.begin()->first == iv &&
           coef.begin()->second == 1;
  }
  bool is_const(int64_t v) const { return affine && coef.empty() && c == v; }
};
Linear linearize(const gpu::IndexExpr& e, const std::vector<std::string>& operands);

}  // namespace vm
}  // namespace afg
