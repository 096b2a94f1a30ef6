// afg_nest.h - C++ host API of the afg nest executor: a B200 executor for the
// reference's lowered loop-nest programs (af::Program, ir.h:36-318), the
// drop-in for af::interpret (interp.h:97-100, interp.cpp:164-696).
//
// The types mirror af::Program field for field, except that every affine map
// result arrives already flattened into a postfix index program (IndexExpr)
// over the map's positional dims, so this header needs no af:: type. The
// adapter a maintainer adds (integration/af_gpu.cpp) converts
// an af::Program into a NestProgram and back-converts the result.
//
// Execution (csrc/nestvm.cu, csrc/nestexec.cpp):
//  * every buffer lives on the device in its declared element type (the
//    interpreter rounds every store to that type, so native storage is
//    lossless); inputs are rounded on upload exactly like interp.cpp:212-213;
//  * each top-level nest is one launch. Nests the dispatcher recognises by
//    their `kind` attribute and structure (matmul-kind nests, conv nests with
//    the conv.* attributes, frontend.cpp:952-968) run on the afg kernels;
//    every other nest runs on the nest VM: the outermost perfectly nested
//    loops whose iterations provably write disjoint elements become the
//    thread grid, and each thread executes the rest of the nest with the
//    interpreter's arithmetic (double precision, rounding to the declared type
//    at every store, integer saturation, half-away quantisation);
//  * `count_metrics` makes every nest run on the VM and counts loads, stores,
//    bytes per memory space and per buffer, flops, fragment ops and
//    correction ops exactly as the interpreter's Metrics (interp.h:60-83).
#pragma once

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "afg_graph.h"

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

namespace afg {
namespace gpu {

enum class MemSpace { Global = 0, Shared = 1, Register = 2 };  // ir.h:34

// Postfix index program over the dims (positional operands) of one map
// result. Words: opcode, then its immediate where it has one.
struct IndexExpr {
  enum Code : int64_t { Const = 0, Dim = 1, Add = 2, MulConst = 3, FloorDiv = 4, Mod = 5 };
  std::vector<int64_t> code;
  static IndexExpr constant(int64_t v) { return {{Const, v}}; }
  static IndexExpr dim(int64_t i) { return {{Dim, i}}; }
};

// af::OpKind / af::ArithKind order (ir.h:97-128) + Round (extension: the
// store rounding roundToType, interp.cpp:88-104, as a value op).
enum class NestOpKind {
  For, Parallel, Load, Store, Arith, MmaLoad, MmaCompute, MmaStore, AsyncCopy, AwaitCopies,
  Alloc, Dealloc
};
enum class ArithOp {
  Add, Mul, Sub, Div, Max, Exp, Negate, Cast, Fma, Select, CmpEq, CmpLt, CmpLe, Quant,
  Dequant, Round
};

struct NestAttr {  // ir.h:57-70
  enum class Kind { Flag, Int, Str, Sym } kind = Kind::Flag;
  int64_t i = 0;
  std::string s;
};

struct NestOperand {  // ir.h:131-142
  bool isImm = false;
  std::string value;
  double imm = 0.0;
  static NestOperand val(std::string v) { return {false, std::move(v), 0.0}; }
  static NestOperand immF(double x) { return {true, {}, x}; }
};

struct NestOp {  // ir.h:146-180
  NestOpKind kind = NestOpKind::For;
  std::map<std::string, NestAttr> attrs;
  // For: ivs.size() == 1; Parallel: one entry per iv. lowers[i] results are
  // maxed, uppers[i] minned (AffineMap::evalMax / evalMin), dims bind to
  // boundOperands.
  std::vector<std::string> ivs;
  std::vector<std::vector<IndexExpr>> lowers, uppers;
  std::vector<std::string> boundOperands;
  int64_t step = 1;
  std::vector<NestOp> body;
  // Load / Store / Mma* / Alloc / Dealloc / AsyncCopy (dst)
  std::string buffer;
  std::vector<IndexExpr> access;
  std::vector<std::string> accessOperands;
  // value-producing ops
  std::string result;
  ArithOp arith = ArithOp::Add;
  std::vector<NestOperand> operands;
  ElementType castType = ElementType::F32;
  double scale = 1.0;
  int mmaRole = 0;
  std::string tag, srcBuffer;

  std::string kindAttr() const {
    auto it = attrs.find("kind");
    return it == attrs.end() ? std::string() : it->second.s;
  }
};

struct NestBuffer {  // ir.h:39-55 (ids keep the leading '%')
  std::string id;
  std::vector<int64_t> shape;
  ElementType dtype = ElementType::F32;
  MemSpace space = MemSpace::Global;
  bool isInput = false;
  bool isOutput = false;
  int64_t numElements() const {
    int64_t n = 1;
    for (int64_t d : shape) n *= d;
    return n;
  }
};

struct NestProgram {  // one af::Function of an af::Program
  std::vector<NestBuffer> buffers;
  std::vector<NestOp> body;
};

struct NestCounters {  // interp.h:46-58
  int64_t loads = 0, stores = 0, loadBytes = 0, storeBytes = 0;
};
struct NestMetrics {  // interp.h:60-83
  NestCounters global, shared, registers;
  int64_t flops = 0;
  int64_t fragmentLoads = 0, fragmentComputes = 0, fragmentStores = 0;
  int64_t nestCount = 0;
  int64_t correctionOps = 0;
  std::map<std::string, NestCounters> perBuffer;
  std::map<std::string, MemSpace> perBufferSpace;
};

struct NestRunOptions {
  void* stream = nullptr;      // cudaStream_t
  bool dispatch = true;        // matmul / conv nests on the afg kernels
  bool tensor_cores = true;    // ... and on tcgen05 when the values allow it
  bool count_metrics = false;  // run everything on the VM, count like the interpreter
};

struct NestRunStats {
  std::vector<std::string> plan;  // one line per launch group
};

// The af::interpret contract: inputs keyed by buffer id ("%x"), one for every
// isInput buffer, shape-checked (InterpError otherwise); returns the isOutput
// buffers keyed by id with the values rounded to their declared type.
// Hard failures (out-of-bounds access) throw InterpError.
std::map<std::string, TensorValue> run_program(const NestProgram& p,
                                               const std::map<std::string, TensorValue>& inputs,
                                               const NestRunOptions& opt = {},
                                               NestMetrics* metrics = nullptr,
                                               NestRunStats* stats = nullptr);

}  // namespace gpu
}  // namespace afg

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
