// ref_shim.cpp - TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// A small extern "C" driver over the UNMODIFIED reference library, built from
// the sources where they lie under /root/reference/proj by oracle/Makefile
// into oracle/_ref/libafref.so. It lets the Python tests / bench reference arm
// run the reference's own CPU path:
//   af::parseGraphJson -> af::lowerGraphToAffine -> af::interpret
//       (frontend.cpp:57-113, :975-979; interp.cpp:690-696)
//   af::oracle::evalGraphReference                 (tests/oracles.cpp:247-407)
//   af::makeRandomInputs / roundToType / compareTensors (interp.cpp:817-853,
//       :88-104, :698-730)
// exactly as the reference's checkLowering (test_frontend.cpp:22-37) does.
#include <cstring>
#include <exception>
#include <map>
#include <string>
#include <vector>

#include "af/frontend.h"
#include "af/interp.h"
#include "af/ir.h"
#include "oracles.h"

namespace {

struct Result {
  std::vector<std::string> names;
  std::vector<af::TensorValue> values;
  std::string metrics;
};

void set_err(char* err, int errlen, const std::string& m) {
  if (err && errlen > 0) {
    std::strncpy(err, m.c_str(), errlen - 1);
    err[errlen - 1] = 0;
  }
}

Result* wrap(const std::map<std::string, af::TensorValue>& m) {
  auto* r = new Result;
  for (const auto& [k, v] : m) {
    r->names.push_back(k);
    r->values.push_back(v);
  }
  return r;
}

}  // namespace

extern "C" {

// Runs a graph through the reference.
//   which = 0 : lowerGraphToAffine + interpret (the reference CPU path)
//   which = 1 : oracle::evalGraphReference     (independent brute force)
// Inputs are keyed by graph tensor id (no '%'); values are taken as given
// (the reference rounds them to the declared type itself).
// Returns a Result handle (outputs keyed "%id") or NULL with `err` set.
void* afref_run(const char* graph_json, int n_in, const char** names, const double** data,
                const int64_t* numel, int which, char* err, int errlen) {
  try {
    std::string text(graph_json);
    af::TensorGraph g = af::parseGraphJson(text);
    af::checkGraph(g);
    std::map<std::string, af::TensorValue> bare, pct;
    for (int i = 0; i < n_in; ++i) {
      const af::TensorDesc* d = g.find(names[i]);
      if (!d) throw af::GraphError(std::string("unknown input ") + names[i]);
      af::TensorValue tv;
      tv.shape = d->shape;
      tv.type = d->dtype;
      if (tv.numElements() != numel[i]) throw af::GraphError("input size mismatch");
      tv.data.assign(data[i], data[i] + numel[i]);
      bare[names[i]] = tv;
      pct[std::string("%") + names[i]] = std::move(tv);
    }
    if (which == 1) return wrap(af::oracle::evalGraphReference(text, bare));
    af::Program p = af::lowerGraphToAffine(g, af::TargetConfig{});
    af::InterpResult res = af::interpret(p, pct);
    Result* r = wrap(res.outputs);
    r->metrics = res.metrics.toJson();
    return r;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return nullptr;
  }
}

// makeRandomInputs on the lowered program of `graph_json` (keys "%id").
void* afref_random_inputs(const char* graph_json, uint64_t seed, double lo, double hi,
                          char* err, int errlen) {
  try {
    af::TensorGraph g = af::parseGraphJson(graph_json);
    af::Program p = af::lowerGraphToAffine(g, af::TargetConfig{});
    return wrap(af::makeRandomInputs(p, seed, lo, hi));
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return nullptr;
  }
}

int afref_result_count(void* h) { return static_cast<int>(static_cast<Result*>(h)->names.size()); }
const char* afref_result_name(void* h, int i) {
  return static_cast<Result*>(h)->names[i].c_str();
}
int afref_result_rank(void* h, int i) {
  return static_cast<int>(static_cast<Result*>(h)->values[i].shape.size());
}
int64_t afref_result_dim(void* h, int i, int d) {
  return static_cast<Result*>(h)->values[i].shape[d];
}
int afref_result_type(void* h, int i) {
  return static_cast<int>(static_cast<Result*>(h)->values[i].type);
}
int64_t afref_result_numel(void* h, int i) {
  return static_cast<Result*>(h)->values[i].numElements();
}
const double* afref_result_data(void* h, int i) {
  return static_cast<Result*>(h)->values[i].data.data();
}
const char* afref_result_metrics(void* h) { return static_cast<Result*>(h)->metrics.c_str(); }
void afref_free(void* h) { delete static_cast<Result*>(h); }

double afref_round_to_type(double v, int t) {
  return af::roundToType(v, static_cast<af::ElementType>(t));
}
double afref_round_to_f16(double v) { return af::roundToF16(v); }
uint64_t afref_std_hash(const char* s) { return std::hash<std::string>{}(std::string(s)); }

// compareTensors(a, b, profile) (interp.cpp:698-730) on flat arrays.
int afref_compare(const double* a, const double* b, int64_t n, int profile, double* max_abs,
                  double* max_rel, int64_t* worst) {
  af::TensorValue ta, tb;
  ta.shape = {n};
  tb.shape = {n};
  ta.data.assign(a, a + n);
  tb.data.assign(b, b + n);
  af::ComparisonReport r = af::compareTensors(ta, tb, static_cast<af::TolProfile>(profile));
  if (max_abs) *max_abs = r.maxAbsErr;
  if (max_rel) *max_rel = r.maxRelErr;
  if (worst) *worst = r.worstIndex;
  return r.passed ? 1 : 0;
}

// conv output geometry of the reference (frontend.cpp:115-149).
void afref_conv_geometry(int64_t inH, int64_t inW, int64_t kH, int64_t kW, int64_t sY,
                         int64_t sX, int64_t dY, int64_t dX, int same, int transposed,
                         int64_t* out4) {
  af::TensorOpNode n;
  n.strideY = sY;
  n.strideX = sX;
  n.dilY = dY;
  n.dilX = dX;
  n.samePadding = same != 0;
  n.transposed = transposed != 0;
  af::ConvGeometry g = af::convGeometry(inH, inW, kH, kW, n);
  out4[0] = g.outH;
  out4[1] = g.outW;
  out4[2] = g.padY;
  out4[3] = g.padX;
}

}  // extern "C"
