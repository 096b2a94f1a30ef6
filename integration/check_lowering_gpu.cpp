// check_lowering_gpu.cpp - the reference's checkLowering
// (tests/test_frontend.cpp:22-37) with the B200 executors swapped in, written
// against the reference's own API and comparison routine. TEST
// INFRASTRUCTURE (links the reference library from oracle/_ref).
//
// For every graph file given on the command line (JSON {"graph":..., "seed":
// ..., "lo":..., "hi":..., "profile": "F32"|"F16Fragment"|"Int", "fixed":
// {id: [values]}}):
//   p = lowerGraphToAffine(g); inputs = makeRandomInputs(p, seed, lo, hi)
//   (fixed constant tensors such as ReLU zeros / causal masks overwrite the
//   random ones); expected = interpret(p, inputs).outputs
//   1. got = af::gpu::execute(g, inputs)          (the graph planner)
//   2. got = af::gpu::interpret(p, inputs)        (the program executor)
//   3. q = orchestrate(p): interpret(q) vs af::gpu::interpret(q), outputs AND
//      metrics (global / shared traffic, flops, fragment counts): the tiled,
//      packed, overlapped, parallelised form of the same program
// and compareOutputs(got, expected, profile) must pass.
#include <cstdio>
#include <fstream>
#include <nlohmann/json.hpp>
#include <sstream>

#include "af/frontend.h"
#include "af/interp.h"
#include "af/tiling.h"
#include "af_gpu.h"

using json = nlohmann::json;

namespace {

bool same_metrics(const af::Metrics& a, const af::Metrics& b, std::string* why) {
  auto eq = [&](const char* what, int64_t x, int64_t y) {
    if (x == y) return true;
    *why += std::string(what) + " " + std::to_string(x) + " vs " + std::to_string(y) + "; ";
    return false;
  };
  bool ok = true;
  ok &= eq("global.loads", a.global.loads, b.global.loads);
  ok &= eq("global.stores", a.global.stores, b.global.stores);
  ok &= eq("shared.loads", a.shared.loads, b.shared.loads);
  ok &= eq("shared.stores", a.shared.stores, b.shared.stores);
  ok &= eq("registers.loads", a.registers.loads, b.registers.loads);
  ok &= eq("flops", a.flops, b.flops);
  ok &= eq("fragmentComputes", a.fragmentComputes, b.fragmentComputes);
  ok &= eq("nestCount", a.nestCount, b.nestCount);
  return ok;
}

}  // namespace

int main(int argc, char** argv) {
  int failures = 0;
  for (int i = 1; i < argc; ++i) {
    std::ifstream f(argv[i]);
    std::stringstream ss;
    ss << f.rdbuf();
    json spec = json::parse(ss.str());
    for (const auto& c : spec.at("cases")) {
      const std::string name = c.at("name");
      const std::string graph = c.at("graph").dump();
      af::TensorGraph g = af::parseGraphJson(graph);
      af::Program p = af::lowerGraphToAffine(g, af::TargetConfig{});
      auto inputs = af::makeRandomInputs(p, c.at("seed").get<uint64_t>(), c.value("lo", 0.0),
                                         c.value("hi", 1.0));
      if (c.contains("fixed"))
        for (const auto& [id, vals] : c.at("fixed").items()) {
          auto& tv = inputs.at("%" + id);
          for (size_t k = 0; k < tv.data.size(); ++k) {
            const auto& v = vals.at(k);
            tv.data[k] = v.is_string() ? (v.get<std::string>() == "-inf" ? -INFINITY : INFINITY)
                                       : v.get<double>();
          }
        }
      auto ref = af::interpret(p, inputs);
      const std::string prof = c.value("profile", std::string("F32"));
      const af::TolProfile tp = prof == "Int"           ? af::TolProfile::Int
                                : prof == "F16Fragment" ? af::TolProfile::F16Fragment
                                                        : af::TolProfile::F32;
      auto check = [&](const char* tag, const std::function<std::map<std::string, af::TensorValue>()>& run,
                       const std::map<std::string, af::TensorValue>& expected) {
        std::map<std::string, af::TensorValue> got;
        try {
          got = run();
        } catch (const std::exception& e) {
          std::printf("FAIL %s %s: %s\n", tag, name.c_str(), e.what());
          ++failures;
          return;
        }
        af::ComparisonReport rep = af::compareOutputs(got, expected, tp);
        std::printf("%s %s %s: maxRel=%.3e maxAbs=%.3e %s\n", rep.passed ? "PASS" : "FAIL", tag,
                    name.c_str(), rep.maxRelErr, rep.maxAbsErr, rep.message.c_str());
        if (!rep.passed) ++failures;
      };
      check("graph", [&] { return af::gpu::execute(g, inputs); }, ref.outputs);
      check("program", [&] { return af::gpu::interpret(p, inputs).outputs; }, ref.outputs);
      // the orchestrated (tiled / packed / overlapped / parallel) program
      af::Program q;
      af::InterpResult refq;
      try {
        q = af::orchestrate(p, af::TargetConfig{});
        refq = af::interpret(q, inputs);
      } catch (const std::exception& e) {  // the reference itself cannot run it
        std::printf("SKIP orchestrated %s: reference orchestrate/interpret: %s\n", name.c_str(),
                    e.what());
        continue;
      }
      af::InterpResult gotq;
      check("orchestrated", [&] {
        gotq = af::gpu::interpret(q, inputs);
        return gotq.outputs;
      }, refq.outputs);
      std::string why;
      if (!same_metrics(gotq.metrics, refq.metrics, &why)) {
        std::printf("FAIL metrics %s: %s\n", name.c_str(), why.c_str());
        ++failures;
      } else {
        std::printf("PASS metrics %s\n", name.c_str());
      }
    }
  }
  std::printf("%d failure(s)\n", failures);
  return failures == 0 ? 0 : 1;
}
