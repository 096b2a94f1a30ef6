// check_lowering_gpu.cpp - the reference's checkLowering
// (tests/test_frontend.cpp:22-37) with the B200 executor swapped in, written
// against the reference's own API and comparison routine. TEST
// INFRASTRUCTURE (links the reference library from oracle/_ref).
//
// For every graph file given on the command line (JSON {"graph":..., "seed":
// ..., "lo":..., "hi":..., "profile": "F32"|"F16Fragment"|"Int", "fixed":
// {id: [values]}}):
//   p = lowerGraphToAffine(g); inputs = makeRandomInputs(p, seed, lo, hi)
//   (fixed constant tensors such as ReLU zeros / causal masks overwrite the
//   random ones); expected = interpret(p, inputs).outputs
//   got = af::gpu::execute(g, inputs)
//   compareOutputs(got, expected, profile) must pass.
#include <cstdio>
#include <fstream>
#include <nlohmann/json.hpp>
#include <sstream>

#include "af/frontend.h"
#include "af/interp.h"
#include "af_gpu.h"

using json = nlohmann::json;

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
      auto expected = af::interpret(p, inputs).outputs;
      std::map<std::string, af::TensorValue> got;
      try {
        got = af::gpu::execute(g, inputs);
      } catch (const std::exception& e) {
        std::printf("FAIL %s: %s\n", name.c_str(), e.what());
        ++failures;
        continue;
      }
      const std::string prof = c.value("profile", std::string("F32"));
      const af::TolProfile tp = prof == "Int"           ? af::TolProfile::Int
                                : prof == "F16Fragment" ? af::TolProfile::F16Fragment
                                                        : af::TolProfile::F32;
      af::ComparisonReport rep = af::compareOutputs(got, expected, tp);
      std::printf("%s %s: maxRel=%.3e maxAbs=%.3e %s\n", rep.passed ? "PASS" : "FAIL",
                  name.c_str(), rep.maxRelErr, rep.maxAbsErr, rep.message.c_str());
      if (!rep.passed) ++failures;
    }
  }
  std::printf("%d failure(s)\n", failures);
  return failures == 0 ? 0 : 1;
}
