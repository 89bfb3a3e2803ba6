// runner_trace.cpp — TEST INFRASTRUCTURE: runs the reference's own runner
// (proj/src/runner.cpp run_scenario -> run_rlhf_step, :152-166, :240-241) on
// its built-in scenarios and writes trace.csv + summary.json per scenario
// (runner::write_outputs).  Linked twice by oracle/Makefile: against the
// reference alone (runner_ref) and against the drop-in B200 library
// (runner_b200: run_rlhf_step from dropin/run_rlhf_step.cpp, every round of
// every shard in one device call); tests/test_gpu_integer.py compares the
// two output trees byte for byte (the reference's own acceptance criterion 11,
// acceptance_test.cpp:609-628, across implementations).
#include <cstdio>
#include <filesystem>
#include <string>

#include "yatt/runner.hpp"
#include "yatt/scenario.hpp"

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s OUT_DIR [scenario ...]\n", argv[0]);
    return 2;
  }
  namespace fs = std::filesystem;
  const fs::path out = argv[1];
  std::vector<std::string> names;
  for (int i = 2; i < argc; ++i) names.push_back(argv[i]);
  if (names.empty()) names = {"builtin:table1", "builtin:sweep", "builtin:demo"};
  for (const auto& ref : names) {
    const yatt::cli::Scenario s = yatt::cli::load_scenario(ref);
    const fs::path dir = out / ref.substr(ref.find(':') + 1);
    fs::create_directories(dir);
    yatt::runner::write_outputs(yatt::runner::run_scenario(s), dir.string());
    std::printf("%s -> %s\n", ref.c_str(), dir.c_str());
  }
  return 0;
}
