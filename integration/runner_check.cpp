// runner_check — f3: the reference's own output path on top of the GPU.
//
// Writes a planner workspace (config.json with a synthetic 4-model score workload, the
// profile and memory CSVs) and runs the reference's runner — run_plan and run_sweep
// (runner.cpp:151-173), which render plan.txt / sweep.csv through render_plan /
// render_sweep_csv and format_double (runner.cpp:69-149, csv.cpp:78-84) — into the output
// directory given on the command line.  Built twice (integration/Makefile):
//   runner_check_b200: select_setup & co. from the C-ABI shim (librw_b200.so, the GPU);
//   runner_check_ref:  the unmodified reference library (CPU).
// tests/test_gpu_integration.py requires the two plan.txt and sweep.csv to be byte-identical.
#include <cmath>
#include <cstdio>
#include <sstream>
#include <string>

#include "helpers.hpp"
#include "routeplan/config.hpp"
#include "routeplan/csv.hpp"
#include "routeplan/runner.hpp"

using namespace routeplan;

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s OUT_DIR\n", argv[0]);
    return 2;
  }
  const std::string out = argv[1];
  testutil::TempDir dir;
  const char* models[] = {"A", "B", "C", "D"};
  std::ostringstream prof;
  prof << "model,tp,rho,metric,load_rps,latency_ms\n";
  for (int i = 0; i < 4; ++i)
    for (int tp : {1, 2})
      for (double rho : {0.5, 1.0}) {  // SURVEY.md §8d profile formula
        const double b = (20.0 + 25.0 * i) / (std::sqrt(static_cast<double>(tp)) * rho);
        const double s = (1.0 + 1.5 * i) / (tp * rho);
        const double loads[3] = {0.0, 20.0, 60.0};
        const double lats[3] = {b, b + 20.0 * s, b + 140.0 * s};
        for (int q = 0; q < 3; ++q)
          prof << models[i] << ',' << tp << ',' << format_double(rho) << ",TTFT,"
               << format_double(loads[q]) << ',' << format_double(lats[q]) << '\n';
      }
  testutil::write_file(dir.file("profiles.csv"), prof.str());
  std::ostringstream mem;
  mem << "model,tp,mem_fraction\n";
  for (const char* mdl : models) mem << mdl << ",1,0.4\n" << mdl << ",2,0.25\n";
  testutil::write_file(dir.file("memory.csv"), mem.str());
  testutil::write_file(dir.file("config.json"),
                       "{\n"
                       "  \"gpu_count\": 8,\n"
                       "  \"arrival_rate_rps\": 40.0,\n"
                       "  \"latency_target_ms\": 120,\n"
                       "  \"metric\": \"TTFT\",\n"
                       "  \"rho_min\": 0.1,\n"
                       "  \"seed\": 1,\n"
                       "  \"parallelism\": 1,\n"
                       "  \"profiles\": \"profiles.csv\",\n"
                       "  \"memory\": \"memory.csv\",\n"
                       "  \"synthetic\": {\"n_prompts\": 3000},\n"
                       "  \"optimizer\": {\"subgradient\": {\"max_iters\": 30},\n"
                       "                \"pga\": {\"max_iters\": 6},\n"
                       "                \"beta\": {\"epsilon\": 0.01}},\n"
                       "  \"models\": [\n"
                       "    {\"name\": \"A\", \"tp_choices\": [1, 2], \"rho_choices\": [0.5, 1.0],"
                       " \"score_beta\": [2, 8]},\n"
                       "    {\"name\": \"B\", \"tp_choices\": [1, 2], \"rho_choices\": [0.5, 1.0],"
                       " \"score_beta\": [4, 6]},\n"
                       "    {\"name\": \"C\", \"tp_choices\": [1], \"rho_choices\": [0.5, 1.0],"
                       " \"score_beta\": [6, 4]},\n"
                       "    {\"name\": \"D\", \"tp_choices\": [1], \"rho_choices\": [0.5, 1.0],"
                       " \"score_beta\": [8, 2]}\n"
                       "  ]\n"
                       "}\n");
  PlannerConfig cfg = load_config(dir.file("config.json"));
  std::ostringstream log;
  const int rc_plan = run_plan(cfg, out, log);
  const int rc_sweep = run_sweep(cfg, out, log);
  std::printf("run_plan %d run_sweep %d\n%s", rc_plan, rc_sweep, log.str().c_str());
  return (rc_plan == 0 || rc_plan == 2) && rc_sweep == 0 ? 0 : 1;
}
