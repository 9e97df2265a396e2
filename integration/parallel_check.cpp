// parallel_check — the drop-in's multi-GPU select_setup against the reference's own.
//
// Built twice from this file (integration/Makefile):
//   parallel_check_b200: `routeplan::select_setup` is the shim's (routeplan_b200_shim.cpp
//       -> rw_sweep / rw_sweep_multi); it runs SearchParams::parallelism = 1, 2, 3 (GPU
//       shards; with one GPU set RW_SHIM_SHARED_GPU=1 so the shards share it);
//   parallel_check_ref:  the unmodified reference library (-DRW_CPU_REF), 4 threads.
// Each run prints one canonical dump of the SearchOutput (every sweep row and the plan as
// hex floats); tests/test_gpu_integration.py requires all dumps to be identical — the
// reference's determinism requirement (test_setup_search.cpp:264-292: results do not
// depend on parallelism) across the CPU build and any number of GPU shards.
// Workload: C1 shape (4 models, 64 retained setups), N = 4000, truncated schedule.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "routeplan/latency.hpp"
#include "routeplan/routing_opt.hpp"
#include "routeplan/setup_search.hpp"
#include "routeplan/workload.hpp"

using namespace routeplan;

static void dump(const char* tag, int parallelism, const SearchOutput& o) {
  std::printf("%s parallelism=%d rows=%zu\n", tag, parallelism, o.sweep.size());
  for (const SweepRecord& r : o.sweep)
    std::printf("row %ld %d %a %a\n", r.setup_id, r.feasible ? 1 : 0, r.score, r.latency_ms);
  const PlanResult& p = o.plan;
  std::printf("plan %d %a %a %a", p.feasible ? 1 : 0, p.score, p.latency_ms, p.beta);
  for (double w : p.w.w) std::printf(" %a", w);
  for (const ModelSetup& ms : p.setup.per_model) std::printf(" %d:%a", ms.tp, ms.rho);
  std::printf("\nend\n");
}

int main() {
  const std::vector<std::string> models = {"A", "B", "C", "D"};
  std::vector<BetaShape> shapes;
  for (int i = 0; i < 4; ++i) shapes.push_back({2.0 + 2.0 * i, 8.0 - 2.0 * i});
  ScoreMatrix scores = synth_scores(4000, models, shapes, 1);

  SetupSpace space;
  space.models = models;
  space.tp_choices = {{1, 2}, {1, 2}, {1}, {1}};
  space.rho_choices = {{0.5, 1.0}, {0.5, 1.0}, {0.5, 1.0}, {0.5, 1.0}};
  MemoryTable mem;
  ProfileLibrary lib;
  for (int i = 0; i < 4; ++i) {
    mem.insert(models[i], 1, 0.4);
    mem.insert(models[i], 2, 0.25);
    for (int tp : {1, 2})
      for (double rho : {0.5, 1.0}) {  // SURVEY.md §8d profile formula
        const double b = (20.0 + 25.0 * i) / (std::sqrt(static_cast<double>(tp)) * rho);
        const double s = (1.0 + 1.5 * i) / (tp * rho);
        LatencyProfile p;
        p.model = models[i];
        p.tp = tp;
        p.rho = rho;
        p.metric = Metric::TTFT;
        p.knots = {{0.0, b}, {20.0, b + 20.0 * s}, {60.0, b + 140.0 * s}};
        lib.profiles[make_profile_key(models[i], tp, rho, Metric::TTFT)] = p;
      }
  }
  SearchContext ctx;
  ctx.gpu_count = 8;
  ctx.rho_floor = 0.1;
  ctx.mem = &mem;
  ctx.opt.scores = &scores;
  ctx.opt.lib = &lib;
  ctx.opt.lambda_rps = 40.0;
  ctx.opt.tau_ms = 120.0;
  ctx.opt.metric = Metric::TTFT;
  ctx.opt.kappa = 1.25;
  SearchParams params;  // truncated schedule: 20 / 5 / span 4
  params.beta.epsilon = (10.0 / 120.0) / 4.0;
  params.beta.pga.max_iters = 5;
  params.beta.pga.dual.max_iters = 20;

#ifdef RW_CPU_REF
  params.parallelism = 4;
  dump("cpu-reference", 4, select_setup(space, ctx, params));
#else
  for (int shards : {1, 2, 3}) {
    params.parallelism = shards;
    dump("gpu-shards", shards, select_setup(space, ctx, params));
  }
#endif
  return 0;
}
