// TEST INFRASTRUCTURE ONLY — generates tests/golden/reference_cases.json.
//
// Replays the instance generators of the reference's own doctest suite (same seeds, same
// testutil builders from /root/reference/proj/tests/helpers.cpp, compiled from where they
// lie) and records what the UNMODIFIED reference library returns for each instance, plus a
// few larger synthetic instances.  Every double is written as a C99 hex float ("%a"), so the
// fixture is bit-exact.  Built and run by oracle/Makefile `golden` (needs /root/reference);
// the fixture is committed and travels without the reference.
//
// Case kinds (fields mirror the reference structs):
//   eval     scores, c, alpha -> g, counts, model_of          (dual_objective / assign_prompts)
//   solve    scores, c, params[, init] -> DualSolution         (solve_dual)
//   simplex  v -> w                                             (project_simplex)
//   latency  profiles, w, lambda, kappa -> SystemLatencyEval + grad
//   optfrac  scores, profiles, beta, ctx, params -> RelaxedSolveResult
//   optbeta  scores, profiles, ctx, params -> BetaSearchResult (+ trace)
#include <cmath>
#include <cstdio>
#include <map>
#include <random>
#include <string>
#include <vector>

#include "helpers.hpp"

using namespace routeplan;

namespace {

FILE* out = nullptr;
bool first_case = true;

std::string hx(double v) {
  char b[64];
  std::snprintf(b, sizeof b, "\"%a\"", v);
  return b;
}
std::string dv(const std::vector<double>& v) {
  std::string s = "[";
  for (size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + hx(v[i]);
  return s + "]";
}
std::string iv(const std::vector<int>& v) {
  std::string s = "[";
  for (size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + std::to_string(v[i]);
  return s + "]";
}
std::string bv(const std::vector<bool>& v) {
  std::string s = "[";
  for (size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + std::string(v[i] ? "1" : "0");
  return s + "]";
}
// score matrices are stored once in the top-level "matrices" list; cases name an index
std::vector<std::string> matrices;
std::map<std::string, int> matrix_id;
std::string scores_json(const ScoreMatrix& s) {
  std::string body = "{\"n\":" + std::to_string(s.n()) + ",\"m\":" + std::to_string(s.m()) +
                     ",\"v\":" + dv(s.scores) + "}";
  auto it = matrix_id.find(body);
  if (it == matrix_id.end()) {
    it = matrix_id.emplace(body, static_cast<int>(matrices.size())).first;
    matrices.push_back(body);
  }
  return std::to_string(it->second);
}
std::string knots_json(const std::vector<std::vector<std::pair<double, double>>>& profs) {
  std::string s = "[";
  for (size_t p = 0; p < profs.size(); ++p) {
    s += (p ? "," : "") + std::string("[");
    for (size_t k = 0; k < profs[p].size(); ++k)
      s += (k ? "," : "") + std::string("[") + hx(profs[p][k].first) + "," +
           hx(profs[p][k].second) + "]";
    s += "]";
  }
  return s + "]";
}
std::string sub_json(const SubgradientParams& p) {
  return "{\"eta0\":" + hx(p.eta0) + ",\"max_iters\":" + std::to_string(p.max_iters) +
         ",\"residual_tol\":" + hx(p.residual_tol) +
         ",\"polish_passes\":" + std::to_string(p.polish_passes) + "}";
}
std::string pga_json(const PgaParams& p) {
  return "{\"eta\":" + hx(p.eta) + ",\"max_iters\":" + std::to_string(p.max_iters) +
         ",\"w_tol\":" + hx(p.w_tol) + ",\"dual\":" + sub_json(p.dual) + "}";
}
std::string beta_json(const BetaSearchParams& p) {
  return "{\"beta_min\":" + hx(p.beta_min) + ",\"beta_max\":" + hx(p.beta_max) +
         ",\"epsilon\":" + hx(p.epsilon) + ",\"pga\":" + pga_json(p.pga) + "}";
}

void emit(const std::string& kind, const std::string& cite, const std::string& body) {
  std::fprintf(out, "%s\n{\"kind\":\"%s\",\"cite\":\"%s\",%s}", first_case ? "" : ",",
               kind.c_str(), cite.c_str(), body.c_str());
  first_case = false;
}

DualPrices prices(std::vector<double> a) {
  DualPrices p;
  p.alpha = std::move(a);
  return p;
}

void case_eval(const std::string& cite, const ScoreMatrix& s, const std::vector<double>& c,
               const std::vector<double>& alpha) {
  TargetCounts t = testutil::make_counts(c);
  double g = dual_objective(s, t, prices(alpha));
  Assignment a = assign_prompts(s, prices(alpha));
  emit("eval", cite,
       "\"scores\":" + scores_json(s) + ",\"c\":" + dv(c) + ",\"alpha\":" + dv(alpha) +
           ",\"g\":" + hx(g) + ",\"counts\":" + iv(a.counts) + ",\"model_of\":" + iv(a.model_of));
}

void case_solve(const std::string& cite, const ScoreMatrix& s, const std::vector<double>& c,
                const SubgradientParams& p = SubgradientParams()) {
  DualSolution d = solve_dual(s, testutil::make_counts(c), p);
  std::string body = "\"scores\":" + scores_json(s) + ",\"c\":" + dv(c) +
                     ",\"params\":" + sub_json(p) + ",\"init_alpha\":" + dv(p.init_alpha) +
                     ",\"alpha_star\":" + dv(d.alpha_star.alpha) + ",\"score\":" + hx(d.score) +
                     ",\"dual_bound\":" + hx(d.dual_bound) +
                     ",\"duality_gap\":" + hx(d.duality_gap) +
                     ",\"assignment\":" + iv(d.assignment) +
                     ",\"count_residual\":" + dv(d.count_residual) +
                     ",\"iterations\":" + std::to_string(d.iterations) +
                     ",\"converged\":" + std::to_string(d.converged ? 1 : 0);
  if (s.n() <= 12) {
    bool integral = true;
    for (double x : c) integral = integral && std::abs(x - std::round(x)) <= 1e-9;
    if (integral) body += ",\"exact\":" + hx(exact_score_oracle(s, testutil::make_counts(c)));
  }
  emit("solve", cite, body);
}

void case_simplex(const std::string& cite, const std::vector<double>& v) {
  RoutingFractions w = project_simplex(v);
  emit("simplex", cite, "\"v\":" + dv(v) + ",\"w\":" + dv(w.w));
}

// single-setup plumbing: model i uses profile i (tp 1, rho 1)
struct Scen {
  ProfileLibrary lib;
  SystemSetup setup;
  std::vector<std::vector<std::pair<double, double>>> knots;
  explicit Scen(const std::vector<std::vector<std::pair<double, double>>>& k) : knots(k) {
    for (size_t i = 0; i < k.size(); ++i) {
      std::string name(1, static_cast<char>('A' + i));
      testutil::add_profile(lib, testutil::make_profile(name, 1, 1.0, Metric::TTFT, k[i]));
      setup.per_model.push_back({name, 1, 1.0});
    }
  }
};

void case_latency(const std::string& cite, const Scen& sc, const std::vector<double>& w,
                  double lambda, double kappa) {
  RoutingFractions f;
  f.w = w;
  SystemLatencyEval e = system_latency_eval(sc.lib, sc.setup, f, lambda, Metric::TTFT, kappa);
  std::vector<double> g = system_latency_grad(sc.lib, sc.setup, f, lambda, Metric::TTFT);
  emit("latency", cite,
       "\"profiles\":" + knots_json(sc.knots) + ",\"w\":" + dv(w) + ",\"lambda\":" + hx(lambda) +
           ",\"kappa\":" + hx(kappa) + ",\"latency\":" + hx(e.latency_ms) +
           ",\"loads\":" + dv(e.per_model_load) + ",\"lats\":" + dv(e.per_model_latency) +
           ",\"oor\":" + bv(e.out_of_range) + ",\"grad\":" + dv(g));
}

std::string ctx_json(double lambda, double tau, double kappa) {
  return "{\"lambda_rps\":" + hx(lambda) + ",\"tau_ms\":" + hx(tau) + ",\"kappa\":" + hx(kappa) +
         "}";
}

void case_optfrac(const std::string& cite, const ScoreMatrix& s, const Scen& sc, double beta,
                  double lambda, double tau, const PgaParams& p = PgaParams()) {
  OptimizeContext ctx;
  ctx.scores = &s;
  ctx.lib = &sc.lib;
  ctx.lambda_rps = lambda;
  ctx.tau_ms = tau;
  RelaxedSolveResult r = optimize_fractions(sc.setup, beta, ctx, p);
  emit("optfrac", cite,
       "\"scores\":" + scores_json(s) + ",\"profiles\":" + knots_json(sc.knots) +
           ",\"beta\":" + hx(beta) + ",\"ctx\":" + ctx_json(lambda, tau, ctx.kappa) +
           ",\"params\":" + pga_json(p) + ",\"w\":" + dv(r.w.w) +
           ",\"objective\":" + hx(r.objective) + ",\"score\":" + hx(r.score) +
           ",\"latency_ms\":" + hx(r.latency_ms) + ",\"iterations\":" +
           std::to_string(r.iterations) + ",\"converged\":" + std::to_string(r.converged ? 1 : 0) +
           ",\"out_of_range\":" + bv(r.out_of_range));
}

void case_optbeta(const std::string& cite, const ScoreMatrix& s, const Scen& sc, double lambda,
                  double tau, const BetaSearchParams& p = BetaSearchParams()) {
  OptimizeContext ctx;
  ctx.scores = &s;
  ctx.lib = &sc.lib;
  ctx.lambda_rps = lambda;
  ctx.tau_ms = tau;
  BetaSearchResult r = optimize_beta(sc.setup, ctx, p);
  std::vector<double> tb, ts, tl;
  std::vector<int> tok;
  for (const auto& st : r.trace) {
    tb.push_back(st.beta);
    ts.push_back(st.score);
    tl.push_back(st.latency_ms);
    tok.push_back(st.feasible ? 1 : 0);
  }
  std::string body = "\"scores\":" + scores_json(s) + ",\"profiles\":" + knots_json(sc.knots) +
                     ",\"ctx\":" + ctx_json(lambda, tau, ctx.kappa) + ",\"params\":" +
                     beta_json(p) + ",\"feasible\":" + std::to_string(r.feasible ? 1 : 0) +
                     ",\"has_beta_star\":" + std::to_string(r.beta_star ? 1 : 0) +
                     ",\"beta_star\":" + hx(r.beta_star.value_or(0.0)) +
                     ",\"w_star\":" + dv(r.w_star ? r.w_star->w : std::vector<double>{}) +
                     ",\"trace_beta\":" + dv(tb) + ",\"trace_score\":" + dv(ts) +
                     ",\"trace_latency\":" + dv(tl) + ",\"trace_ok\":" + iv(tok);
  if (r.feasible)
    body += ",\"best\":{\"w\":" + dv(r.best.w.w) + ",\"objective\":" + hx(r.best.objective) +
            ",\"score\":" + hx(r.best.score) + ",\"latency_ms\":" + hx(r.best.latency_ms) +
            ",\"iterations\":" + std::to_string(r.best.iterations) +
            ",\"converged\":" + std::to_string(r.best.converged ? 1 : 0) +
            ",\"out_of_range\":" + bv(r.best.out_of_range) + "}";
  emit("optbeta", cite, body);
}

std::vector<std::pair<double, double>> const_knots(double lat, double max_load) {
  return {{0.0, lat}, {max_load, lat}};
}

// test_latency.cpp:27-38
std::vector<std::pair<double, double>> random_knots(std::mt19937_64& rng) {
  std::uniform_real_distribution<double> unif(0.0, 1.0);
  int k = 3 + static_cast<int>(rng() % 4);
  std::vector<std::pair<double, double>> knots;
  double load = 0.0, lat = 20.0 + 200.0 * unif(rng);
  for (int i = 0; i < k; ++i) {
    knots.emplace_back(load, lat);
    load += 1.0 + 9.0 * unif(rng);
    lat += 300.0 * unif(rng);
  }
  return knots;
}

ScoreMatrix synth(int n, int m, uint64_t seed) {
  std::vector<std::string> models;
  std::vector<BetaShape> shapes;
  for (int i = 0; i < m; ++i) {
    models.push_back(std::string(1, static_cast<char>('A' + i)));
    double t = m > 1 ? static_cast<double>(i) / (m - 1) : 0.5;
    shapes.push_back({2.0 + 6.0 * t, 8.0 - 6.0 * t});
  }
  return synth_scores(n, models, shapes, seed);
}

// SURVEY.md §8d linear profile formula (model i at tp 1, rho 1)
std::vector<std::pair<double, double>> survey_knots(int i) {
  double b = 20.0 + 25.0 * i, s = 1.0 + 1.5 * i;
  return {{0.0, b}, {20.0, b + 20.0 * s}, {60.0, b + 140.0 * s}};
}

}  // namespace

int main(int argc, char** argv) {
  out = std::fopen(argc > 1 ? argv[1] : "reference_cases.json", "w");
  if (!out) return 1;
  std::fprintf(out, "{\"generator\":\"oracle/golden_gen.cpp\",\"cases\":[");

  // ---- test_score_dual.cpp --------------------------------------------------------------
  ScoreMatrix ex = testutil::make_scores({{0.9, 0.8}, {0.4, 0.7}});
  case_eval("test_score_dual.cpp:21-32", ex, {1.0, 1.0}, {0.0, 0.0});
  case_eval("test_score_dual.cpp:29-31", ex, {1.0, 1.0}, {0.5, 0.0});
  case_eval("test_score_dual.cpp:49-51", ex, {1.0, 1.0}, {0.1, 0.1});
  case_eval("test_score_dual.cpp:35-36", testutil::make_scores({{0.5, 0.5}}), {1.0, 0.0}, {0.0, 0.0});
  case_eval("test_score_dual.cpp:37-38", testutil::make_scores({{0.3, 0.7, 0.7}}), {0.0, 1.0, 0.0},
            {0.0, 0.0, 0.0});
  {  // shift invariance (:57-72)
    std::mt19937_64 rng(11);
    std::uniform_real_distribution<double> unif(-1.0, 1.0);
    for (int trial = 0; trial < 50; ++trial) {
      ScoreMatrix s = testutil::random_scores(12, 3, rng);
      TargetCounts c = testutil::random_integer_counts(12, 3, rng);
      std::vector<double> alpha{unif(rng), unif(rng), unif(rng)};
      double t = unif(rng);
      std::vector<double> shifted = alpha;
      for (double& a : shifted) a += t;
      case_eval("test_score_dual.cpp:57-72", s, c.counts, alpha);
      case_eval("test_score_dual.cpp:57-72", s, c.counts, shifted);
    }
  }
  case_solve("test_score_dual.cpp:74-81", ex, {1.0, 1.0});
  {  // forced + single model (:83-101)
    std::mt19937_64 rng(13);
    ScoreMatrix s = testutil::random_scores(9, 2, rng);
    case_solve("test_score_dual.cpp:83-92", s, {9.0, 0.0});
    ScoreMatrix one = testutil::random_scores(7, 1, rng);
    case_solve("test_score_dual.cpp:94-100", one, {7.0});
  }
  {  // weak duality prices (:134-149)
    std::mt19937_64 rng(31);
    std::uniform_real_distribution<double> unif(-1.0, 1.0);
    for (int trial = 0; trial < 30; ++trial) {
      int n = 4 + static_cast<int>(rng() % 5);
      int m = 2 + static_cast<int>(rng() % 2);
      ScoreMatrix s = testutil::random_scores(n, m, rng);
      TargetCounts c = testutil::random_integer_counts(n, m, rng);
      for (int k = 0; k < 10; ++k) {
        std::vector<double> alpha(m);
        for (double& a : alpha) a = unif(rng);
        if (k < 2) case_eval("test_score_dual.cpp:134-149", s, c.counts, alpha);
      }
    }
  }
  {  // strong duality (:151-164)
    std::mt19937_64 rng(41);
    for (int trial = 0; trial < 60; ++trial) {
      int n = 4 + 2 * static_cast<int>(rng() % 3);
      int m = 2 + static_cast<int>(rng() % 2);
      ScoreMatrix s = testutil::random_scores(n, m, rng);
      TargetCounts c = testutil::random_integer_counts(n, m, rng);
      case_solve("test_score_dual.cpp:151-164", s, c.counts);
    }
  }
  {  // duality-gap diagnostics (:166-181)
    std::mt19937_64 rng(43);
    for (int trial = 0; trial < 20; ++trial) {
      int n = 6 + static_cast<int>(rng() % 5);
      ScoreMatrix s = testutil::random_scores(n, 3, rng);
      TargetCounts c = testutil::random_integer_counts(n, 3, rng);
      case_solve("test_score_dual.cpp:166-181", s, c.counts);
    }
  }
  {  // convexity / subgradient (:183-208), first 40 of 200 trials
    std::mt19937_64 rng(51);
    std::uniform_real_distribution<double> unif(-1.0, 1.0);
    ScoreMatrix s = testutil::random_scores(30, 3, rng);
    std::vector<double> w = testutil::random_simplex(3, 2.0, rng);
    std::vector<double> c{30 * w[0], 30 * w[1], 30 * w[2]};
    for (int trial = 0; trial < 40; ++trial) {
      std::vector<double> a(3), b(3), mid(3);
      for (int i = 0; i < 3; ++i) {
        a[i] = unif(rng);
        b[i] = unif(rng);
        mid[i] = 0.5 * (a[i] + b[i]);
      }
      case_eval("test_score_dual.cpp:183-208", s, c, a);
      case_eval("test_score_dual.cpp:183-208", s, c, mid);
    }
  }
  {  // concavity in w (:210-226)
    std::mt19937_64 rng(61);
    ScoreMatrix s = testutil::random_scores(24, 3, rng);
    for (int trial = 0; trial < 10; ++trial) {
      std::vector<double> w1 = testutil::random_simplex(3, 1.5, rng);
      std::vector<double> w2 = testutil::random_simplex(3, 1.5, rng);
      std::vector<double> mid(3);
      for (int i = 0; i < 3; ++i) mid[i] = 0.5 * (w1[i] + w2[i]);
      case_solve("test_score_dual.cpp:210-226", s, {24 * w1[0], 24 * w1[1], 24 * w1[2]});
      case_solve("test_score_dual.cpp:210-226", s, {24 * mid[0], 24 * mid[1], 24 * mid[2]});
    }
  }
  {  // gauge + residuals (:228-241)
    std::mt19937_64 rng(71);
    ScoreMatrix s = testutil::random_scores(40, 3, rng);
    std::vector<double> w = testutil::random_simplex(3, 5.0, rng);
    case_solve("test_score_dual.cpp:228-241", s, {40 * w[0], 40 * w[1], 40 * w[2]});
  }

  // ---- test_latency.cpp -----------------------------------------------------------------
  {
    Scen two({{{0, 100}, {10, 200}}, {{0, 50}, {10, 150}}});
    case_latency("test_latency.cpp:137-146", two, {1.0, 0.0}, 10.0, 1.25);
    case_latency("test_latency.cpp:137-146", two, {0.5, 0.5}, 10.0, 1.25);
    Scen flat({{{0, 100}, {10, 100}}, {{0, 100}, {10, 100}}});
    case_latency("test_latency.cpp:129-136", flat, {0.5, 0.5}, 10.0, 1.25);
    Scen one({{{0, 100}, {10, 200}}});
    case_latency("test_latency.cpp:171-172", one, {1.0}, 10.0, 1.25);
    Scen g3({{{0, 100}, {10, 200}}, {{0, 42}, {10, 200}}});
    case_latency("test_latency.cpp:174-177", g3, {1.0, 0.0}, 10.0, 1.25);
    Scen oor({{{0, 100}, {10, 200}}, {{0, 50}, {100, 60}}});
    case_latency("test_latency.cpp:260-280", oor, {0.5, 0.5}, 20.0, 1.25);
    case_latency("test_latency.cpp:260-280", oor, {0.8, 0.2}, 20.0, 1.25);
    Scen shifted({{{2, 80}, {10, 200}}, {{0, 100}, {10, 200}}});
    case_latency("test_latency.cpp:97-99", shifted, {0.05, 0.95}, 20.0, 1.25);
    case_latency("test_latency.cpp:89-96", shifted, {0.75, 0.25}, 20.0, 1.25);
  }
  {  // random profiles, gradient test instances (:197-238)
    std::mt19937_64 rng(91);
    std::uniform_real_distribution<double> unif(0.0, 1.0);
    for (int t = 0; t < 40; ++t) {
      int m = 2 + static_cast<int>(rng() % 2);
      std::vector<std::vector<std::pair<double, double>>> ks;
      for (int i = 0; i < m; ++i) ks.push_back(random_knots(rng));
      double lambda = 1.0 + 12.0 * unif(rng);
      std::vector<double> w = testutil::random_simplex(m, 4.0, rng);
      case_latency("test_latency.cpp:197-238", Scen(ks), w, lambda, 1.25);
    }
  }

  // ---- test_routing_opt.cpp -------------------------------------------------------------
  case_simplex("test_routing_opt.cpp:41-56", {0.2, 0.8});
  case_simplex("test_routing_opt.cpp:41-56", {1.0, 1.0});
  case_simplex("test_routing_opt.cpp:41-56", {2.0, -1.0});
  {
    std::mt19937_64 rng(7);  // (:58-82)
    std::uniform_real_distribution<double> unif(-2.0, 2.0);
    for (int trial = 0; trial < 60; ++trial) {
      int m = 2 + trial % 2;
      std::vector<double> v(m);
      for (double& x : v) x = unif(rng);
      case_simplex("test_routing_opt.cpp:58-82", v);
    }
    std::mt19937_64 r2(8);
    for (int trial = 0; trial < 40; ++trial) {
      int m = 2 + static_cast<int>(r2() % 15);
      std::vector<double> v(m);
      for (double& x : v) x = unif(r2);
      case_simplex("routing_opt.cpp:37-68 (wide M)", v);
    }
  }
  {
    std::mt19937_64 rng(17);  // (:84-96)
    ScoreMatrix s = testutil::random_scores(10, 1, rng);
    case_optfrac("test_routing_opt.cpp:84-96", s, Scen({const_knots(50.0, 20.0)}), 0.5, 5.0,
                 100.0);
  }
  {
    std::mt19937_64 rng(19);  // (:98-110)
    std::uniform_real_distribution<double> hi(0.6, 0.95), lo(0.05, 0.4);
    std::vector<std::vector<double>> rows;
    for (int j = 0; j < 40; ++j) rows.push_back({hi(rng), lo(rng)});
    case_optfrac("test_routing_opt.cpp:98-110", testutil::make_scores(rows),
                 Scen({const_knots(80.0, 50.0), const_knots(80.0, 50.0)}), 0.0, 10.0, 1000.0);
  }
  {
    std::mt19937_64 rng(23);  // (:112-119)
    case_optfrac("test_routing_opt.cpp:112-119", testutil::random_scores(30, 2, rng),
                 Scen({const_knots(500.0, 50.0), const_knots(5.0, 50.0)}), 1e6, 10.0, 100.0);
  }
  {
    std::mt19937_64 rng(29);  // (:121-140)
    case_optfrac("test_routing_opt.cpp:121-140", testutil::random_scores(25, 3, rng),
                 Scen({const_knots(60.0, 50.0), const_knots(90.0, 50.0), const_knots(30.0, 50.0)}),
                 0.7, 12.0, 80.0);
  }
  {
    std::mt19937_64 rng(31);  // (:142-158)
    ScoreMatrix s = testutil::random_scores(8, 1, rng);
    case_optbeta("test_routing_opt.cpp:142-158", s, Scen({const_knots(50.0, 20.0)}), 5.0, 100.0);
    case_optbeta("test_routing_opt.cpp:142-158", s, Scen({const_knots(150.0, 20.0)}), 5.0, 100.0);
  }
  {
    std::mt19937_64 rng(37);  // (:160-178)
    ScoreMatrix s = testutil::random_scores(8, 1, rng);
    Scen sc({const_knots(50.0, 20.0)});
    BetaSearchParams p8;
    p8.beta_min = 0.0;
    p8.beta_max = 1.0;
    p8.epsilon = 1.0 / 8.0;
    case_optbeta("test_routing_opt.cpp:160-178", s, sc, 5.0, 100.0, p8);
    case_optbeta("test_routing_opt.cpp:160-178", s, sc, 5.0, 100.0);
    BetaSearchParams p5;
    p5.beta_min = 0.25;
    p5.beta_max = 0.25 + 0.3;
    p5.epsilon = 0.01;
    case_optbeta("test_routing_opt.cpp:160-178", s, sc, 5.0, 100.0, p5);
  }
  {
    std::mt19937_64 rng(41);  // (:180-193)
    case_optbeta("test_routing_opt.cpp:180-193", testutil::random_scores(20, 2, rng),
                 Scen({const_knots(500.0, 50.0), {{0.0, 5.0}, {2.0, 6.0}}}), 20.0, 50.0);
  }
  {
    std::mt19937_64 rng(43);  // (:195-215), 2 of 4 trials
    for (int trial = 0; trial < 2; ++trial) {
      ScoreMatrix s = testutil::random_scores(60, 2, rng);
      BetaSearchParams params;
      params.beta_min = 0.0;
      params.beta_max = 1e-12;
      params.epsilon = 1e-13;
      case_optbeta("test_routing_opt.cpp:195-215", s,
                   Scen({const_knots(60.0, 100.0), const_knots(60.0, 100.0)}), 10.0, 1e18, params);
    }
  }

  // ---- larger synthetic instances (workload.cpp synth_scores, SURVEY §8d profiles) -------
  {
    ScoreMatrix s = synth(2000, 4, 1);
    std::mt19937_64 rng(5);
    std::uniform_real_distribution<double> unif(-0.3, 0.3);
    for (int k = 0; k < 6; ++k) {
      std::vector<double> a(4);
      for (double& x : a) x = k ? unif(rng) : 0.0;
      case_eval("score_dual.cpp:25-49 (synth 2000x4)", s, {500, 500, 500, 500}, a);
    }
    SubgradientParams p;
    p.max_iters = 60;
    case_solve("score_dual.cpp:232-327 (synth, integral c)", s, {500, 500, 500, 500}, p);
    case_solve("score_dual.cpp:232-327 (synth, fractional c)", s, {311.5, 600.25, 488.25, 600}, p);
    p.init_alpha = {0.05, 0.0, 0.1, 0.02};
    case_solve("score_dual.cpp:251-258 (warm start)", s, {311.5, 600.25, 488.25, 600}, p);
    Scen sc({survey_knots(0), survey_knots(1), survey_knots(2), survey_knots(3)});
    PgaParams pp;
    pp.max_iters = 8;
    pp.dual.max_iters = 40;
    case_optfrac("routing_opt.cpp:70-136 (synth)", s, sc, 0.02, 40.0, 120.0, pp);
    BetaSearchParams bp;
    bp.pga = pp;
    bp.epsilon = (10.0 / 120.0) / 16.0;
    case_optbeta("routing_opt.cpp:138-173 (synth)", s, sc, 40.0, 120.0, bp);
  }
  {
    ScoreMatrix s = synth(1500, 8, 2);
    SubgradientParams p;
    p.max_iters = 50;
    case_solve("score_dual.cpp:232-327 (synth 1500x8 integral)", s,
               {187, 188, 187, 188, 187, 188, 187, 188}, p);
    std::vector<double> a{0.0, 0.01, 0.02, -0.01, 0.03, 0.0, 0.05, 0.04};
    case_eval("score_dual.cpp:25-49 (synth 1500x8)", s, {187, 188, 187, 188, 187, 188, 187, 188}, a);
  }
  std::fprintf(out, "\n],\"matrices\":[");
  for (size_t k = 0; k < matrices.size(); ++k)
    std::fprintf(out, "%s\n%s", k ? "," : "", matrices[k].c_str());
  std::fprintf(out, "\n]}\n");
  std::fclose(out);
  return 0;
}
