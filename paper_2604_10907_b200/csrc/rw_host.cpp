// rw_host.cpp — host-side pieces of the path that stay on the CPU: the synthetic workload
// generator, setup enumeration + retention (host path), and the
// order-deterministic reduction over per-setup records.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "rw_b200.h"

namespace {
thread_local std::string g_host_err;
constexpr double kEps = 1e-9;  // setup_search.cpp:16
}  // namespace

extern "C" {

// ---- f2: binary score files ---------------------------------------------
// The reference ingests scores as CSV (load_scores, workload.cpp:32-62: one strtod per
// entry — 160M of them at 10M x 16).  A .f64 score file is one read:
//   "RWSCORE1" | int64 n | int64 m | m x (int32 len, name bytes) | n*m float64, row-major
// (little-endian; scores[j * m + i] as workload.hpp:15).  Entries are validated like
// ScoreMatrix::validate (workload.cpp:23-29): finite and inside [0, 1].
static const char kMagic[8] = {'R', 'W', 'S', 'C', 'O', 'R', 'E', '1'};

const char* rw_host_last_error(void) { return g_host_err.c_str(); }

int rw_write_scores_f64(const char* path, int64_t n, int32_t m, const char* const* models,
                        const double* scores) {
  if (!path || n < 1 || m < 1 || !scores) return RW_ERR_VALIDATION;
  FILE* f = std::fopen(path, "wb");
  if (!f) {
    g_host_err = std::string("cannot write ") + path;
    return RW_ERR_CONFIG;
  }
  const int64_t hdr[2] = {n, (int64_t)m};
  bool ok = std::fwrite(kMagic, 1, 8, f) == 8 && std::fwrite(hdr, 8, 2, f) == 2;
  for (int i = 0; ok && i < m; ++i) {
    const char* name = models ? models[i] : "";
    const int32_t len = (int32_t)std::strlen(name);
    ok = std::fwrite(&len, 4, 1, f) == 1 && std::fwrite(name, 1, len, f) == (size_t)len;
  }
  ok = ok && std::fwrite(scores, sizeof(double), (size_t)n * m, f) == (size_t)n * m;
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) g_host_err = std::string("short write to ") + path;
  return ok ? RW_OK : RW_ERR_CONFIG;
}

// Header only when out == NULL (n, m and the names, '\0'-separated, into names[cap]).
int rw_read_scores_f64(const char* path, int64_t* n_out, int32_t* m_out, double* out,
                       int64_t out_cap, char* names, int64_t names_cap) {
  FILE* f = path ? std::fopen(path, "rb") : nullptr;
  if (!f) {
    g_host_err = std::string(path ? path : "(null)") + ": cannot open score file";
    return RW_ERR_CONFIG;  // a missing input file is a ConfigError in the reference
  }
  char magic[8];
  int64_t hdr[2];
  int rc = RW_OK;
  if (std::fread(magic, 1, 8, f) != 8 || std::memcmp(magic, kMagic, 8) != 0 ||
      std::fread(hdr, 8, 2, f) != 2 || hdr[0] < 1 || hdr[1] < 1 || hdr[1] > (1 << 20)) {
    g_host_err = std::string(path) + ": not a RWSCORE1 score file";
    std::fclose(f);
    return RW_ERR_CONFIG;
  }
  const int64_t n = hdr[0], m = hdr[1];
  std::vector<std::string> model(m);
  int64_t used = 0;
  for (int64_t i = 0; i < m; ++i) {
    int32_t len = 0;
    if (std::fread(&len, 4, 1, f) != 1 || len < 0 || len > 4096) rc = RW_ERR_CONFIG;
    if (rc) break;
    model[i].resize(len);
    if (len && std::fread(&model[i][0], 1, len, f) != (size_t)len) rc = RW_ERR_CONFIG;
    if (names && used + len + 1 <= names_cap) {
      std::memcpy(names + used, model[i].data(), len);
      names[used + len] = '\0';
    }
    used += len + 1;
  }
  if (rc) {
    g_host_err = std::string(path) + ": truncated header";
    std::fclose(f);
    return rc;
  }
  if (n_out) *n_out = n;
  if (m_out) *m_out = (int32_t)m;
  if (!out) {
    std::fclose(f);
    return RW_OK;
  }
  if (out_cap < n * m) {
    std::fclose(f);
    g_host_err = "rw_read_scores_f64: output buffer too small";
    return RW_ERR_VALIDATION;
  }
  if (std::fread(out, sizeof(double), (size_t)(n * m), f) != (size_t)(n * m)) {
    std::fclose(f);
    g_host_err = std::string(path) + ": truncated score data";
    return RW_ERR_CONFIG;
  }
  std::fclose(f);
  for (int64_t k = 0; k < n * m; ++k) {  // ScoreMatrix::validate (workload.cpp:23-29)
    const double v = out[k];
    if (!std::isfinite(v) || v < 0.0 || v > 1.0) {
      char buf[64];
      std::snprintf(buf, sizeof buf, "%.17g", v);
      g_host_err = "score matrix: entry for prompt 'p" + std::to_string(k / m + 1) +
                   "', model '" + model[k % m] + "' is " + buf + ", outside [0, 1]";
      return RW_ERR_VALIDATION;
    }
  }
  return RW_OK;
}

// workload.cpp:78-112: column i ~ Beta(a_i, b_i) = X/(X+Y), X~Gamma(a_i), Y~Gamma(b_i); one
// mt19937_64 for the whole matrix, columns drawn in model order, rows in prompt order.
int rw_synth_scores(int32_t n, int32_t m, const double* a, const double* b, uint64_t seed,
                    double* out) {
  if (n < 1 || m < 1) return RW_ERR_VALIDATION;
  for (int i = 0; i < m; ++i)
    if (!(a[i] > 0.0) || !(b[i] > 0.0)) return RW_ERR_VALIDATION;
  std::mt19937_64 engine(seed);
  for (int i = 0; i < m; ++i) {
    std::gamma_distribution<double> gx(a[i], 1.0), gy(b[i], 1.0);
    for (int j = 0; j < n; ++j) {
      double x = gx(engine);
      double y = gy(engine);
      while (x + y <= 0.0) {
        x = gx(engine);
        y = gy(engine);
      }
      out[static_cast<size_t>(j) * m + i] = x / (x + y);
    }
  }
  return RW_OK;
}

int rw_enumerate_retain(int32_t m, const int32_t* name_rank, const int32_t* tp_off,
                        const int32_t* tp_val, const int32_t* rho_off, const double* rho_val,
                        int32_t n_mem, const int32_t* mem_model, const int32_t* mem_tp,
                        const double* mem_frac, int32_t gpu_count, double rho_floor, int64_t cap,
                        int64_t* n_enum, int32_t* verdict, int32_t* tp_out, double* rho_out) {
  if (m < 1) return RW_ERR_VALIDATION;
  if (gpu_count < 1) return RW_ERR_VALIDATION;                      // :143
  if (!(rho_floor > 0.0) || rho_floor > 1.0) return RW_ERR_VALIDATION;  // :144-145
  // per-model flattened choices, tp-major (setup_search.cpp:104-108)
  std::vector<std::vector<std::pair<int, double>>> choice(m);
  for (int i = 0; i < m; ++i) {
    if (tp_off[i + 1] <= tp_off[i] || rho_off[i + 1] <= rho_off[i]) return RW_ERR_VALIDATION;
    for (int a = tp_off[i]; a < tp_off[i + 1]; ++a)
      for (int r = rho_off[i]; r < rho_off[i + 1]; ++r) choice[i].push_back({tp_val[a], rho_val[r]});
  }
  auto mem_at = [&](int model, int tp, double* frac) {
    for (int k = 0; k < n_mem; ++k)
      if (mem_model[k] == model && mem_tp[k] == tp) {
        *frac = mem_frac[k];
        return true;
      }
    return false;
  };
  int64_t total = 1;
  for (const auto& c : choice) total *= static_cast<int64_t>(c.size());
  *n_enum = total;
  // Every candidate's verdict is independent: the enumeration range is split over host
  // threads (f1), each running the odometer from its chunk's first id.
  auto run_range = [&](int64_t lo, int64_t hi) -> int {
  std::vector<size_t> idx(m, 0);
  {
    int64_t rem = lo;  // mixed-radix digits of lo, model 0 most significant
    for (int pos = m - 1; pos >= 0; --pos) {
      idx[pos] = (size_t)(rem % (int64_t)choice[pos].size());
      rem /= (int64_t)choice[pos].size();
    }
  }
  struct Shard {
    int model;
    double frac;
  };
  std::vector<Shard> shards;
  std::vector<size_t> order;
  std::vector<double> remaining;
  std::vector<uint64_t> occupied;  // bit per model (m <= 64)
  for (int64_t id = lo; id < hi; ++id) {
    // demand window (:146-148)
    double demand = 0.0;
    for (int i = 0; i < m; ++i) demand += choice[i][idx[i]].first * choice[i][idx[i]].second;
    int v = 0;
    if (demand < gpu_count * rho_floor - kEps) v = 1;
    else if (demand > gpu_count + kEps) v = 2;
    else {
      // FFD with anti-affinity (:55-97)
      shards.clear();
      for (int i = 0; i < m; ++i) {
        double frac;
        if (!mem_at(i, choice[i][idx[i]].first, &frac)) return RW_ERR_CONFIG;
        if (!(frac > 0.0) || frac > 1.0) return RW_ERR_VALIDATION;
        for (int s = 0; s < choice[i][idx[i]].first; ++s) shards.push_back({i, frac});
      }
      order.resize(shards.size());
      for (size_t k = 0; k < order.size(); ++k) order[k] = k;
      std::stable_sort(order.begin(), order.end(), [&](size_t x, size_t y) {
        if (shards[x].frac != shards[y].frac) return shards[x].frac > shards[y].frac;
        int rx = name_rank ? name_rank[shards[x].model] : shards[x].model;
        int ry = name_rank ? name_rank[shards[y].model] : shards[y].model;
        return rx < ry;
      });
      remaining.assign(gpu_count, 1.0);
      occupied.assign(gpu_count, 0ull);
      bool ok = true;
      for (size_t k : order) {
        const Shard& sh = shards[k];
        bool placed = false;
        for (int g = 0; g < gpu_count; ++g) {
          if (remaining[g] >= sh.frac - kEps && !((occupied[g] >> sh.model) & 1ull)) {
            remaining[g] -= sh.frac;
            occupied[g] |= 1ull << sh.model;
            placed = true;
            break;
          }
        }
        if (!placed) {
          ok = false;
          break;
        }
      }
      v = ok ? 0 : 3;
    }
    verdict[id] = v;
    for (int i = 0; i < m; ++i) {
      tp_out[id * m + i] = choice[i][idx[i]].first;
      rho_out[id * m + i] = choice[i][idx[i]].second;
    }
    // odometer, model 0 most significant (:115-128)
    for (int pos = m - 1; pos >= 0; --pos) {
      if (++idx[pos] < choice[pos].size()) break;
      idx[pos] = 0;
    }
  }
  return RW_OK;
  };
  const int64_t count = std::min(total, cap);
  const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
  const int nt = (int)std::min<int64_t>(hw, std::max<int64_t>(1, count / 4096));
  if (nt <= 1) return run_range(0, count);
  std::vector<int> rcs(nt, RW_OK);
  std::vector<std::thread> pool;
  for (int t = 0; t < nt; ++t)
    pool.emplace_back([&, t] { rcs[t] = run_range(count * t / nt, count * (t + 1) / nt); });
  for (auto& th : pool) th.join();
  for (int rc : rcs)
    if (rc != RW_OK) return rc;  // the first failing chunk in enumeration order
  return RW_OK;
}

int64_t rw_reduce_records(int64_t n, const rw_setup_record* r) {
  // setup_search.cpp:246-253 scans in enumeration order keeping the first on full ties;
  // with records in arbitrary (sharded) order the equivalent key is (score desc,
  // latency asc, setup_id asc).
  int64_t best = -1;
  for (int64_t k = 0; k < n; ++k) {
    if (!r[k].feasible) continue;
    if (best < 0) {
      best = k;
      continue;
    }
    const rw_setup_record& a = r[k];
    const rw_setup_record& b = r[best];
    if (a.score > b.score || (a.score == b.score && a.latency_ms < b.latency_ms) ||
        (a.score == b.score && a.latency_ms == b.latency_ms && a.setup_id < b.setup_id))
      best = k;
  }
  return best;
}

}  // extern "C"
