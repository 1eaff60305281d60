// gpu_tune — the reference schedule search (ccopt::tune, autotune.hpp:285-315)
// with candidates ranked by MEASURED device time on B200 instead of the
// simulated cost model.
//
// The search space is the reference's own: ccopt::enumerate_schedules
// (autotune.hpp:237-281, the fusion pre-pass plus bounded BFS over the
// transformation directives). Every candidate is
//   - applied with ccopt::apply_schedule,
//   - executed `reps` times on coconet::GpuEngine (fresh inputs from
//     gen_decl_values each time, exactly like the reference's tune),
//   - verified against ccopt::oracle_results on the base program with
//     ccopt::compare_results; a deviation above tol throws CandidateFailed, as
//     the reference does (it signals a transformation or lowering bug),
// and keeps the reference's simulated_time / comm_bytes / kernel_steps next to
// the measured median device_ms. The winner is the fastest measured candidate;
// ties (within 1e-9 relative) break like the reference: fewer kernel steps,
// then the schedule string. `simulated_winner` is the reference's own pick on
// the same candidates, so the two rankings can be compared.
#pragma once

#include <algorithm>
#include <cmath>
#include <vector>

#include "ccopt/autotune.hpp"
#include "coconet/gpu_engine.hpp"

namespace coconet {

struct GpuCandidate {
  ccopt::Candidate ref;          // schedule, simulated_time, comm_bytes, kernel_steps, deviation
  double device_ms = 0.0;        // median over reps
  std::vector<double> device_ms_reps;
  uint64_t digest = 0;
};

struct GpuTuneReport {
  std::vector<GpuCandidate> candidates;
  size_t winner = 0;            // by measured device time
  size_t simulated_winner = 0;  // the reference's cost-model pick
};

inline bool better(double a, double b, int ka, int kb, const std::string& sa, const std::string& sb) {
  const double scale = std::max({1.0, std::abs(a), std::abs(b)});
  const bool tie = std::abs(a - b) <= 1e-9 * scale;
  return (!tie && a < b) || (tie && (ka < kb || (ka == kb && sa < sb)));
}

inline GpuTuneReport gpu_tune(const ccopt::Program& base, const ccopt::TuneConfig& cfg, GpuOptions opt = {},
                              int reps = 3) {
  using namespace ccopt;
  GpuTuneReport rep;
  auto oracle_ref = oracle_results(base, gen_decl_values(base, cfg.seed), cfg.seed);
  for (auto& sched : enumerate_schedules(base, cfg)) {
    Program p = apply_schedule(base, sched);
    GpuCandidate c;
    c.ref.schedule = sched;
    for (int i = 0; i < std::max(1, reps); ++i) {
      GpuEngine eng(p, cfg.comm, cfg.seed, opt);
      RunReport run = eng.run(gen_decl_values(p, cfg.seed));
      c.device_ms_reps.push_back(eng.device_ms());
      if (i == 0) {
        c.ref.simulated_time = run.simulated_time;
        for (auto b : run.comm_bytes) c.ref.comm_bytes += b;
        c.ref.kernel_steps = run.kernel_steps;
        c.ref.deviation = compare_results(oracle_ref, run.results);
        c.digest = run.digest;
        if (c.ref.deviation > cfg.tol)
          throw Error(ErrCode::CandidateFailed,
                      "schedule [" + sched.str() + "] deviates " + std::to_string(c.ref.deviation));
      }
    }
    std::vector<double> s = c.device_ms_reps;
    std::sort(s.begin(), s.end());
    c.device_ms = s[s.size() / 2];
    rep.candidates.push_back(std::move(c));
  }
  for (size_t i = 1; i < rep.candidates.size(); ++i) {
    const GpuCandidate& a = rep.candidates[i];
    const GpuCandidate& w = rep.candidates[rep.winner];
    const GpuCandidate& sw = rep.candidates[rep.simulated_winner];
    if (better(a.device_ms, w.device_ms, a.ref.kernel_steps, w.ref.kernel_steps, a.ref.schedule.str(),
               w.ref.schedule.str()))
      rep.winner = i;
    if (better(a.ref.simulated_time, sw.ref.simulated_time, a.ref.kernel_steps, sw.ref.kernel_steps,
               a.ref.schedule.str(), sw.ref.schedule.str()))
      rep.simulated_winner = i;
  }
  return rep;
}

// tune_report_to_json (autotune.hpp:317-333) plus the measured fields.
inline ccopt::Json gpu_tune_report_to_json(const GpuTuneReport& rep) {
  using namespace ccopt;
  Json j;
  j["candidates"] = Json::array();
  for (auto& c : rep.candidates) {
    Json cj;
    cj["schedule"] = schedule_to_json(c.ref.schedule);
    cj["simulated_time"] = c.ref.simulated_time;
    cj["comm_bytes"] = c.ref.comm_bytes;
    cj["kernel_steps"] = c.ref.kernel_steps;
    cj["deviation"] = c.ref.deviation;
    cj["device_ms"] = c.device_ms;
    cj["device_ms_reps"] = c.device_ms_reps;
    char buf[32];
    std::snprintf(buf, sizeof buf, "%016llx", (unsigned long long)c.digest);
    cj["digest"] = buf;
    j["candidates"].push_back(cj);
  }
  j["winner"] = rep.winner;
  j["winner_schedule"] = schedule_to_json(rep.candidates.at(rep.winner).ref.schedule);
  j["ranked_by"] = "device_ms";
  j["simulated_winner"] = rep.simulated_winner;
  j["simulated_winner_schedule"] = schedule_to_json(rep.candidates.at(rep.simulated_winner).ref.schedule);
  return j;
}

}  // namespace coconet
