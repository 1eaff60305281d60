// libcoconet_engine.so — the drop-in host (include/coconet/gpu_engine.hpp)
// behind a small C entry point, mirroring the `ccopt run` flow
// (tools/ccopt.cpp:184-193): program JSON (+ schedule) -> gen_decl_values ->
// GpuEngine::run -> RunReport. Built against the reference's DSL headers, which
// are the drop-in surface (json_io.hpp, transform.hpp, runtime.hpp).
#include <cstring>
#include <string>

#include "ccopt/json_io.hpp"
#include "ccopt/transform.hpp"
#include "coconet/gpu_engine.hpp"
#include "coconet/gpu_tune.hpp"

namespace {

thread_local std::string g_err;

struct Session {
  ccopt::Program base, sched;
  ccopt::ValueMap in_base, in_sched;
  ccopt::RunReport rep;
  bool ran = false;
  double device_ms = 0;
  uint64_t launches = 0;
  std::vector<std::string> lowering;
};

int fail(const ccopt::Error& e) {
  g_err = e.what();
  return -(int(e.code()) + 1);
}
int fail_std(const std::exception& e) {
  g_err = e.what();
  return -1000;
}

std::map<std::string, int64_t> dims_of(const char* j) {
  std::map<std::string, int64_t> d;
  if (j && *j) {
    const ccopt::Json parsed = ccopt::Json::parse(j);  // keep alive across the loop
    for (auto& [k, v] : parsed.items()) d[k] = v.get<int64_t>();
  }
  return d;
}

int copy_out(const std::string& s, char* buf, int64_t len) {
  if (int64_t(s.size()) + 1 > len) return -int(s.size() + 1);
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return int(s.size());
}

}  // namespace

extern "C" {

const char* coconet_engine_last_error() { return g_err.c_str(); }

// program + schedule (apply_schedule), or program + an already scheduled
// program (sched_json), as JSON texts; dims = size symbols.
void* coconet_engine_open(const char* program_json, const char* schedule_json, const char* sched_json,
                          const char* dims_json) {
  try {
    auto* s = new Session();
    auto dims = dims_of(dims_json);
    s->base = ccopt::program_from_json(ccopt::Json::parse(program_json), dims);
    if (sched_json && *sched_json)
      s->sched = ccopt::program_from_json(ccopt::Json::parse(sched_json), dims);
    else if (schedule_json && *schedule_json)
      s->sched = ccopt::apply_schedule(s->base, ccopt::schedule_from_json(ccopt::Json::parse(schedule_json)));
    else
      s->sched = s->base;
    return s;
  } catch (const ccopt::Error& e) {
    fail(e);
  } catch (const std::exception& e) {
    fail_std(e);
  }
  return nullptr;
}

void coconet_engine_close(void* h) { delete static_cast<Session*>(h); }

int coconet_engine_gen(void* h, uint64_t seed) {
  auto* s = static_cast<Session*>(h);
  try {
    s->in_base = ccopt::gen_decl_values(s->base, seed);
    s->in_sched = ccopt::gen_decl_values(s->sched, seed);
    return 0;
  } catch (const ccopt::Error& e) {
    return fail(e);
  }
}

// rank's global view of a decl (sliced decls keep their slice), both programs
int coconet_engine_set(void* h, const char* name, int rank, const float* data, int64_t n) {
  auto* s = static_cast<Session*>(h);
  try {
    for (ccopt::ValueMap* m : {&s->in_base, &s->in_sched}) {
      ccopt::TensorVal& t = m->at(name);
      if (n != ccopt::num_elems(t.view.global)) throw ccopt::Error(ccopt::ErrCode::ShapeMismatch, "set size");
      auto& dst = t.per_rank.at(size_t(rank));
      if (t.view.layout.is_sliced())
        for (int64_t li = 0; li < t.view.local_elems(); ++li) dst[size_t(li)] = data[t.view.to_global(rank, li)];
      else
        std::memcpy(dst.data(), data, size_t(n) * sizeof(float));
    }
    return 0;
  } catch (const ccopt::Error& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail_std(e);
  }
}

// World all-gather supplied by the caller for DISTRIBUTED runs (rank order,
// `bytes` in, world * bytes out; collective over every process).
typedef void (*coconet_engine_allgather_fn)(const void* in, size_t bytes, void* out, void* user);

// which: 0 = scheduled program, 1 = base program. rank < 0: VIRTUAL (every
// rank in this process); rank >= 0: DISTRIBUTED, this process is world rank
// `rank` of `world` and `allgather` bootstraps the peer mappings and
// assembles the results (every process gets the same report).
int coconet_engine_run_dist(void* h, uint64_t seed, int which, int device, int math, int fused, int rank, int world,
                            coconet_engine_allgather_fn allgather, void* user) {
  auto* s = static_cast<Session*>(h);
  try {
    coconet::GpuOptions opt;
    opt.device = device;
    opt.math = math;
    opt.fused_kernels = fused != 0;
    if (rank >= 0) {
      opt.comm.rank = rank;
      opt.comm.world = world;
      opt.comm.allgather = [allgather, user](const void* in, size_t bytes, void* out) { allgather(in, bytes, out, user); };
    }
    const ccopt::Program& p = which == 0 ? s->sched : s->base;
    coconet::GpuEngine e(p, ccopt::CommConfig{}, seed, opt);
    s->rep = e.run(which == 0 ? s->in_sched : s->in_base);
    s->device_ms = e.device_ms();
    s->launches = e.launches();
    s->lowering = e.lowering();
    s->ran = true;
    return 0;
  } catch (const ccopt::Error& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail_std(e);
  }
}

int coconet_engine_run(void* h, uint64_t seed, int which, int device, int math, int fused) {
  return coconet_engine_run_dist(h, seed, which, device, math, fused, -1, 0, nullptr, nullptr);
}

uint64_t coconet_engine_digest(void* h) { return static_cast<Session*>(h)->rep.digest; }

int coconet_engine_report(void* h, char* buf, int64_t len) {
  auto* s = static_cast<Session*>(h);
  ccopt::Json j;
  j["comm_bytes"] = s->rep.comm_bytes;
  j["intergroup_bytes"] = s->rep.intergroup_bytes;
  j["traffic_saved_bytes"] = s->rep.traffic_saved_bytes;
  j["kernel_steps"] = s->rep.kernel_steps;
  j["memory_elems"] = s->rep.memory_elems;
  j["simulated_time"] = s->rep.simulated_time;
  j["digest"] = s->rep.digest;
  j["device_ms"] = s->device_ms;
  j["launches"] = s->launches;
  j["lowering"] = s->lowering;
  return copy_out(j.dump(), buf, len);
}

int coconet_engine_result(void* h, const char* key, int idx, float* out, int64_t n) {
  auto* s = static_cast<Session*>(h);
  try {
    const auto& arr = s->rep.results.at(key).data.at(size_t(idx));
    if (int64_t(arr.size()) != n) throw ccopt::Error(ccopt::ErrCode::ShapeMismatch, "result size");
    std::memcpy(out, arr.data(), size_t(n) * sizeof(float));
    return 0;
  } catch (const ccopt::Error& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail_std(e);
  }
}

// ccopt tune with candidates ranked by measured device time (gpu_tune.hpp):
// program JSON + size symbols -> the tune report JSON in buf (returns its
// length, -needed if buf is too small, or a negative status).
int coconet_engine_tune(const char* program_json, const char* dims_json, uint64_t seed, double tol, int device,
                        int math, int reps, char* buf, int64_t len) {
  try {
    ccopt::Program p = ccopt::program_from_json(ccopt::Json::parse(program_json), dims_of(dims_json));
    ccopt::TuneConfig cfg;
    cfg.seed = seed;
    cfg.tol = tol;
    coconet::GpuOptions opt;
    opt.device = device;
    opt.math = math;
    return copy_out(coconet::gpu_tune_report_to_json(coconet::gpu_tune(p, cfg, opt, reps)).dump(), buf, len);
  } catch (const ccopt::Error& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail_std(e);
  }
}

}  // extern "C"
