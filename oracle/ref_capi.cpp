// C-ABI shim over the UNMODIFIED reference (ccopt) headers, compiled in place
// from /root/reference/proj/include by oracle/Makefile into oracle/_ref/.
//
// TEST INFRASTRUCTURE ONLY. This is the checker: the parity tests, smoke() and
// bench.py's cpu_baseline / --impl reference leg load it to run the
// reference's own sequential oracle (oracle.hpp:181-190) and simulated Engine
// (runtime.hpp:98-138) on exactly the inputs the GPU path sees. Nothing in the
// product package links or calls it.
//
// Mirrors the `ccopt run` flow (tools/ccopt.cpp:184-193): load program JSON
// (json_io.hpp:307-357), apply a schedule (transform.hpp:594-604), generate
// inputs (state.hpp:55-74), run oracle + Engine, compare (state.hpp:251-265),
// digest (state.hpp:267-274).

#include <chrono>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "ccopt/json_io.hpp"
#include "ccopt/oracle.hpp"
#include "ccopt/runtime.hpp"
#include "ccopt/transform.hpp"

using namespace ccopt;

namespace {

thread_local std::string g_err;

struct Run {
  bool done = false;
  std::map<std::string, Collected> results;
  RunReport report;  // valid for engine runs
  double wall_s = 0;
  ValueMap vals;     // final value map (oracle runs keep it for node lookups)
};

struct Session {
  Program base;
  Program sched;
  bool has_sched = false;
  ValueMap in_base, in_sched;
  Run runs[3];  // 0 = oracle(base), 1 = Engine(sched), 2 = Engine(base)
};

int fail(const Error& e) {
  g_err = e.what();
  return -(int(e.code()) + 1);
}
int fail_std(const std::exception& e) {
  g_err = e.what();
  return -1000;
}

std::map<std::string, int64_t> parse_dims(const char* dims_json) {
  std::map<std::string, int64_t> dims;
  Json j = Json::parse(dims_json);
  for (auto& [k, v] : j.items()) dims[k] = v.get<int64_t>();
  return dims;
}

// Writes rank `rank`'s view of a global array into a TensorVal: Local and
// Replicated take the whole array; Sliced keeps the rank's own slice.
void assign_rank(TensorVal& t, int rank, const float* data, int64_t n) {
  int64_t total = num_elems(t.view.global);
  if (n != total) throw Error(ErrCode::ShapeMismatch, "set: element count mismatch");
  auto& dst = t.per_rank.at(size_t(rank));
  if (t.view.layout.is_sliced()) {
    for (int64_t li = 0; li < t.view.local_elems(); ++li)
      dst[size_t(li)] = data[t.view.to_global(rank, li)];
  } else {
    std::memcpy(dst.data(), data, size_t(n) * sizeof(float));
  }
}

const Run& need_run(Session* s, int which) {
  if (which < 0 || which > 2 || !s->runs[which].done)
    throw Error(ErrCode::InvalidInput, "run " + std::to_string(which) + " has not been executed");
  return s->runs[which];
}

int copy_out(const std::string& text, char* buf, int64_t len) {
  if (int64_t(text.size()) + 1 > len) return -int(text.size() + 1);
  std::memcpy(buf, text.c_str(), text.size() + 1);
  return int(text.size());
}

}  // namespace

extern "C" {

const char* ccref_last_error() { return g_err.c_str(); }

void* ccref_open(const char* program_json, const char* schedule_json, const char* dims_json) {
  try {
    auto* s = new Session();
    auto dims = parse_dims(dims_json);
    s->base = program_from_json(Json::parse(program_json), dims);
    auto diags = validate_program(s->base);
    if (!diags.empty()) throw Error(ErrCode::InvalidInput, "invalid program: " + diags[0]);
    if (schedule_json && *schedule_json) {
      s->sched = apply_schedule(s->base, schedule_from_json(Json::parse(schedule_json)));
      s->has_sched = true;
    } else {
      s->sched = s->base;
    }
    return s;
  } catch (const Error& e) {
    fail(e);
  } catch (const std::exception& e) {
    fail_std(e);
  }
  return nullptr;
}

// Opens an already-transformed program (e.g. an authored fused LAMB program)
// together with its unscheduled base, both as JSON text.
void* ccref_open_pair(const char* base_json, const char* sched_json, const char* dims_json) {
  try {
    auto* s = new Session();
    auto dims = parse_dims(dims_json);
    s->base = program_from_json(Json::parse(base_json), dims);
    s->sched = program_from_json(Json::parse(sched_json), dims);
    s->has_sched = true;
    return s;
  } catch (const Error& e) {
    fail(e);
  } catch (const std::exception& e) {
    fail_std(e);
  }
  return nullptr;
}

void ccref_close(void* h) { delete static_cast<Session*>(h); }

int ccref_gen(void* h, uint64_t seed) {
  auto* s = static_cast<Session*>(h);
  try {
    s->in_base = gen_decl_values(s->base, seed);
    s->in_sched = gen_decl_values(s->sched, seed);
    for (auto& r : s->runs) r = Run{};
    return 0;
  } catch (const Error& e) {
    return fail(e);
  }
}

// Overrides a decl's value on one (group-relative) rank, in both the base and
// the scheduled input maps. `data` is the rank's global view (whole tensor).
int ccref_set(void* h, const char* name, int rank, const float* data, int64_t n) {
  auto* s = static_cast<Session*>(h);
  try {
    for (ValueMap* m : {&s->in_base, &s->in_sched}) {
      auto it = m->find(name);
      if (it == m->end()) throw Error(ErrCode::UnknownId, std::string("no decl ") + name);
      assign_rank(it->second, rank, data, n);
    }
    return 0;
  } catch (const Error& e) {
    return fail(e);
  }
}

// Reads a decl's generated input on one rank as its global view (sliced decls
// fill only the rank's own slice; the rest is zero).
int ccref_get_input(void* h, const char* name, int rank, float* out, int64_t n) {
  auto* s = static_cast<Session*>(h);
  try {
    const TensorVal& t = s->in_base.at(name);
    if (n != num_elems(t.view.global)) throw Error(ErrCode::ShapeMismatch, "get_input size");
    const auto& src = t.per_rank.at(size_t(rank));
    if (t.view.layout.is_sliced()) {
      std::memset(out, 0, size_t(n) * sizeof(float));
      for (int64_t li = 0; li < t.view.local_elems(); ++li)
        out[t.view.to_global(rank, li)] = src[size_t(li)];
    } else {
      std::memcpy(out, src.data(), size_t(n) * sizeof(float));
    }
    return 0;
  } catch (const Error& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail_std(e);
  }
}

// which: 0 = oracle on the base program, 1 = Engine on the scheduled program,
// 2 = Engine on the base program. threaded selects ExecMode::Threaded.
int ccref_run(void* h, uint64_t seed, int which, int threaded, double* wall_s) {
  auto* s = static_cast<Session*>(h);
  try {
    Run& r = s->runs[which];
    r = Run{};
    auto t0 = std::chrono::steady_clock::now();
    if (which == 0) {
      r.vals = oracle_execute(s->base, s->in_base, seed);
      r.results = collect_results(s->base, r.vals);
    } else {
      CommConfig cfg;
      cfg.mode = threaded ? ExecMode::Threaded : ExecMode::RoundRobin;
      const Program& p = which == 1 ? s->sched : s->base;
      const ValueMap& in = which == 1 ? s->in_sched : s->in_base;
      r.report = Engine(p, cfg, seed).run(in);
      r.results = r.report.results;
    }
    r.wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    r.done = true;
    if (wall_s) *wall_s = r.wall_s;
    return 0;
  } catch (const Error& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail_std(e);
  }
}

// Times Engine::run alone (inputs copied before the clock starts), as
// BASELINE.md §2 does. Returns seconds.
double ccref_time_engine(void* h, uint64_t seed, int which, int threaded) {
  auto* s = static_cast<Session*>(h);
  try {
    CommConfig cfg;
    cfg.mode = threaded ? ExecMode::Threaded : ExecMode::RoundRobin;
    const Program& p = which == 1 ? s->sched : s->base;
    ValueMap in = which == 1 ? s->in_sched : s->in_base;
    Engine e(p, cfg, seed);
    auto t0 = std::chrono::steady_clock::now();
    RunReport rep = e.run(std::move(in));
    double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    s->runs[which].report = rep;
    s->runs[which].results = rep.results;
    s->runs[which].wall_s = dt;
    s->runs[which].done = true;
    return dt;
  } catch (const Error& e) {
    fail(e);
  } catch (const std::exception& e) {
    fail_std(e);
  }
  return -1.0;
}

// Result keys of a run, newline separated, in map (digest) order.
int ccref_result_keys(void* h, int which, char* buf, int64_t len) {
  try {
    const Run& r = need_run(static_cast<Session*>(h), which);
    std::string out;
    for (auto& [k, c] : r.results) out += k + "\t" + std::to_string(c.data.size()) + "\t" +
                                          std::to_string(num_elems(c.shape)) + "\n";
    return copy_out(out, buf, len);
  } catch (const Error& e) {
    return fail(e);
  }
}

// Copies one collected result array (per_rank index `idx`, 0 for
// replicated/sliced values) into `out`.
int ccref_result(void* h, int which, const char* key, int idx, float* out, int64_t n) {
  try {
    const Run& r = need_run(static_cast<Session*>(h), which);
    const Collected& c = r.results.at(key);
    const auto& arr = c.data.at(size_t(idx));
    if (int64_t(arr.size()) != n) throw Error(ErrCode::ShapeMismatch, "result size");
    std::memcpy(out, arr.data(), size_t(n) * sizeof(float));
    return 0;
  } catch (const Error& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail_std(e);
  }
}

// Value of any node or decl after an oracle run, rank `rank`, local storage.
int ccref_value(void* h, const char* id, int rank, float* out, int64_t n) {
  try {
    const Run& r = need_run(static_cast<Session*>(h), 0);
    const auto& arr = r.vals.at(id).per_rank.at(size_t(rank));
    if (int64_t(arr.size()) != n) throw Error(ErrCode::ShapeMismatch, "value size");
    std::memcpy(out, arr.data(), size_t(n) * sizeof(float));
    return 0;
  } catch (const Error& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail_std(e);
  }
}

uint64_t ccref_digest(void* h, int which) {
  try {
    return digest_results(need_run(static_cast<Session*>(h), which).results);
  } catch (const Error& e) {
    fail(e);
    return 0;
  }
}

double ccref_compare(void* h, int a, int b) {
  try {
    auto* s = static_cast<Session*>(h);
    return compare_results(need_run(s, a).results, need_run(s, b).results);
  } catch (const Error& e) {
    fail(e);
    return -1.0;
  }
}

// RunReport counters of an Engine run as JSON (runtime.hpp:32-42).
int ccref_report(void* h, int which, char* buf, int64_t len) {
  try {
    const Run& r = need_run(static_cast<Session*>(h), which);
    Json j;
    j["comm_bytes"] = r.report.comm_bytes;
    j["intergroup_bytes"] = r.report.intergroup_bytes;
    j["traffic_saved_bytes"] = r.report.traffic_saved_bytes;
    j["kernel_steps"] = r.report.kernel_steps;
    j["memory_elems"] = r.report.memory_elems;
    j["simulated_time"] = r.report.simulated_time;
    j["digest"] = r.report.digest;
    j["wall_s"] = r.wall_s;
    return copy_out(j.dump(), buf, len);
  } catch (const Error& e) {
    return fail(e);
  }
}

// which: 0 = base, 1 = scheduled program, via program_to_json (json_io.hpp:359-401).
int ccref_program_json(void* h, int which, char* buf, int64_t len) {
  auto* s = static_cast<Session*>(h);
  return copy_out(program_to_json(which == 0 ? s->base : s->sched).dump(), buf, len);
}

uint64_t ccref_fnv1a(const void* data, int64_t n, uint64_t h) { return fnv1a(data, size_t(n), h); }

double ccref_counter_uniform(uint64_t seed, uint64_t key, uint64_t idx) {
  return counter_uniform(seed, key, idx);
}

// build_bucket_table (runtime.hpp:592-614): writes (tensor index, offset,
// extent) per bucket; returns the bucket count (or -needed if cap too small).
int64_t ccref_bucket_table(int n, const int64_t* counts, int64_t* tensor, int64_t* offset,
                           int64_t* extent, int64_t cap) {
  try {
    std::vector<std::pair<std::string, int64_t>> ts;
    for (int i = 0; i < n; ++i) ts.push_back({std::to_string(i), counts[i]});
    BucketTable t = build_bucket_table(ts);
    if (int64_t(t.buckets.size()) > cap) return -int64_t(t.buckets.size());
    for (size_t b = 0; b < t.buckets.size(); ++b) {
      tensor[b] = std::stoll(t.buckets[b].tensor);
      offset[b] = t.buckets[b].offset;
      extent[b] = t.buckets[b].extent;
    }
    return int64_t(t.buckets.size());
  } catch (const Error& e) {
    return fail(e);
  }
}

int64_t ccref_bucket_metadata_bytes(int n, const int64_t* counts) {
  std::vector<std::pair<std::string, int64_t>> ts;
  for (int i = 0; i < n; ++i) ts.push_back({std::to_string(i), counts[i]});
  return build_bucket_table(ts).metadata_bytes();
}

// scattered_collective (runtime.hpp:624-675) over `n` tensors, `world` ranks.
// data: for tensor i, rank r: data[i][r*counts[i] ...]; results written to out
// with the same layout. Returns 0 or a negative ErrCode.
int ccref_scattered_allreduce(int n, const int64_t* counts, int world, const float* const* data,
                              float* const* out) {
  try {
    std::vector<std::pair<std::string, int64_t>> sizes;
    std::map<std::string, std::vector<std::vector<float>>> tensors;
    for (int i = 0; i < n; ++i) {
      std::string name = "t" + std::to_string(i);
      sizes.push_back({name, counts[i]});
      auto& pr = tensors[name];
      pr.assign(size_t(world), std::vector<float>(size_t(counts[i])));
      for (int r = 0; r < world; ++r)
        std::memcpy(pr[size_t(r)].data(), data[i] + int64_t(r) * counts[i],
                    size_t(counts[i]) * sizeof(float));
    }
    BucketTable table = build_bucket_table(sizes);
    ScatteredResult res = scattered_collective(CommConfig{}, table, OpKind::AllReduce,
                                               Reducer::Sum, tensors, world);
    for (int i = 0; i < n; ++i) {
      auto& pr = res.per_tensor.at("t" + std::to_string(i));
      for (int r = 0; r < world; ++r)
        std::memcpy(out[i] + int64_t(r) * counts[i], pr[size_t(r)].data(),
                    size_t(counts[i]) * sizeof(float));
    }
    return 0;
  } catch (const Error& e) {
    return fail(e);
  }
}

}  // extern "C"
