// coconet-ccopt — the reference's command-line front end (tools/ccopt.cpp) with
// a CUDA backend. Same subcommands, options, JSON reports and
// exit codes (0 ok / 1 check failed or deviation > tol / 2 error,
// tools/ccopt.cpp:252-273), hand-parsed (the reference uses CLI11, absent here):
//
//   check | transform | oracle | diff   the reference's DSL functions, unchanged
//   run   [--backend cuda|sim]         cuda (default): GpuEngine on B200, the
//                                      cmd_run flow (:184-193) with device_ms and
//                                      the lowering added to the report;
//                                      sim: the reference Engine
//   tune  [--backend cuda|sim]         cuda: coconet::gpu_tune (candidates ranked
//                                      by measured device time); sim: ccopt::tune
//
// CUDA-only options: --device D, --math exact|fast, --reps R (tune; run: R fresh engines,
// device_ms = median after the first), --no-fused.
// Tensor files (the reference's write_tensor_file / read_tensor_file format,
// json_io.hpp:580-608: little-endian f32 + JSON sidecar), run only:
//   --input NAME=BASE   decl NAME's global tensor from BASE.{bin,json} instead
//                       of gen_decl_values (sliced decls take their slice)
//   --dump DIR          every result array as DIR/<key>_r<rank>.{bin,json}
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <iostream>
#include <string>
#include <vector>

#include "ccopt/autotune.hpp"
#include "ccopt/diff.hpp"
#include "ccopt/json_io.hpp"
#include "ccopt/oracle.hpp"
#include "ccopt/runtime.hpp"
#include "ccopt/transform.hpp"
#include "coconet/gpu_engine.hpp"
#include "coconet/gpu_tune.hpp"

using namespace ccopt;

namespace {

struct Opts {
  std::string cmd, program_path, schedule_path, out_path, other_path;
  std::vector<std::string> sizes;
  std::vector<std::string> inputs;  // NAME=BASE
  std::string dump_dir;
  int ranks = 4, channels = 2;
  std::string protocol = "simple";
  double alpha = 0.5, beta = 2000.0, gamma = 2000.0, lambda = 0.5;
  bool alpha_set = false, beta_set = false;
  int64_t tile = 1 << 16;
  uint64_t seed = 1;
  double tol = 1e-5;
  bool threaded = false, wall_time = false;
  // CUDA backend
  std::string backend = "cuda";
  int device = 0, reps = 3;
  int math = COCONET_MATH_EXACT;
  bool fused = true;
};

[[noreturn]] void usage(const std::string& why) {
  std::cerr << "error: " << why << "\n"
            << "usage: coconet-ccopt {check|transform|run|oracle|tune|diff} PROGRAM.json [OTHER.json]\n"
               "  [--schedule S.json] [--ranks W] [--size NAME=VALUE]... [--seed N] [--tol T] [--out F]\n"
               "  [--channels C] [--protocol ll|simple] [--alpha A] [--beta B] [--gamma G] [--lambda L]\n"
               "  [--tile T] [--threaded] [--wall-time]\n"
               "  [--backend cuda|sim] [--device D] [--math exact|fast] [--reps R] [--no-fused]\n"
               "  [--input NAME=BASE]... [--dump DIR]\n";
  std::exit(2);
}

Opts parse(int argc, char** argv) {
  Opts o;
  if (argc < 2) usage("missing subcommand");
  o.cmd = argv[1];
  std::vector<std::string> pos;
  for (int i = 2; i < argc; ++i) {
    std::string a = argv[i];
    auto val = [&]() -> std::string {
      if (i + 1 >= argc) usage(a + " needs a value");
      return argv[++i];
    };
    if (a == "--schedule") o.schedule_path = val();
    else if (a == "--ranks") o.ranks = std::stoi(val());
    else if (a == "--size") o.sizes.push_back(val());
    else if (a == "--channels") o.channels = std::stoi(val());
    else if (a == "--protocol") {
      o.protocol = val();
      if (o.protocol != "ll" && o.protocol != "simple") usage("--protocol must be ll or simple");
    } else if (a == "--alpha") o.alpha = std::stod(val()), o.alpha_set = true;
    else if (a == "--beta") o.beta = std::stod(val()), o.beta_set = true;
    else if (a == "--gamma") o.gamma = std::stod(val());
    else if (a == "--lambda") o.lambda = std::stod(val());
    else if (a == "--tile") o.tile = std::stoll(val());
    else if (a == "--seed") o.seed = std::stoull(val());
    else if (a == "--out") o.out_path = val();
    else if (a == "--tol") o.tol = std::stod(val());
    else if (a == "--threaded") o.threaded = true;
    else if (a == "--wall-time") o.wall_time = true;
    else if (a == "--backend") {
      o.backend = val();
      if (o.backend != "cuda" && o.backend != "sim") usage("--backend must be cuda or sim");
    } else if (a == "--device") o.device = std::stoi(val());
    else if (a == "--reps") o.reps = std::stoi(val());
    else if (a == "--math") {
      std::string m = val();
      if (m == "exact") o.math = COCONET_MATH_EXACT;
      else if (m == "fast") o.math = COCONET_MATH_FAST;
      else usage("--math must be exact or fast");
    } else if (a == "--no-fused") o.fused = false;
    else if (a == "--input") o.inputs.push_back(val());
    else if (a == "--dump") o.dump_dir = val();
    else if (!a.empty() && a[0] == '-') usage("unknown option " + a);
    else pos.push_back(a);
  }
  if (pos.empty()) usage("missing program file");
  o.program_path = pos[0];
  if (o.cmd == "diff") {
    if (pos.size() < 2) usage("diff needs a second program");
    o.other_path = pos[1];
  } else if (pos.size() > 1) {
    usage("unexpected argument " + pos[1]);
  }
  return o;
}

// size_symbols / comm_config / load_program: tools/ccopt.cpp:61-104
std::map<std::string, int64_t> size_symbols(const Opts& o) {
  std::map<std::string, int64_t> syms{{"B", 2}, {"S", 8}, {"H", 64}, {"N", 1024}};
  for (auto& s : o.sizes) {
    auto eq = s.find('=');
    if (eq == std::string::npos) throw Error(ErrCode::ParseError, "--size expects NAME=VALUE, got '" + s + "'");
    syms[s.substr(0, eq)] = std::stoll(s.substr(eq + 1));
  }
  syms["W"] = o.ranks;
  return syms;
}

CommConfig comm_config(const Opts& o) {
  CommConfig cfg;
  cfg.channels = o.channels;
  cfg.buffer_tile_elems = o.tile;
  cfg.alpha = o.alpha;
  cfg.beta = o.beta;
  cfg.gamma = o.gamma;
  cfg.lambda = o.lambda;
  cfg.mode = o.threaded ? ExecMode::Threaded : ExecMode::RoundRobin;
  if (o.protocol == "ll") {
    cfg.protocol = Protocol::LowLatency;
    if (!o.alpha_set) cfg.alpha = o.alpha / 4;
    if (!o.beta_set) cfg.beta = o.beta / 2;
  }
  return cfg;
}

Program load_program(const Opts& o, const std::string& path) {
  Program p = program_from_json(load_json_file(path), size_symbols(o));
  auto diags = validate_program(p);
  if (!diags.empty()) {
    std::string msg = "invalid program:";
    for (auto& d : diags) msg += "\n  " + d;
    throw Error(ErrCode::InvalidInput, msg);
  }
  return p;
}

Program transformed(const Opts& o, const std::string& path, Provenance* prov = nullptr) {
  Program p = load_program(o, path);
  if (!o.schedule_path.empty())
    p = apply_schedule(std::move(p), schedule_from_json(load_json_file(o.schedule_path)), prov);
  return p;
}

void emit(const Opts& o, const Json& j) {
  if (o.out_path.empty()) std::cout << j.dump(2) << "\n";
  else save_json_file(o.out_path, j);
}

std::string hex(uint64_t h) {
  char buf[32];
  std::snprintf(buf, sizeof buf, "%016llx", (unsigned long long)h);
  return buf;
}

Json results_summary(const std::map<std::string, Collected>& res) {
  Json j = Json::object();
  for (auto& [key, c] : res) {
    Json e;
    e["shape"] = c.shape;
    e["per_rank"] = c.per_rank;
    uint64_t h = 0xcbf29ce484222325ull;
    for (auto& arr : c.data) h = fnv1a(arr.data(), arr.size() * sizeof(float), h);
    e["digest"] = hex(h);
    j[key] = e;
  }
  return j;
}

Json run_report_json(const Opts& o, const RunReport& rep, double deviation) {
  Json j;
  j["simulated_time"] = rep.simulated_time;
  if (o.wall_time) j["wall_time"] = rep.wall_time;
  j["kernel_steps"] = rep.kernel_steps;
  j["comm_bytes"] = rep.comm_bytes;
  j["intergroup_bytes"] = rep.intergroup_bytes;
  j["traffic_saved_bytes"] = rep.traffic_saved_bytes;
  j["memory_elems"] = rep.memory_elems;
  j["digest"] = hex(rep.digest);
  j["deviation"] = deviation;
  j["results"] = results_summary(rep.results);
  return j;
}

coconet::GpuOptions gpu_options(const Opts& o) {
  coconet::GpuOptions g;
  g.device = o.device;
  g.math = o.math;
  g.fused_kernels = o.fused;
  return g;
}

int cmd_check(const Opts& o) {
  Program p = program_from_json(load_json_file(o.program_path), size_symbols(o));
  auto diags = validate_program(p);
  Json j;
  j["name"] = p.name;
  j["world_size"] = p.world_size();
  j["diagnostics"] = diags;
  j["nodes"] = Json::array();
  for (auto& n : p.nodes) {
    Json nj;
    nj["id"] = n.id;
    nj["kind"] = op_kind_name(n.kind);
    nj["shape"] = n.out_shape;
    nj["layout"] = n.out_layout.str();
    nj["group"] = n.group;
    j["nodes"].push_back(nj);
  }
  emit(o, j);
  return diags.empty() ? 0 : 1;
}

int cmd_transform(const Opts& o) {
  Provenance prov;
  Program p = transformed(o, o.program_path, &prov);
  Json j;
  j["program"] = program_to_json(p);
  j["provenance"] = Json::array();
  for (auto& [from, to] : prov) j["provenance"].push_back({{"from", from}, {"to", to}});
  emit(o, j);
  return 0;
}

// gen_decl_values with --input overrides: each rank's storage of decl NAME
// takes the file's global tensor through its DistView (state.hpp:17-50).
ValueMap decl_values(const Opts& o, const Program& p) {
  ValueMap vals = gen_decl_values(p, o.seed);
  for (auto& spec : o.inputs) {
    const auto eq = spec.find('=');
    if (eq == std::string::npos) throw Error(ErrCode::ParseError, "--input expects NAME=BASE, got '" + spec + "'");
    const std::string name = spec.substr(0, eq), base = spec.substr(eq + 1);
    auto it = vals.find(name);
    if (it == vals.end()) throw Error(ErrCode::UnknownId, "--input: no decl '" + name + "'");
    Shape shape;
    std::vector<float> data = read_tensor_file(base, nullptr, &shape);
    TensorVal& t = it->second;
    if (shape != t.view.global) throw Error(ErrCode::ShapeMismatch, "--input " + name + ": shape differs from the decl");
    for (size_t r = 0; r < t.per_rank.size(); ++r)
      for (int64_t li = 0; li < t.view.local_elems(); ++li)
        t.per_rank[r][size_t(li)] = t.view.layout.is_sliced() ? data[size_t(t.view.to_global(int(r), li))]
                                                              : data[size_t(li)];
  }
  return vals;
}

void dump_results(const Opts& o, const std::map<std::string, Collected>& res) {
  if (o.dump_dir.empty()) return;
  for (auto& [key, c] : res)
    for (size_t r = 0; r < c.data.size(); ++r) {
      std::string stem = key;
      for (auto& ch : stem)
        if (ch == ':' || ch == '/') ch = '_';
      const Shape shape = int64_t(c.data[r].size()) == num_elems(c.shape) ? c.shape : Shape{int64_t(c.data[r].size())};
      write_tensor_file(o.dump_dir + "/" + stem + "_r" + std::to_string(r), key, shape, Elem::F32, c.data[r]);
    }
}

int cmd_run(const Opts& o) {
  Program base = load_program(o, o.program_path);
  Program p = transformed(o, o.program_path);
  auto oracle_ref = oracle_results(base, decl_values(o, base), o.seed);
  Json j;
  double dev = 0;
  if (o.backend == "cuda") {
    // --reps R runs the program R times on fresh engines: the report is the
    // first run's; device_ms is the median of the later runs (the first one
    // also pays the lazy loading of its kernels), device_ms_first the first
    std::vector<double> ms;
    RunReport rep;
    std::vector<std::string> lowering;
    for (int i = 0; i < std::max(1, o.reps); ++i) {
      coconet::GpuEngine eng(p, comm_config(o), o.seed, gpu_options(o));
      RunReport r = eng.run(decl_values(o, p));
      ms.push_back(eng.device_ms());
      if (i == 0) {
        rep = std::move(r);
        lowering = eng.lowering();
      } else if (r.digest != rep.digest) {
        throw Error(ErrCode::InvalidInput, "run " + std::to_string(i) + " differs from run 0");
      }
    }
    dev = compare_results(oracle_ref, rep.results);
    dump_results(o, rep.results);
    j = run_report_json(o, rep, dev);
    j["backend"] = "cuda";
    std::vector<double> warm(ms.begin() + (ms.size() > 1 ? 1 : 0), ms.end());
    std::sort(warm.begin(), warm.end());
    j["device_ms"] = warm[warm.size() / 2];
    j["device_ms_first"] = ms[0];
    j["runs"] = int(ms.size());
    j["lowering"] = lowering;
    j["math"] = o.math == COCONET_MATH_EXACT ? "exact" : "fast";
  } else {
    Engine eng(p, comm_config(o), o.seed);
    RunReport rep = eng.run(decl_values(o, p));
    dev = compare_results(oracle_ref, rep.results);
    dump_results(o, rep.results);
    j = run_report_json(o, rep, dev);
    j["backend"] = "sim";
  }
  emit(o, j);
  return dev > o.tol ? 1 : 0;
}

int cmd_oracle(const Opts& o) {
  Program p = load_program(o, o.program_path);
  auto res = oracle_results(p, gen_decl_values(p, o.seed), o.seed);
  Json j;
  j["results"] = results_summary(res);
  j["digest"] = hex(digest_results(res));
  emit(o, j);
  return 0;
}

int cmd_tune(const Opts& o) {
  Program p = load_program(o, o.program_path);
  TuneConfig cfg;
  cfg.comm = comm_config(o);
  cfg.seed = o.seed;
  cfg.tol = o.tol;
  if (o.backend == "cuda") {
    Json j = coconet::gpu_tune_report_to_json(coconet::gpu_tune(p, cfg, gpu_options(o), o.reps));
    j["backend"] = "cuda";
    emit(o, j);
  } else {
    Json j = tune_report_to_json(tune(p, cfg));
    j["backend"] = "sim";
    emit(o, j);
  }
  return 0;
}

int cmd_diff(const Opts& o) {
  Program a = load_program(o, o.program_path);
  Program b = transformed(o, o.other_path);
  auto entries = diff_programs(a, b);
  emit(o, diff_to_json(entries));
  return entries.empty() ? 0 : 1;
}

}  // namespace

int main(int argc, char** argv) {
  Opts o = parse(argc, argv);
  try {
    if (o.cmd == "check") return cmd_check(o);
    if (o.cmd == "transform") return cmd_transform(o);
    if (o.cmd == "run") return cmd_run(o);
    if (o.cmd == "oracle") return cmd_oracle(o);
    if (o.cmd == "tune") return cmd_tune(o);
    if (o.cmd == "diff") return cmd_diff(o);
  } catch (const Error& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  }
  usage("unknown subcommand " + o.cmd);
}
