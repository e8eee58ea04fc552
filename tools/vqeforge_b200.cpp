// vqeforge (B200 build): the reference CLI surface (tools/vqeforge.cpp:
// pes | bench | scaling | exact | dump-hamiltonian, --dump-hamiltonian,
// --version) over the B200 engine, same flags, outputs (pes.csv/json,
// bench.csv/json, scaling.csv/json) and exit codes: 0 ok, 1 failure,
// 2 usage / invalid input (vqeforge.cpp:366-394).  CLI11 is not available in
// this image, so flags are parsed by hand ("--flag value" and
// "--flag=value", as CLI11 accepts).  Additions: `scaling --gradient
// adjoint`.  `--workers` / `--worker-list` count GPU workers (one host
// thread + stream per worker, round-robin over visible devices).
//
// Attribution: the argument parser (Args) is new, but the command bodies
// (parse_int_list, write_outputs, run_pes, run_bench, run_scaling) follow the
// flow of the reference CLI, /root/reference/proj/tools/vqeforge.cpp:36-270
// (Copyright 2026 VQE Forge contributors, Apache License 2.0), because their
// stdout lines, output files and manifest keys must match the reference
// byte for byte.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <iostream>
#include <map>
#include <optional>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "vqeforge_b200/report.hpp"
#include "vqeforge_b200/vqeforge.hpp"

namespace {

using nlohmann::json;

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Minimal option table: value options and boolean flags of one subcommand.
class Args {
 public:
  Args(int argc, char** argv, int begin, std::set<std::string> values, std::set<std::string> flags)
      : values_(std::move(values)), flags_(std::move(flags)) {
    for (int i = begin; i < argc; ++i) {
      std::string a = argv[i];
      if (a.rfind("--", 0) != 0) throw UsageError("unexpected argument: " + a);
      std::string val;
      bool has_val = false;
      const auto eq = a.find('=');
      if (eq != std::string::npos) {
        val = a.substr(eq + 1);
        a = a.substr(0, eq);
        has_val = true;
      }
      if (flags_.count(a)) {
        if (has_val) throw UsageError(a + " takes no value");
        set_.insert(a);
        continue;
      }
      if (!values_.count(a)) throw UsageError("unknown option: " + a);
      if (!has_val) {
        if (i + 1 >= argc) throw UsageError(a + " requires a value");
        val = argv[++i];
      }
      got_[a] = val;
    }
  }
  bool flag(const std::string& f) const { return set_.count(f) > 0; }
  bool has(const std::string& o) const { return got_.count(o) > 0; }
  std::string str(const std::string& o, const std::string& dflt) const { return has(o) ? got_.at(o) : dflt; }
  double num(const std::string& o, double dflt) const {
    if (!has(o)) return dflt;
    const std::string& v = got_.at(o);
    std::size_t pos = 0;
    double x = 0.0;
    try {
      x = std::stod(v, &pos);
    } catch (const std::exception&) {
      pos = 0;
    }
    if (pos != v.size()) throw UsageError(o + ": '" + v + "' is not a number");
    return x;
  }
  long integer(const std::string& o, long dflt) const {
    if (!has(o)) return dflt;
    const std::string& v = got_.at(o);
    std::size_t pos = 0;
    long x = 0;
    try {
      x = std::stol(v, &pos);
    } catch (const std::exception&) {
      pos = 0;
    }
    if (pos != v.size()) throw UsageError(o + ": '" + v + "' is not an integer");
    return x;
  }

 private:
  std::set<std::string> values_, flags_, set_;
  std::map<std::string, std::string> got_;
};

// vqeforge.cpp:36-55
std::vector<int> parse_int_list(const std::string& text, const std::string& flag) {
  std::vector<int> values;
  std::string item;
  std::istringstream in(text);
  while (std::getline(in, item, ',')) {
    std::size_t pos = 0;
    int v = 0;
    try {
      v = std::stoi(item, &pos);
    } catch (const std::exception&) {
      pos = 0;
    }
    if (pos != item.size() || v < 1) throw std::invalid_argument(flag + ": '" + item + "' is not a positive integer");
    values.push_back(v);
  }
  if (values.empty()) throw std::invalid_argument(flag + ": empty list");
  return values;
}

void write_outputs(const std::string& out_dir, const std::string& stem, const std::string& csv, const json& full) {
  namespace fs = std::filesystem;
  fs::create_directories(out_dir);
  const fs::path dir(out_dir);
  vqeforge::write_text_file((dir / (stem + ".csv")).string(), csv);
  vqeforge::write_text_file((dir / (stem + ".json")).string(), full.dump(2) + "\n");
}

int run_pes(const Args& a) {  // vqeforge.cpp:81-132
  const double d_min = a.num("--dmin", 0.1), d_max = a.num("--dmax", 3.0), lr = a.num("--lr", 0.01);
  const int points = static_cast<int>(a.integer("--points", 100));
  const int iterations = static_cast<int>(a.integer("--iterations", 200));
  const int workers_req = static_cast<int>(a.integer("--workers", 1));
  const std::string out_dir = a.str("--out-dir", ".");
  std::optional<double> tol;
  if (a.has("--tol")) tol = a.num("--tol", 0.0);
  vqeforge::SweepConfig config;
  config.d_min = d_min;
  config.d_max = d_max;
  config.n_points = points;
  config.workers = vqeforge::effective_workers(workers_req);
  config.adam.learning_rate = lr;
  config.adam.max_iterations = iterations;
  config.adam.gradient_tolerance = tol;

  vqeforge::RunManifest manifest;
  manifest.command = "pes";
  manifest.config = json{{"d_min", d_min},
                         {"d_max", d_max},
                         {"points", points},
                         {"iterations", iterations},
                         {"learning_rate", lr},
                         {"tolerance", tol ? json(*tol) : json(nullptr)},
                         {"workers_requested", workers_req},
                         {"workers", config.workers},
                         {"out_dir", out_dir}};
  manifest.started_at = vqeforge::iso8601_utc_now();
  const vqeforge::SweepReport report = vqeforge::run_sweep(config);
  manifest.finished_at = vqeforge::iso8601_utc_now();
  write_outputs(out_dir, "pes", vqeforge::pes_csv(report), vqeforge::pes_json(manifest, report));

  const vqeforge::SweepPoint* best = nullptr;
  int failures = 0;
  for (const auto& p : report.points) {
    if (!p.ok) {
      ++failures;
      continue;
    }
    if (best == nullptr || p.energy_hartree < best->energy_hartree) best = &p;
  }
  if (best != nullptr)
    std::printf(
        "equilibrium estimate: d = %.6f angstrom, E = %.6f hartree "
        "(grid argmin over %zu points, %d workers, %.3f s)\n",
        best->bond_angstrom, best->energy_hartree, report.points.size(), config.workers, report.total_wall_seconds);
  if (failures > 0) {
    std::cerr << failures << " of " << report.points.size() << " sweep points failed; see pes.json for details\n";
    return 1;
  }
  return 0;
}

int run_bench(const Args& a) {  // vqeforge.cpp:146-216
  const bool paper_hpc = a.flag("--paper-hpc");
  const int iterations = paper_hpc ? 300 : static_cast<int>(a.integer("--iterations", 200));
  const double d_min = a.num("--dmin", 0.1), d_max = a.num("--dmax", 3.0), lr = a.num("--lr", 0.01);
  const double serial_fraction = a.num("--serial-fraction", 0.05);
  const int points = static_cast<int>(a.integer("--points", 100));
  const std::string out_dir = a.str("--out-dir", ".");
  const std::vector<int> requested = parse_int_list(a.str("--worker-list", "1,2,4,8"), "--worker-list");
  std::vector<int> workers;
  if (std::find(requested.begin(), requested.end(), 1) == requested.end()) workers.push_back(1);
  for (int w : requested) {
    const int eff = vqeforge::effective_workers(w);
    if (std::find(workers.begin(), workers.end(), eff) == workers.end()) workers.push_back(eff);
  }
  vqeforge::RunManifest manifest;
  manifest.command = "bench";
  manifest.config = json{{"worker_list_requested", requested},
                         {"worker_list", workers},
                         {"d_min", d_min},
                         {"d_max", d_max},
                         {"points", points},
                         {"iterations", iterations},
                         {"learning_rate", lr},
                         {"serial_fraction", serial_fraction},
                         {"paper_hpc", paper_hpc},
                         {"out_dir", out_dir}};
  manifest.started_at = vqeforge::iso8601_utc_now();
  bool all_ok = true;
  double t1 = 0.0;
  std::vector<vqeforge::BenchRow> rows;
  for (int w : workers) {
    vqeforge::SweepConfig config;
    config.d_min = d_min;
    config.d_max = d_max;
    config.n_points = points;
    config.workers = w;
    config.adam.learning_rate = lr;
    config.adam.max_iterations = iterations;
    const vqeforge::SweepReport report = vqeforge::run_sweep(config);
    all_ok = all_ok && report.all_ok;
    if (w == 1) t1 = report.total_wall_seconds;
    vqeforge::BenchRow row;
    row.workers = w;
    row.total_seconds = report.total_wall_seconds;
    row.speedup_vs_w1 = vqeforge::measured_speedup(t1, report.total_wall_seconds);
    row.efficiency = vqeforge::parallel_efficiency(t1, report.total_wall_seconds, w);
    row.amdahl_speedup = vqeforge::amdahl_speedup(serial_fraction, w);
    rows.push_back(row);
    std::printf("workers=%d total=%.3fs speedup=%.2f efficiency=%.2f\n", w, row.total_seconds, row.speedup_vs_w1,
                row.efficiency);
  }
  manifest.finished_at = vqeforge::iso8601_utc_now();
  for (std::size_t i = 1; i < rows.size(); ++i)
    if (rows[i].speedup_vs_w1 < rows[i - 1].speedup_vs_w1)
      std::cerr << "warning: speedup not monotone between workers=" << rows[i - 1].workers
                << " and workers=" << rows[i].workers << "\n";
  write_outputs(out_dir, "bench", vqeforge::bench_csv(rows), vqeforge::bench_json(manifest, rows));
  return all_ok ? 0 : 1;
}

int run_scaling(const Args& a) {  // vqeforge.cpp:231-270
  vqeforge::ScalingConfig config;
  config.qubits.clear();
  for (int n : parse_int_list(a.str("--qubits", "4,8,12,14,16,18,20"), "--qubits"))
    config.qubits.push_back(static_cast<std::uint32_t>(n));
  config.layers = static_cast<std::uint32_t>(a.integer("--layers", 2));
  config.iterations = static_cast<int>(a.integer("--iterations", 5));
  config.learning_rate = a.num("--lr", 0.05);
  config.coupling = a.num("--coupling", 1.0);
  config.field = a.num("--field", 1.0);
  config.z_sum_mode = a.flag("--z-sum");
  config.theta_init = a.num("--theta-init", 0.1);
  config.force = a.flag("--force");
  const std::string grad = a.str("--gradient", "shift");
  if (grad != "shift" && grad != "adjoint") throw std::invalid_argument("--gradient: expected shift or adjoint");
  config.adjoint = grad == "adjoint";
  const std::string out_dir = a.str("--out-dir", ".");
  vqeforge::RunManifest manifest;
  manifest.command = "scaling";
  manifest.config = json{{"qubits", config.qubits},         {"layers", config.layers},
                         {"iterations", config.iterations}, {"learning_rate", config.learning_rate},
                         {"coupling", config.coupling},     {"field", config.field},
                         {"z_sum", config.z_sum_mode},      {"theta_init", config.theta_init},
                         {"force", config.force},           {"out_dir", out_dir}};
  manifest.started_at = vqeforge::iso8601_utc_now();
  const auto records = vqeforge::run_scaling_study(config);
  manifest.finished_at = vqeforge::iso8601_utc_now();
  for (const auto& r : records)
    std::printf("n_qubits=%u state_bytes=%llu runtime=%.3fs energy=%.6f\n", r.n_qubits,
                static_cast<unsigned long long>(r.state_bytes), r.runtime_seconds, r.final_energy);
  write_outputs(out_dir, "scaling", vqeforge::scaling_csv(records), vqeforge::scaling_json(manifest, records));
  return 0;
}

double bond_arg(const Args& a) {
  if (!a.has("--bond")) throw UsageError("--bond is required");
  return a.num("--bond", 0.0);
}

int usage(std::ostream& os) {
  os << "vqeforge: variational ground-state solver for minimal-basis H2 with parallel bond-length sweeps and\n"
        "register-scaling studies (B200 engine)\n"
        "usage: vqeforge [--version] [--dump-hamiltonian BOND] <pes|bench|scaling|exact|dump-hamiltonian> [options]\n";
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc < 2) {
      usage(std::cerr);
      return 2;
    }
    const std::string first = argv[1];
    if (first == "--help" || first == "-h") return usage(std::cout);
    if (first == "--version") {
      std::printf("%s\n", vqeforge::kVersion);
      return 0;
    }
    if (first.rfind("--dump-hamiltonian", 0) == 0) {
      const Args a(argc, argv, 1, {"--dump-hamiltonian"}, {});
      std::fputs(vqeforge::to_text(vqeforge::build_h2_hamiltonian(a.num("--dump-hamiltonian", 0.0))).c_str(), stdout);
      return 0;
    }
    if (first == "pes")
      return run_pes(Args(argc, argv, 2, {"--dmin", "--dmax", "--points", "--iterations", "--lr", "--tol", "--workers",
                                          "--out-dir"}, {}));
    if (first == "bench")
      return run_bench(Args(argc, argv, 2, {"--worker-list", "--dmin", "--dmax", "--points", "--iterations", "--lr",
                                            "--serial-fraction", "--out-dir"}, {"--paper-hpc"}));
    if (first == "scaling")
      return run_scaling(Args(argc, argv, 2, {"--qubits", "--layers", "--iterations", "--lr", "--coupling", "--field",
                                              "--theta-init", "--out-dir", "--gradient"}, {"--z-sum", "--force"}));
    if (first == "exact") {
      const Args a(argc, argv, 2, {"--bond"}, {});
      std::printf("%.6f\n", vqeforge::exact_ground_energy(vqeforge::build_h2_hamiltonian(bond_arg(a))));
      return 0;
    }
    if (first == "dump-hamiltonian") {
      const Args a(argc, argv, 2, {"--bond"}, {});
      std::fputs(vqeforge::to_text(vqeforge::build_h2_hamiltonian(bond_arg(a))).c_str(), stdout);
      return 0;
    }
    std::cerr << "unknown subcommand: " << first << "\n";
    usage(std::cerr);
    return 2;
  } catch (const UsageError& e) {
    std::cerr << e.what() << "\n";
    return 2;
  } catch (const vqeforge::BondLengthOutOfRange& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  } catch (const std::invalid_argument& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
