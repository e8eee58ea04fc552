// Test program: renders a fixed set of results through the report writers
// and prints every file body.  Built twice by tests/test_report_formats.py:
// against this repo's include/vqeforge_b200/report.hpp (default) and, when
// /root/reference is present, against the reference's own
// vqeforge/report.hpp (-DUSE_REFERENCE_REPORT); the two outputs must be
// byte-identical (acceptance_main.cpp:280-307 compares pes.csv bytes).
#include <cmath>
#include <iostream>
#include <limits>
#include <string>
#include <vector>

#ifdef USE_REFERENCE_REPORT
#include "vqeforge/report.hpp"
#else
#include "vqeforge_b200/report.hpp"
#endif

using namespace vqeforge;

int main() {
  SweepReport rep;
  const double nan = std::numeric_limits<double>::quiet_NaN();
  const double bonds[4] = {0.1, 0.74444444444444435, 1.6, 3.0};
  const double es[4] = {2.7099611466632689, -1.1372294545471588, -0.93162910279126354, nan};
  for (int i = 0; i < 4; ++i) {
    SweepPoint p;
    p.bond_angstrom = bonds[i];
    p.energy_hartree = es[i];
    if (i < 3) p.theta_star = {-0.2273881119456275 * (i + 1), 1e-300};
    p.iterations = i == 3 ? 0 : 200 - 7 * i;
    p.wall_seconds = 1.25e-5 * (i + 1);
    p.ok = i != 3;
    if (i == 3) p.error = "bond length 3 outside \"range\"";
    rep.points.push_back(p);
  }
  rep.per_worker_seconds = {0.00123, 4.5e-7};
  rep.total_wall_seconds = 0.0056789012345678;
  rep.all_ok = false;

  std::vector<BenchRow> rows(2);
  rows[0].workers = 1;
  rows[0].total_seconds = 0.12;
  rows[1].workers = 8;
  rows[1].total_seconds = 0.068;
  rows[1].speedup_vs_w1 = 0.12 / 0.068;
  rows[1].efficiency = 0.12 / 0.068 / 8;
  rows[1].amdahl_speedup = 1.0 / (0.3 + 0.7 / 8);

  std::vector<ScalingRecord> recs(2);
  recs[0].n_qubits = 4;
  recs[0].state_bytes = 256;
  recs[0].runtime_seconds = 6.1e-5;
  recs[0].final_energy = -3.9999999999876;
  recs[0].iterations_run = 150;
  recs[1].n_qubits = 26;
  recs[1].state_bytes = std::uint64_t{1} << 30;
  recs[1].runtime_seconds = 0.126;
  recs[1].final_energy = -31.123456789012345;
  recs[1].iterations_run = 5;

  RunManifest m;
  m.command = "pes";
  m.config = nlohmann::json{{"d_min", 0.1}, {"workers", 8}, {"name", "x"}};
  m.host = "box";
  m.started_at = "2026-01-01T00:00:00Z";
  m.finished_at = "2026-01-01T00:00:01Z";

  std::cout << "--pes.csv\n" << pes_csv(rep) << "--bench.csv\n" << bench_csv(rows) << "--scaling.csv\n"
            << scaling_csv(recs) << "--pes.json\n" << pes_json(m, rep).dump(2) << "\n--bench.json\n"
            << bench_json(m, rows).dump(2) << "\n--scaling.json\n" << scaling_json(m, recs).dump(2)
            << "\n--parse\n";
  for (const auto& row : parse_csv(pes_csv(rep))) {
    for (const auto& f : row) std::cout << '[' << f << ']';
    std::cout << '\n';
  }
  std::cout << "--format_sig " << format_sig(1.0 / 3.0) << ' ' << format_sig(1e-300) << ' ' << format_sig(2.5, 3)
            << '\n';
  return 0;
}
