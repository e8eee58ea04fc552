// Host entry points for the H2 Hamiltonian (chem.hpp:280-482 semantics)
// built on the shared chem.cuh core.  The fused PES kernel runs the same
// core on the device; this path serves the drop-in build_h2_hamiltonian /
// run_hartree_fock API and the tests.
#include <algorithm>
#include <array>
#include <mutex>
#include <string>

#include "chem.cuh"
#include "chem_host.h"
#include "common.cuh"
#include "pauli_host.h"

namespace vqf {
namespace chem {

const ChemConsts& consts() {
  static const ChemConsts k = make_consts();
  return k;
}

void check_bond(double d) {
  if (!(d >= kMinBond && d <= kMaxBond))
    throw Error(VQF_DOMAIN_ERROR, "bond length " + fstr(d) + " angstrom outside [" + fstr(kMinBond) + ", " +
                                      fstr(kMaxBond) + "]");
}

std::string nonconvergence_msg(double d) {
  return "SCF failed to converge within " + std::to_string(kScfMax) + " iterations at bond length " + fstr(d) +
         " angstrom";
}

std::string nonhermitian_msg(double imag) { return "non-Hermitian Pauli coefficient: imag = " + fstr(imag); }

// Contribution -> Pauli-string map of the Jordan-Wigner expansion: bond
// independent, so built once on the host (jw_meta over every contribution
// slot) and shipped to each device once.
const JwTable& jw_table() {
  static const JwTable t = [] {
    JwTable j{};
    std::array<std::vector<int>, 256> lists;
    for (int idx = 0; idx < kNumContrib; ++idx) {
      int key, m, slot;
      double scale;
      jw_meta(idx, key, m, slot, scale);
      lists[key].push_back(idx);
    }
    std::vector<int> keys;
    for (int k = 0; k < 256; ++k)
      if (!lists[k].empty()) keys.push_back(k);
    std::sort(keys.begin(), keys.end(), [](int a, int b) { return key_order(a) < key_order(b); });
    j.n_keys = static_cast<int>(keys.size());
    int e = 0;
    for (int t = 0; t < j.n_keys; ++t) {
      j.keys[t] = keys[t];
      j.start[t] = e;
      for (int idx : lists[keys[t]]) {
        int key, m, slot;
        double scale;
        jw_meta(idx, key, m, slot, scale);
        j.slot[e] = slot;
        j.coef[e] = (m == 2 || m == 3) ? -scale : scale;
        j.part[e] = (m & 1);
        ++e;
      }
    }
    j.start[j.n_keys] = e;
    return j;
  }();
  return t;
}

const JwTable* jw_table_device(int device) {
  static std::mutex mu;
  static std::vector<std::pair<int, JwTable*>> cache;
  std::lock_guard<std::mutex> lock(mu);
  for (auto& [d, ptr] : cache)
    if (d == device) return ptr;
  JwTable* ptr = nullptr;
  VQF_CUDA(cudaSetDevice(device));
  VQF_CUDA(cudaMalloc(&ptr, sizeof(JwTable)));
  VQF_CUDA(cudaMemcpy(ptr, &jw_table(), sizeof(JwTable), cudaMemcpyHostToDevice));
  cache.emplace_back(device, ptr);
  return ptr;
}

HfOut hartree_fock(double bond_angstrom, double C[2][2]) {
  check_bond(bond_angstrom);
  const ChemConsts& k = consts();
  const double d = bond_angstrom * kAngstromToBohr;
  AoInts I;
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j) one_electron(k, d, i, j, I);
  for (int ijkl = 0; ijkl < 16; ++ijkl) {
    double sum = 0.0;
    for (int r = 0; r < 81; ++r) sum += eri_term(k, d, ijkl * 81 + r);
    I.eri[ijkl] = sum;
  }
  HfOut o;
  scf(I, d, o, C);
  if (!o.converged) throw_runtime(nonconvergence_msg(bond_angstrom));
  double mo[16];
  for (int idx = 0; idx < 16; ++idx) mo[idx] = mo_chem(C, I.eri, idx);
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j)
      for (int kk = 0; kk < 2; ++kk)
        for (int l = 0; l < 2; ++l) o.eri_mo[((i * 2 + j) * 2 + kk) * 2 + l] = mo[((i * 2 + kk) * 2 + j) * 2 + l];
  return o;
}

std::vector<host::Term> build_h2(double bond_angstrom) {
  double C[2][2];
  const HfOut o = hartree_fock(bond_angstrom, C);
  std::array<double, 256> re{}, im{};
  std::array<int, 256> seen{};
  std::vector<int> order;
  for (int idx = 0; idx < kNumContrib; ++idx) {
    int key;
    double r, i;
    if (!jw_contribution(idx, o.hmo, o.eri_mo, o.e_nuc, key, r, i)) continue;
    if (!seen[key]) {
      seen[key] = 1;
      order.push_back(key);
      re[key] = r;
      im[key] = i;
    } else {
      re[key] += r;
      im[key] += i;
    }
  }
  std::vector<host::Term> ts;
  for (int key : order) {
    host::Term t;
    t.coeff = {re[key], im[key]};
    for (int q = 0; q < 4; ++q) {
      const int a = axis_of((key >> q) & 1, (key >> (4 + q)) & 1);
      if (a) t.axes.emplace_back(static_cast<uint32_t>(q), static_cast<uint8_t>(a));
    }
    ts.push_back(std::move(t));
  }
  host::canonicalize(ts);  // keys are already unique: drop + sort only
  for (auto& t : ts) {
    if (std::abs(t.coeff.imag()) >= 1e-10) throw_runtime(nonhermitian_msg(t.coeff.imag()));
    t.coeff = {t.coeff.real(), 0.0};
  }
  return ts;
}

}  // namespace chem
}  // namespace vqf

using namespace vqf;

extern "C" {

int vqf_build_h2_hamiltonian(double bond_angstrom, vqf_hamiltonian_out* out) {
  return guarded([&] { host::terms_to_csr(chem::build_h2(bond_angstrom), out); });
}

int vqf_hartree_fock(double bond_angstrom, double* out4) {
  return guarded([&] {
    double C[2][2];
    const chem::HfOut o = chem::hartree_fock(bond_angstrom, C);
    out4[0] = o.hf_energy;
    out4[1] = o.e_elec;
    out4[2] = o.e_nuc;
    out4[3] = o.scf_iterations;
  });
}

}  // extern "C"
