// CPU check of the shared-memory engine's host compilation
// (compile_block_program, csrc/vqe_block.cu): the frame-tracked rotation
// passes and the transformed Hamiltonian are replayed on the host exactly as
// k_vqe_block walks them, and the energy is compared with a direct
// application of the hardware-efficient ansatz (vqe.hpp:81-93, the
// reference's apply_gate arithmetic) and the reference expectation formula
// (statevector.hpp:217-249) on seeded random Pauli sums.
// Usage: block_frame_check  -> prints "ok <cases>" or exits non-zero.
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "vqe_block.cuh"

using cplx = std::complex<double>;

namespace {

uint32_t insert_zeros(uint32_t k, const uint32_t* piv, int r) {
  for (int j = 0; j < r; ++j) {
    const uint32_t lo = k & ((1u << piv[j]) - 1u);
    k = ((k ^ lo) << 1) | lo;
  }
  return k;
}

double engine_energy(const vqf::BlockProgram& pr, const std::vector<double>& theta) {
  const uint32_t D = 1u << pr.n;
  const int R = static_cast<int>(pr.R);
  std::vector<cplx> psi(D, 0.0);
  psi[pr.init_index] = 1.0;
  for (const auto& bp : pr.passes) {
    for (uint32_t b = 0; b < (D >> R); ++b) {
      const uint32_t base = insert_zeros(b, bp.piv, R);
      std::vector<uint32_t> idx(1u << R);
      std::vector<cplx> x(1u << R);
      for (int m = 0; m < (1 << R); ++m) {
        uint32_t o = base;
        for (int j = 0; j < R; ++j)
          if ((m >> j) & 1) o ^= bp.vec[j];
        idx[m] = o;
        x[m] = psi[o];
      }
      for (int j = 0; j < R; ++j) {
        if (bp.param[j] < 0) continue;
        const double c = std::cos(0.5 * theta[bp.param[j]]), s0 = std::sin(0.5 * theta[bp.param[j]]);
        // one orientation per coset, from the base (as k_vqe_block)
        const bool one = ((__builtin_popcount(bp.row[j] & base) ^ (bp.cbits >> j)) & 1u) != 0u;
        const double s = one ? -s0 : s0;
        for (int m = 0; m < (1 << R); ++m) {
          if ((m >> j) & 1) continue;
          // the slot holding logical 0 must be the m_j = 0 member
          if ((((__builtin_popcount(bp.row[j] & idx[m]) ^ (bp.cbits >> j)) & 1u) != 0u) != one) {
            std::printf("FAIL: coset orientation differs from its base\n");
            std::exit(1);
          }
          if (vqf::block_slot(idx[m]) != (vqf::block_slot(base) ^ [&] {
                uint32_t o = 0;
                for (int i = 0; i < R; ++i)
                  if ((m >> i) & 1) o ^= bp.svec[i];
                return o;
              }())) {
            std::printf("FAIL: slot map not linear\n");
            std::exit(1);
          }
          const cplx t0 = x[m], t1 = x[m | (1 << j)];
          x[m] = c * t0 - s * t1;
          x[m | (1 << j)] = s * t0 + c * t1;
        }
      }
      for (int m = 0; m < (1 << R); ++m) psi[idx[m]] = x[m];
    }
  }
  cplx acc = 0.0;
  for (uint32_t t = pr.group_off[0]; t < pr.group_off[1]; ++t)
    for (uint32_t i = 0; i < D; ++i) {
      const double p = std::norm(psi[i]);
      const cplx cb(pr.terms[t].cb_re, pr.terms[t].cb_im);
      acc += ((__builtin_popcount(pr.terms[t].yz & i) & 1) ? -p : p) * cb;
    }
  for (size_t g = 1; g < pr.group_flip.size(); ++g) {
    const uint32_t F = pr.group_flip[g];
    for (uint32_t t = pr.group_off[g]; t < pr.group_off[g + 1]; ++t)
      for (uint32_t i = 0; i < D; ++i) {
        const cplx v = std::conj(psi[i]) * psi[i ^ F];
        const cplx cb(pr.terms[t].cb_re, pr.terms[t].cb_im);
        acc += ((__builtin_popcount(pr.terms[t].yz & i) & 1) ? -v : v) * cb;
      }
  }
  if (pr.herm) {  // the real form must give the same value
    double re = 0.0;
    for (uint32_t t = pr.group_off[0]; t < pr.group_off[1]; ++t)
      for (uint32_t i = 0; i < D; ++i)
        re += ((__builtin_popcount(pr.rterms[t].yz & i) & 1) ? -1.0 : 1.0) * pr.rterms[t].a * std::norm(psi[i]);
    for (size_t g = 1; g < pr.group_flip.size(); ++g) {
      const uint32_t F = pr.group_flip[g];
      const uint32_t pv = 31u - static_cast<uint32_t>(__builtin_clz(F));
      for (uint32_t i = 0; i < D; ++i) {
        if ((i >> pv) & 1u) continue;
        const cplx v = std::conj(psi[i]) * psi[i ^ F];
        for (uint32_t t = pr.group_off[g]; t < pr.group_off[g + 1]; ++t) {
          const double w = pr.rterms[t].odd ? 2.0 * v.imag() : 2.0 * v.real();
          re += ((__builtin_popcount(pr.rterms[t].yz & i) & 1) ? -1.0 : 1.0) * pr.rterms[t].a * w;
        }
      }
    }
    if (!(std::abs(re - acc.real()) < 1e-12)) {
      std::printf("FAIL: real form %.17g vs complex %.17g\n", re, acc.real());
      std::exit(1);
    }
  }
  if (std::abs(acc.imag()) > 1e-10) std::printf("imag residue %g\n", acc.imag());
  return acc.real();
}

double direct_energy(uint32_t n, uint32_t layers, const std::vector<double>& theta,
                     const std::vector<vqf::MaskTerm>& terms) {
  const uint32_t D = 1u << n;
  std::vector<cplx> psi(D, 0.0);
  psi[0] = 1.0;
  auto bit = [&](uint32_t q) { return 1u << (n - 1 - q); };
  size_t k = 0;
  for (uint32_t l = 0; l < layers; ++l) {
    for (uint32_t q = 0; q < n; ++q) {
      const double c = std::cos(0.5 * theta[k]), s = std::sin(0.5 * theta[k]);
      ++k;
      const uint32_t m = bit(q);
      for (uint32_t i = 0; i < D; ++i)
        if (!(i & m)) {
          const cplx a0 = psi[i], a1 = psi[i | m];
          psi[i] = c * a0 - s * a1;
          psi[i | m] = s * a0 + c * a1;
        }
    }
    for (uint32_t q = 0; q + 1 < n; ++q) {
      const uint32_t cm = bit(q), tm = bit(q + 1);
      for (uint32_t i = 0; i < D; ++i)
        if ((i & cm) && !(i & tm)) std::swap(psi[i], psi[i | tm]);
    }
  }
  cplx total = 0.0;
  for (const auto& t : terms) {
    cplx acc = 0.0;
    for (uint32_t i = 0; i < D; ++i) {
      const cplx v = std::conj(psi[i]) * psi[i ^ static_cast<uint32_t>(t.flip)];
      acc += (__builtin_popcountll(i & t.yz) & 1) ? -v : v;
    }
    total += cplx(t.cb_re, t.cb_im) * acc;
  }
  return total.real();
}

}  // namespace

int main() {
  std::mt19937 rng(20260804);
  int cases = 0, herm_cases = 0;
  for (uint32_t n : {4u, 5u, 6u, 7u, 9u, 12u, 13u, 14u, 15u}) {
    for (uint32_t layers : {1u, 2u, 3u}) {
      // random Pauli sum: 12 strings, X/Y/Z/I per wire, real coefficients
      std::vector<double> coeffs;
      std::vector<uint32_t> offs{0}, qs;
      std::vector<uint8_t> ax;
      std::uniform_int_distribution<int> pick(0, 3);
      std::uniform_real_distribution<double> cd(-1.0, 1.0);
      const int T = 12;
      for (int t = 0; t < T; ++t) {
        coeffs.push_back(cd(rng));
        coeffs.push_back(0.0);
        for (uint32_t q = 0; q < n; ++q) {
          const int a = pick(rng);
          if (a == 0) continue;
          qs.push_back(q);
          ax.push_back(static_cast<uint8_t>(a));  // VQF_AXIS_X / _Y / _Z
        }
        offs.push_back(static_cast<uint32_t>(qs.size()));
      }
      vqf_hamiltonian h{n, static_cast<uint32_t>(T), coeffs.data(), offs.data(), qs.data(), ax.data()};
      const vqf::CompiledHam ch = vqf::compile_hamiltonian(&h);
      herm_cases += 1;
      for (int32_t dtype : {VQF_F64, VQF_F32}) {
        if (n > static_cast<uint32_t>(vqf::block_max_n(dtype))) continue;
        const vqf::BlockProgram pr = vqf::compile_block_program(VQF_ANSATZ_HARDWARE_EFFICIENT, layers, n, ch, dtype);
        if (!pr.herm) {
          std::printf("FAIL: real-coefficient sum not in real form\n");
          return 1;
        }
        for (int rep = 0; rep < 2; ++rep) {
          std::vector<double> theta(layers * n);
          for (double& x : theta) x = 3.0 * cd(rng);
          const double e1 = engine_energy(pr, theta), e0 = direct_energy(n, layers, theta, ch.terms);
          if (!(std::abs(e1 - e0) < 1e-12)) {
            std::printf("FAIL n=%u layers=%u: engine %.17g direct %.17g\n", n, layers, e1, e0);
            return 1;
          }
          ++cases;
        }
      }
    }
  }
  // a complex coefficient keeps the general (complex) path
  {
    std::vector<double> coeffs{1.0, 0.0, 0.0, 0.5};
    std::vector<uint32_t> offs{0, 1, 2}, qs{0, 3};
    std::vector<uint8_t> ax{VQF_AXIS_X, VQF_AXIS_Z};
    vqf_hamiltonian h{6, 2, coeffs.data(), offs.data(), qs.data(), ax.data()};
    const vqf::BlockProgram pr =
        vqf::compile_block_program(VQF_ANSATZ_HARDWARE_EFFICIENT, 2, 6, vqf::compile_hamiltonian(&h), VQF_F64);
    if (pr.herm) {
      std::printf("FAIL: complex coefficient took the real form\n");
      return 1;
    }
  }
  std::printf("ok %d (%d Hamiltonians)\n", cases, herm_cases);
  return 0;
}
