// Host-side Pauli algebra and driver arithmetic shared by the C ABI and
// the sweep / VQE drivers.  Semantics follow the reference:
//   canonicalize          pauli.hpp:180-201
//   bond_grid             sweep.hpp:68-85
//   split_chunks          sweep.hpp:93-107
//   adam_step             vqe.hpp:152-174
//   build_tfim/z_sum      sweep.hpp:209-235
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <utility>
#include <vector>

#include "common.cuh"

namespace vqf {
namespace host {

struct Term {
  std::complex<double> coeff;
  std::vector<std::pair<uint32_t, uint8_t>> axes;  // sorted by qubit
};

inline bool axes_less(const Term& a, const Term& b) {
  return std::lexicographical_compare(a.axes.begin(), a.axes.end(), b.axes.begin(), b.axes.end(),
                                      [](const auto& x, const auto& y) {
                                        if (x.first != y.first) return x.first < y.first;
                                        return x.second < y.second;
                                      });
}

// Merge like terms in order of first appearance, drop |c| < 1e-12, sort.
inline void canonicalize(std::vector<Term>& ts) {
  std::vector<Term> merged;
  merged.reserve(ts.size());
  for (auto& t : ts) {
    auto it = std::find_if(merged.begin(), merged.end(), [&](const Term& m) { return m.axes == t.axes; });
    if (it == merged.end())
      merged.push_back(std::move(t));
    else
      it->coeff += t.coeff;
  }
  std::vector<Term> kept;
  for (auto& t : merged)
    if (std::abs(t.coeff) >= 1e-12) kept.push_back(std::move(t));
  std::sort(kept.begin(), kept.end(), axes_less);
  ts = std::move(kept);
}

inline std::vector<Term> terms_from_csr(const vqf_hamiltonian* h, bool validate) {
  if (h == nullptr) throw_invalid("null hamiltonian");
  std::vector<Term> ts(h->n_terms);
  for (uint32_t t = 0; t < h->n_terms; ++t) {
    ts[t].coeff = {h->coeffs[2 * t], h->coeffs[2 * t + 1]};
    for (uint32_t k = h->offsets[t]; k < h->offsets[t + 1]; ++k) ts[t].axes.emplace_back(h->qubits[k], h->axes[k]);
    if (validate) {  // PauliTerm ctor, pauli.hpp:73-88
      std::sort(ts[t].axes.begin(), ts[t].axes.end(),
                [](const auto& a, const auto& b) { return a.first < b.first; });
      for (size_t i = 0; i < ts[t].axes.size(); ++i) {
        if (ts[t].axes[i].second == 0) throw_invalid("explicit identity entry in PauliTerm");
        if (i > 0 && ts[t].axes[i].first == ts[t].axes[i - 1].first)
          throw_invalid("duplicate qubit index in PauliTerm");
      }
      if (!std::isfinite(ts[t].coeff.real()) || !std::isfinite(ts[t].coeff.imag()))
        throw_invalid("non-finite PauliTerm coefficient");
      if (!ts[t].axes.empty() && ts[t].axes.back().first >= h->n_qubits)
        throw_invalid("PauliTerm index exceeds register size");
    }
  }
  return ts;
}

inline void terms_to_csr(const std::vector<Term>& ts, vqf_hamiltonian_out* o) {
  if (o == nullptr) throw_invalid("null hamiltonian_out");
  if (ts.size() > o->cap_terms) throw_invalid("hamiltonian_out: term capacity exceeded");
  uint32_t k = 0;
  o->offsets[0] = 0;
  for (size_t t = 0; t < ts.size(); ++t) {
    o->coeffs[2 * t] = ts[t].coeff.real();
    o->coeffs[2 * t + 1] = ts[t].coeff.imag();
    for (const auto& [q, a] : ts[t].axes) {
      if (k >= o->cap_axes) throw_invalid("hamiltonian_out: axis capacity exceeded");
      o->qubits[k] = q;
      o->axes[k] = a;
      ++k;
    }
    o->offsets[t + 1] = k;
  }
  o->n_terms = static_cast<uint32_t>(ts.size());
}

inline std::vector<Term> build_tfim(uint32_t n, double coupling, double field) {
  std::vector<Term> ts;
  for (uint32_t q = 0; q + 1 < n; ++q) ts.push_back({{-coupling, 0.0}, {{q, 3}, {q + 1, 3}}});
  for (uint32_t q = 0; q < n; ++q) ts.push_back({{-field, 0.0}, {{q, 1}}});
  canonicalize(ts);
  return ts;
}

inline std::vector<Term> build_z_sum(uint32_t n) {
  std::vector<Term> ts;
  for (uint32_t q = 0; q < n; ++q) ts.push_back({{1.0, 0.0}, {{q, 3}}});
  canonicalize(ts);
  return ts;
}

inline void bond_grid(double d_min, double d_max, int32_t n_points, double* out) {
  if (n_points == 1) {
    out[0] = d_min;
    return;
  }
  const double span = d_max - d_min;
  for (int i = 0; i < n_points - 1; ++i)
    out[i] = d_min + span * static_cast<double>(i) / static_cast<double>(n_points - 1);
  out[n_points - 1] = d_max;
}

inline void split_chunks(uint64_t n_items, uint64_t n_chunks, uint64_t* be) {
  const uint64_t base = n_items / n_chunks, extra = n_items % n_chunks;
  uint64_t begin = 0;
  for (uint64_t c = 0; c < n_chunks; ++c) {
    const uint64_t len = base + (c < extra ? 1 : 0);
    be[2 * c] = begin;
    be[2 * c + 1] = begin + len;
    begin += len;
  }
}

// Reciprocal bias-correction factors 1 / (1 - beta^t), t = 1..T, with
// 1 - beta^t computed by the host libm pow exactly as adam_step does
// (vqe.hpp:161-162).  The device multiplies by them instead of dividing
// (one IEEE division less on the per-iteration critical path); m_hat and
// v_hat then differ from the reference's quotients by at most 1 ulp.
inline void bias_tables(const vqf_adam_config& c, int32_t T, std::vector<double>& bc1, std::vector<double>& bc2) {
  bc1.resize(std::max(T, 1));
  bc2.resize(std::max(T, 1));
  for (int32_t t = 1; t <= T; ++t) {
    bc1[t - 1] = 1.0 / (1.0 - std::pow(c.beta1, static_cast<double>(t)));
    bc2[t - 1] = 1.0 / (1.0 - std::pow(c.beta2, static_cast<double>(t)));
  }
}

inline void adam_step(const double* m, const double* v, int64_t step, const double* grad, const double* theta,
                      uint32_t n, const vqf_adam_config& c, double* theta_out, double* m_out, double* v_out,
                      int64_t* step_out) {
  const int64_t t = step + 1;
  const double bc1 = 1.0 - std::pow(c.beta1, static_cast<double>(t));
  const double bc2 = 1.0 - std::pow(c.beta2, static_cast<double>(t));
  for (uint32_t k = 0; k < n; ++k) {
    const double mk = c.beta1 * m[k] + (1.0 - c.beta1) * grad[k];
    const double vk = c.beta2 * v[k] + (1.0 - c.beta2) * grad[k] * grad[k];
    const double m_hat = mk / bc1;
    const double v_hat = vk / bc2;
    theta_out[k] = theta[k] - c.learning_rate * m_hat / (std::sqrt(v_hat) + c.epsilon);
    m_out[k] = mk;
    v_out[k] = vk;
  }
  *step_out = t;
}

}  // namespace host
}  // namespace vqf
