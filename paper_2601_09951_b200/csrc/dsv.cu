// Distributed state vector (BASELINE config 5: 34-35 qubits over 8 B200),
// behind the C ABI vqf_dsv_* (include/vqf_b200.h).
//
// world = 2^g shards of 2^(n-g) amplitudes.  Qubits sit at positions:
// 0..g-1 global (rank bit g-1-p), g..n-1 local (local index bit n-1-p =
// engine wire p-g of the shard).  The layout starts as the identity and is
// updated lazily (never swapped back):
//
//  * plan_circuit: a gate touching global qubits first swaps each of them
//    with a local position not used by the gate, evicting the qubit whose
//    next use in the circuit lies furthest ahead (Belady; ties go to the top
//    local bit, whose half-shard is one contiguous block); maximal runs of
//    local gates become one LOCAL op (fused tile passes per shard).
//  * plan_expectation: terms without X/Y on global positions are evaluated
//    per shard (a Z on a global position is the rank's sign); the largest
//    group of terms sharing a global flip set F is made local by swapping F
//    with local positions on which every term of the group acts as I or Z,
//    and the loop repeats on the new layout; terms that flip global qubits
//    and leave no I/Z local position are evaluated across shard pairs
//    (CROSS).  The shard totals are summed in rank order (virtual ranks) or
//    all-reduced (processes), then the imaginary-residue check of
//    statevector.hpp:244-247 applies to the total.
//
// Execution: a SWAP exchanges, on every rank r, the half of its shard whose
// local bit b differs from r's bit for the global position with the same
// half of rank r ^ mask.  Virtual ranks swap the two halves in place on the
// device; processes stream them through comm->sendrecv in chunk_bytes
// pieces via two preallocated device buffers (pack / send+receive / unpack;
// the half is read straight from the shard when its runs are at least a
// chunk long).  CROSS terms on processes fetch the partner shard chunk by
// chunk (chunk bits = top local bits; the chunk index is flipped by the
// terms' local flips on those bits), so no rank ever holds a second shard.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <limits>
#include <memory>
#include <string>
#include <vector>

#include "sv.cuh"

struct vqf_dsv_state {
  uint32_t n = 0, g = 0, nl = 0, world = 1;
  int32_t dtype = VQF_F64, device = 0;
  std::vector<uint32_t> pos, at;  // qubit -> position, position -> qubit
  bool virt = true;
  vqf_dsv_comm comm{};
  std::vector<uint32_t> ranks;      // shards held here
  std::vector<vqf_sv> shards;       // same order
  uint64_t chunk_bytes = 0;
  void* buf[2] = {nullptr, nullptr};  // exchange staging (processes)
  double* part = nullptr;             // cross-chunk partials (device)
  double* part_host = nullptr;
  uint64_t swaps = 0, bytes_sent = 0;
};

namespace vqf {
namespace {

constexpr uint64_t kDefaultChunk = 256ull << 20;
constexpr int kThreadsD = 256;

template <typename T>
struct V2D;
template <>
struct V2D<double> {
  using type = double2;
};
template <>
struct V2D<float> {
  using type = float2;
};

struct Layout {
  uint32_t n, g;
  std::vector<uint32_t>& pos;
  std::vector<uint32_t>& at;
  bool global(uint32_t p) const { return p < g; }
  uint32_t rank_bit(uint32_t p) const { return g - 1 - p; }    // global position -> rank bit
  uint32_t local_bit(uint32_t p) const { return n - 1 - p; }   // local position -> local index bit
  void swap(uint32_t pg, uint32_t pl) {
    const uint32_t a = at[pg], b = at[pl];
    at[pg] = b;
    at[pl] = a;
    pos[a] = pl;
    pos[b] = pg;
  }
};

void check_layout(uint32_t n, uint32_t world, const uint32_t* pos, uint32_t& g) {
  if (world == 0 || (world & (world - 1)) != 0) throw_invalid("distributed state: world size must be a power of two");
  g = static_cast<uint32_t>(__builtin_ctz(world));
  if (n < g + 5) throw_invalid("distributed state: need at least 5 local qubits per shard");
  if (n > 48) throw_invalid("distributed state: at most 48 qubits");
  std::vector<char> seen(n, 0);
  for (uint32_t q = 0; q < n; ++q) {
    if (pos[q] >= n || seen[pos[q]]) throw_invalid("distributed state: layout is not a permutation");
    seen[pos[q]] = 1;
  }
}

// ------------------------------------------------------------ planners
void plan_circuit(Layout& L, const vqf_gate* gates, uint32_t ng, std::vector<vqf_dsv_op>& ops,
                  std::vector<vqf_gate>& mapped) {
  // dependency order: gates sharing a wire keep their order; among ready
  // gates the earliest one whose wires are all local runs first (commuting
  // gates on disjoint wires may move ahead: rounding-level reordering, as
  // the tile scheduler does), else the earliest ready gate swaps its global
  // wires in
  std::vector<std::vector<uint32_t>> preds(ng);
  std::vector<int64_t> last(L.n, -1);
  for (uint32_t i = 0; i < ng; ++i)
    for (uint32_t w = 0; w < gates[i].n_wires; ++w) {
      const uint32_t q = gates[i].wires[w];
      if (last[q] >= 0) preds[i].push_back(static_cast<uint32_t>(last[q]));
      last[q] = i;
    }
  std::vector<char> done(ng, 0);
  // next use of qubit q among gates not yet placed (Belady eviction)
  std::vector<std::vector<uint32_t>> uses(L.n);
  for (uint32_t i = 0; i < ng; ++i)
    for (uint32_t w = 0; w < gates[i].n_wires; ++w) uses[gates[i].wires[w]].push_back(i);
  const auto next_use = [&](uint32_t q) -> uint64_t {
    for (uint32_t i : uses[q])
      if (!done[i]) return i;
    return std::numeric_limits<uint64_t>::max();
  };
  const auto is_ready = [&](uint32_t i) {
    for (uint32_t p : preds[i])
      if (!done[p]) return false;
    return true;
  };
  const auto all_local = [&](uint32_t i) {
    for (uint32_t w = 0; w < gates[i].n_wires; ++w)
      if (L.global(L.pos[gates[i].wires[w]])) return false;
    return true;
  };
  mapped.clear();
  uint32_t run_first = 0;
  const auto flush = [&] {
    if (mapped.size() > run_first)
      ops.push_back(vqf_dsv_op{VQF_DSV_LOCAL, 0, 0, run_first, static_cast<uint32_t>(mapped.size()) - run_first});
    run_first = static_cast<uint32_t>(mapped.size());
  };
  uint32_t placed = 0, lo = 0;
  while (placed < ng) {
    while (lo < ng && done[lo]) ++lo;
    int64_t pick = -1;
    for (uint32_t i = lo; i < ng; ++i)
      if (!done[i] && is_ready(i) && all_local(i)) {
        pick = i;
        break;
      }
    if (pick < 0) {
      for (uint32_t i = lo; i < ng && pick < 0; ++i)
        if (!done[i] && is_ready(i)) pick = i;
      const vqf_gate& gt = gates[pick];
      done[pick] = 1;  // its own use does not count as a future use
      for (uint32_t w = 0; w < gt.n_wires; ++w) {
        const uint32_t q = gt.wires[w];
        if (!L.global(L.pos[q])) continue;
        // victim: a local position whose qubit is not in this gate, used
        // furthest ahead; ties to the top local bit (lowest position)
        uint32_t best = UINT32_MAX;
        uint64_t best_use = 0;
        for (uint32_t p = L.g; p < L.n; ++p) {
          const uint32_t v = L.at[p];
          bool in_gate = false;
          for (uint32_t k = 0; k < gt.n_wires; ++k) in_gate = in_gate || gt.wires[k] == v;
          if (in_gate) continue;
          const uint64_t u = next_use(v);
          if (best == UINT32_MAX || u > best_use) {
            best = p;
            best_use = u;
          }
        }
        if (best == UINT32_MAX) throw_invalid("distributed state: no free local position for a swap");
        flush();
        ops.push_back(vqf_dsv_op{VQF_DSV_SWAP, L.pos[q], best, 0, 0});
        L.swap(L.pos[q], best);
      }
    }
    const vqf_gate& gt = gates[pick];
    done[pick] = 1;
    vqf_gate m = gt;
    for (uint32_t w = 0; w < gt.n_wires; ++w) m.wires[w] = L.pos[gt.wires[w]] - L.g;
    mapped.push_back(m);
    ++placed;
  }
  flush();
}

struct TermAxes {
  std::vector<std::pair<uint32_t, uint8_t>> axes;  // (qubit, axis)
};

vqf_dsv_term plan_term(const Layout& L, uint32_t t, const TermAxes& ta) {
  vqf_dsv_term o{};
  o.term = t;
  for (const auto& [q, a] : ta.axes) {
    const uint32_t p = L.pos[q];
    if (L.global(p)) {
      const uint32_t bit = 1u << L.rank_bit(p);
      if (a == VQF_AXIS_X || a == VQF_AXIS_Y) o.g_flip |= bit;
      if (a == VQF_AXIS_Y || a == VQF_AXIS_Z) o.g_yz |= bit;
      if (a == VQF_AXIS_Y) ++o.g_ny;
    } else {
      const uint64_t bit = uint64_t{1} << L.local_bit(p);
      if (a == VQF_AXIS_X || a == VQF_AXIS_Y) o.l_flip |= bit;
      if (a == VQF_AXIS_Y || a == VQF_AXIS_Z) o.l_yz |= bit;
      if (a == VQF_AXIS_Y) ++o.l_ny;
    }
  }
  return o;
}

// I or Z on position p for every term of `ts`
bool iz_on(const Layout& L, const std::vector<TermAxes>& terms, const std::vector<uint32_t>& ts, uint32_t p) {
  const uint32_t q = L.at[p];
  for (uint32_t t : ts)
    for (const auto& [qq, a] : terms[t].axes)
      if (qq == q && (a == VQF_AXIS_X || a == VQF_AXIS_Y)) return false;
  return true;
}

void plan_expectation(Layout& L, const std::vector<TermAxes>& terms, std::vector<vqf_dsv_op>& ops,
                      std::vector<vqf_dsv_term>& out) {
  std::vector<uint32_t> rest(terms.size());
  for (uint32_t t = 0; t < rest.size(); ++t) rest[t] = t;
  const auto gflip = [&](uint32_t t) {
    uint32_t f = 0;
    for (const auto& [q, a] : terms[t].axes)
      if (L.global(L.pos[q]) && (a == VQF_AXIS_X || a == VQF_AXIS_Y)) f |= 1u << L.pos[q];  // position mask
    return f;
  };
  while (!rest.empty()) {
    // 1. every term with no global flip, under the current layout
    std::vector<uint32_t> later;
    const uint32_t first = static_cast<uint32_t>(out.size());
    for (uint32_t t : rest) {
      if (gflip(t) == 0) out.push_back(plan_term(L, t, terms[t]));
      else later.push_back(t);
    }
    if (out.size() > first)
      ops.push_back(vqf_dsv_op{VQF_DSV_EVAL, 0, 0, first, static_cast<uint32_t>(out.size()) - first});
    rest.swap(later);
    if (rest.empty()) break;
    // 2. the most common global flip set
    std::vector<std::pair<uint32_t, uint32_t>> count;  // (flip, terms)
    for (uint32_t t : rest) {
      const uint32_t f = gflip(t);
      auto it = std::find_if(count.begin(), count.end(), [&](const auto& e) { return e.first == f; });
      if (it == count.end()) count.emplace_back(f, 1);
      else ++it->second;
    }
    const uint32_t F = std::max_element(count.begin(), count.end(), [](const auto& a, const auto& b) {
                         return a.second < b.second;
                       })->first;
    std::vector<uint32_t> fpos;
    for (uint32_t p = 0; p < L.g; ++p)
      if ((F >> p) & 1u) fpos.push_back(p);
    // 3. greedy subgroup keeping >= |F| local I/Z positions (top bits first)
    std::vector<uint32_t> cand;
    for (uint32_t p = L.g; p < L.n; ++p) cand.push_back(p);
    std::vector<uint32_t> sub, keep;
    for (uint32_t t : rest) {
      if (gflip(t) != F) {
        keep.push_back(t);
        continue;
      }
      std::vector<uint32_t> c2;
      for (uint32_t p : cand)
        if (iz_on(L, terms, {t}, p)) c2.push_back(p);
      if (c2.size() >= fpos.size()) {
        cand.swap(c2);
        sub.push_back(t);
      } else {
        keep.push_back(t);
      }
    }
    if (sub.empty()) {
      // flips F and X/Y on (nearly) every local qubit: cross-shard pairs
      const uint32_t cf = static_cast<uint32_t>(out.size());
      std::vector<uint32_t> keep2;
      for (uint32_t t : rest) {
        if (gflip(t) == F) out.push_back(plan_term(L, t, terms[t]));
        else keep2.push_back(t);
      }
      uint32_t mask = 0;
      for (uint32_t p : fpos) mask |= 1u << L.rank_bit(p);
      ops.push_back(vqf_dsv_op{VQF_DSV_CROSS, mask, 0, cf, static_cast<uint32_t>(out.size()) - cf});
      rest.swap(keep2);
      continue;
    }
    for (size_t k = 0; k < fpos.size(); ++k) {
      ops.push_back(vqf_dsv_op{VQF_DSV_SWAP, fpos[k], cand[k], 0, 0});
      L.swap(fpos[k], cand[k]);
    }
    // sub now has no global flips; the loop evaluates it (and re-classifies the rest)
    rest.clear();
    rest.insert(rest.end(), sub.begin(), sub.end());
    rest.insert(rest.end(), keep.begin(), keep.end());
  }
}

std::vector<TermAxes> term_axes(const vqf_hamiltonian* h) {
  if (h == nullptr) throw_invalid("null hamiltonian");
  std::vector<TermAxes> out(h->n_terms);
  for (uint32_t t = 0; t < h->n_terms; ++t)
    for (uint32_t k = h->offsets[t]; k < h->offsets[t + 1]; ++k) {
      if (h->qubits[k] >= h->n_qubits) throw_invalid("PauliTerm index exceeds register size");
      out[t].axes.emplace_back(h->qubits[k], h->axes[k]);
    }
  return out;
}

// coefficient of a planned term on rank r (see vqf_dsv_term)
std::complex<double> term_coeff(const vqf_hamiltonian* h, const vqf_dsv_term& pt, uint32_t r) {
  std::complex<double> c(h->coeffs[2 * pt.term], h->coeffs[2 * pt.term + 1]);
  static const std::complex<double> mi[4] = {{1, 0}, {0, -1}, {-1, 0}, {0, 1}};  // (-i)^k
  c *= mi[(pt.l_ny + pt.g_ny) & 3u];
  if (__builtin_popcount(r & pt.g_yz) & 1) c = -c;
  return c;
}

CompiledHam shard_terms(const vqf_hamiltonian* h, const vqf_dsv_term* pts, uint32_t count, uint32_t nl, uint32_t r) {
  CompiledHam c;
  c.n_qubits = nl;
  std::vector<MaskTerm> raw;
  for (uint32_t k = 0; k < count; ++k) {
    const auto cb = term_coeff(h, pts[k], r);
    raw.push_back(MaskTerm{pts[k].l_flip, pts[k].l_yz, cb.real(), cb.imag()});
  }
  c.group_flip.push_back(0);
  for (const auto& m : raw)
    if (m.flip != 0 && std::find(c.group_flip.begin(), c.group_flip.end(), m.flip) == c.group_flip.end())
      c.group_flip.push_back(m.flip);
  c.group_offset.push_back(0);
  for (uint64_t f : c.group_flip) {
    for (const auto& m : raw)
      if (m.flip == f) c.terms.push_back(m);
    c.group_offset.push_back(static_cast<uint32_t>(c.terms.size()));
  }
  return c;
}

// ------------------------------------------------------------- kernels
__device__ __forceinline__ uint64_t put_bit(uint64_t k, uint32_t b, uint32_t v) {
  const uint64_t low = k & ((uint64_t{1} << b) - 1);
  return ((k >> b) << (b + 1)) | (uint64_t(v) << b) | low;
}

// swap x[half(b, vx)] <-> y[half(b, vy)] element by element (virtual ranks)
template <typename A>
__global__ void k_swap_halves(A* __restrict__ x, A* __restrict__ y, uint32_t b, uint32_t vx, uint32_t vy,
                              uint64_t half) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < half; k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = put_bit(k, b, vx), j = put_bit(k, b, vy);
    const A t = x[i];
    x[i] = y[j];
    y[j] = t;
  }
}

// buf[k - k0] = x[half(b, v)[k]] for k in [k0, k0 + count) (and back)
template <typename A, bool PACK>
__global__ void k_pack_half(A* __restrict__ x, A* __restrict__ buf, uint32_t b, uint32_t v, uint64_t k0,
                            uint64_t count) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < count; k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = put_bit(k0 + k, b, v);
    if (PACK) buf[k] = x[i];
    else x[i] = buf[k];
  }
}

// partial sums of sum_l conj(a[l]) cb_t (-1)^popc((base + l) & yz_t) b[l ^ flip_t]
// over a chunk (flip_t restricted to the chunk's bits); one complex partial
// per block, summed in block order on the host
template <typename A>
__global__ void k_cross_chunk(const A* __restrict__ a, const A* __restrict__ b, uint64_t len, uint64_t base,
                              const MaskTerm* __restrict__ terms, uint32_t nt, double* __restrict__ part) {
  double re = 0.0, im = 0.0;
  for (uint64_t l = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; l < len; l += (uint64_t)gridDim.x * blockDim.x) {
    const A x = a[l];
    for (uint32_t t = 0; t < nt; ++t) {
      const MaskTerm m = terms[t];
      const A y = b[l ^ m.flip];
      // conj(x) * y
      const double vr = (double)x.x * y.x + (double)x.y * y.y, vi = (double)x.x * y.y - (double)x.y * y.x;
      const double s = (__popcll((base + l) & m.yz) & 1) ? -1.0 : 1.0;
      re += s * (m.cb_re * vr - m.cb_im * vi);
      im += s * (m.cb_re * vi + m.cb_im * vr);
    }
  }
  __shared__ double sr[kThreadsD], si[kThreadsD];
  sr[threadIdx.x] = re;
  si[threadIdx.x] = im;
  __syncthreads();
  for (int o = kThreadsD / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      sr[threadIdx.x] += sr[threadIdx.x + o];
      si[threadIdx.x] += si[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = sr[0];
    part[2 * blockIdx.x + 1] = si[0];
  }
}

constexpr int kCrossBlocks = 296;

unsigned grid_of(uint64_t n) { return static_cast<unsigned>(std::min<uint64_t>((n + kThreadsD - 1) / kThreadsD, 148 * 16)); }

// ------------------------------------------------------------ executor
struct Exec {
  vqf_dsv_state* d;
  size_t amp() const { return d->dtype == VQF_F64 ? 16 : 8; }
  vqf_statevector* shard(uint32_t r) const {
    for (size_t i = 0; i < d->ranks.size(); ++i)
      if (d->ranks[i] == r) return d->shards[i];
    throw Error(VQF_LOGIC_ERROR, "distributed state: shard not held here");
  }
  cudaStream_t stream() const { return d->shards[0]->stream; }

  template <typename A>
  void swap_virtual(uint32_t pg, uint32_t pl) {
    const uint32_t rb = d->g - 1 - pg, b = d->n - 1 - pl;
    const uint64_t half = uint64_t{1} << (d->nl - 1);
    for (uint32_t r = 0; r < d->world; ++r) {
      const uint32_t p = r ^ (1u << rb);
      if (p < r) continue;
      const uint32_t vr = 1u - ((r >> rb) & 1u), vp = 1u - ((p >> rb) & 1u);
      k_swap_halves<A><<<grid_of(half), kThreadsD, 0, stream()>>>(static_cast<A*>(shard(r)->amps),
                                                                   static_cast<A*>(shard(p)->amps), b, vr, vp, half);
      VQF_LAUNCHED();
    }
    VQF_CUDA(cudaGetLastError());
    d->bytes_sent += static_cast<uint64_t>(d->world) * half * amp();
  }

  template <typename A>
  void swap_comm(uint32_t pg, uint32_t pl) {
    const uint32_t rb = d->g - 1 - pg, b = d->n - 1 - pl;
    const uint32_t r = d->comm.rank, peer = r ^ (1u << rb);
    const uint32_t v = 1u - ((r >> rb) & 1u);
    A* x = static_cast<A*>(shard(r)->amps);
    const uint64_t half = uint64_t{1} << (d->nl - 1);
    const uint64_t C = std::max<uint64_t>(1, d->chunk_bytes / sizeof(A));
    const uint64_t run = uint64_t{1} << b;  // contiguous run length of the half
    for (uint64_t k0 = 0; k0 < half; k0 += C) {
      const uint64_t cnt = std::min(C, half - k0);
      const void* send = nullptr;
      if (run >= cnt && (k0 % run) + cnt <= run) {
        send = x + put_bit_host(k0, b, v);  // one contiguous piece of the shard
      } else {
        k_pack_half<A, true><<<grid_of(cnt), kThreadsD, 0, stream()>>>(x, static_cast<A*>(d->buf[0]), b, v, k0, cnt);
        VQF_LAUNCHED();
        send = d->buf[0];
      }
      if (d->comm.sendrecv(d->comm.user, send, d->buf[1], cnt * sizeof(A), static_cast<int32_t>(peer), stream()) != 0)
        throw Error(VQF_RUNTIME_ERROR, "distributed state: sendrecv failed");
      k_pack_half<A, false><<<grid_of(cnt), kThreadsD, 0, stream()>>>(x, static_cast<A*>(d->buf[1]), b, v, k0, cnt);
      VQF_LAUNCHED();
      d->bytes_sent += cnt * sizeof(A);
    }
    VQF_CUDA(cudaGetLastError());
  }

  static uint64_t put_bit_host(uint64_t k, uint32_t b, uint32_t v) {
    const uint64_t low = k & ((uint64_t{1} << b) - 1);
    return ((k >> b) << (b + 1)) | (uint64_t(v) << b) | low;
  }

  void swap(uint32_t pg, uint32_t pl) {
    if (d->virt) {
      if (d->dtype == VQF_F64) swap_virtual<double2>(pg, pl);
      else swap_virtual<float2>(pg, pl);
    } else {
      if (d->dtype == VQF_F64) swap_comm<double2>(pg, pl);
      else swap_comm<float2>(pg, pl);
    }
    ++d->swaps;
    Layout L{d->n, d->g, d->pos, d->at};
    L.swap(pg, pl);
  }

  void local(const vqf_gate* gates, uint32_t count) {
    for (vqf_sv s : d->shards)
      if (vqf_apply_circuit(s, gates, count) != VQF_OK) throw Error(VQF_CUDA_ERROR, vqf_last_error());
  }

  std::complex<double> eval(const vqf_hamiltonian* h, const vqf_dsv_term* pts, uint32_t count) {
    std::complex<double> tot = 0.0;
    for (size_t i = 0; i < d->ranks.size(); ++i) {
      const CompiledHam c = shard_terms(h, pts, count, d->nl, d->ranks[i]);
      double out[2];
      sv_expectation(d->shards[i], c, out);
      tot += std::complex<double>(out[0], out[1]);
    }
    return tot;
  }

  template <typename A>
  std::complex<double> cross_chunks(const A* a, const A* b, uint64_t len, uint64_t base, const CompiledHam& c) {
    MaskTerm* td = nullptr;
    VQF_CUDA(cudaMallocAsync(&td, std::max<size_t>(1, c.terms.size()) * sizeof(MaskTerm), stream()));
    VQF_CUDA(cudaMemcpyAsync(td, c.terms.data(), c.terms.size() * sizeof(MaskTerm), cudaMemcpyHostToDevice, stream()));
    k_cross_chunk<A><<<kCrossBlocks, kThreadsD, 0, stream()>>>(a, b, len, base, td,
                                                               static_cast<uint32_t>(c.terms.size()), d->part);
    VQF_LAUNCHED();
    VQF_CUDA(cudaMemcpyAsync(d->part_host, d->part, 2 * kCrossBlocks * sizeof(double), cudaMemcpyDeviceToHost,
                             stream()));
    VQF_CUDA(cudaFreeAsync(td, stream()));
    VQF_CUDA(cudaStreamSynchronize(stream()));
    std::complex<double> s = 0.0;
    for (int k = 0; k < kCrossBlocks; ++k) s += std::complex<double>(d->part_host[2 * k], d->part_host[2 * k + 1]);
    return s;
  }

  template <typename A>
  std::complex<double> cross(const vqf_hamiltonian* h, uint32_t mask, const vqf_dsv_term* pts, uint32_t count) {
    std::complex<double> tot = 0.0;
    const uint64_t D = uint64_t{1} << d->nl;
    if (d->virt) {
      for (uint32_t r = 0; r < d->world; ++r) {
        const CompiledHam c = shard_terms(h, pts, count, d->nl, r);
        tot += cross_chunks<A>(static_cast<const A*>(shard(r)->amps), static_cast<const A*>(shard(r ^ mask)->amps), D,
                               0, c);
      }
      return tot;
    }
    // processes: chunk bits = the top local bits; a term's local flip on
    // them pairs chunk c with partner chunk c ^ fh (grouped by fh)
    const uint32_t r = d->comm.rank, peer = r ^ mask;
    uint64_t C = std::max<uint64_t>(1, d->chunk_bytes / sizeof(A));
    C = uint64_t{1} << (63 - __builtin_clzll(std::min<uint64_t>(C, D)));  // power of two <= shard
    const uint32_t cb = static_cast<uint32_t>(__builtin_ctzll(C));
    const uint64_t n_chunks = D / C, low = C - 1;
    std::vector<uint64_t> fhs;
    for (uint32_t k = 0; k < count; ++k) {
      const uint64_t fh = pts[k].l_flip >> cb;
      if (std::find(fhs.begin(), fhs.end(), fh) == fhs.end()) fhs.push_back(fh);
    }
    const A* x = static_cast<const A*>(shard(r)->amps);
    for (uint64_t fh : fhs) {
      std::vector<vqf_dsv_term> sub;
      for (uint32_t k = 0; k < count; ++k)
        if ((pts[k].l_flip >> cb) == fh) {
          vqf_dsv_term t = pts[k];
          t.l_flip &= low;
          sub.push_back(t);
        }
      const CompiledHam c0 = shard_terms(h, sub.data(), static_cast<uint32_t>(sub.size()), d->nl, r);
      for (uint64_t ch = 0; ch < n_chunks; ++ch) {
        const uint64_t pc = ch ^ fh;
        // both ranks run the same chunk loop: each sends its chunk pc, which
        // is exactly what the partner needs at this step
        if (d->comm.sendrecv(d->comm.user, x + pc * C, d->buf[1], C * sizeof(A), static_cast<int32_t>(peer),
                             stream()) != 0)
          throw Error(VQF_RUNTIME_ERROR, "distributed state: sendrecv failed");
        d->bytes_sent += C * sizeof(A);
        tot += cross_chunks<A>(x + ch * C, static_cast<const A*>(d->buf[1]), C, ch * C, c0);
      }
    }
    return tot;
  }
};

vqf_dsv_state* checked(vqf_dsv d) {
  if (d == nullptr) throw_invalid("null distributed state");
  return d;
}

}  // namespace
}  // namespace vqf

using namespace vqf;

extern "C" {

int vqf_dsv_plan_circuit(uint32_t n_qubits, uint32_t world, uint32_t* position_of_qubit, const vqf_gate* gates,
                         uint32_t n_gates, vqf_dsv_op* ops, uint32_t cap_ops, uint32_t* n_ops,
                         vqf_gate* mapped_gates) {
  return guarded([&] {
    if (position_of_qubit == nullptr || (n_gates && gates == nullptr) || n_ops == nullptr)
      throw_invalid("null argument");
    uint32_t g = 0;
    check_layout(n_qubits, world, position_of_qubit, g);
    vqf_statevector probe;
    probe.n_qubits = n_qubits;
    for (uint32_t i = 0; i < n_gates; ++i) sv_check_gate(&probe, gates[i]);
    std::vector<uint32_t> pos(position_of_qubit, position_of_qubit + n_qubits), at(n_qubits);
    for (uint32_t q = 0; q < n_qubits; ++q) at[pos[q]] = q;
    Layout L{n_qubits, g, pos, at};
    std::vector<vqf_dsv_op> o;
    std::vector<vqf_gate> m;
    plan_circuit(L, gates, n_gates, o, m);
    *n_ops = static_cast<uint32_t>(o.size());
    if (o.size() > cap_ops) throw_invalid("distributed plan: op capacity too small");
    if (ops) std::copy(o.begin(), o.end(), ops);
    if (mapped_gates) std::copy(m.begin(), m.end(), mapped_gates);
    std::copy(pos.begin(), pos.end(), position_of_qubit);
  });
}

int vqf_dsv_plan_expectation(uint32_t n_qubits, uint32_t world, uint32_t* position_of_qubit,
                             const vqf_hamiltonian* h, vqf_dsv_op* ops, uint32_t cap_ops, uint32_t* n_ops,
                             vqf_dsv_term* terms_out) {
  return guarded([&] {
    if (position_of_qubit == nullptr || n_ops == nullptr) throw_invalid("null argument");
    uint32_t g = 0;
    check_layout(n_qubits, world, position_of_qubit, g);
    if (h == nullptr || h->n_qubits != n_qubits) throw_invalid("expectation: qubit count mismatch");
    const auto ta = term_axes(h);
    std::vector<uint32_t> pos(position_of_qubit, position_of_qubit + n_qubits), at(n_qubits);
    for (uint32_t q = 0; q < n_qubits; ++q) at[pos[q]] = q;
    Layout L{n_qubits, g, pos, at};
    std::vector<vqf_dsv_op> o;
    std::vector<vqf_dsv_term> pts;
    plan_expectation(L, ta, o, pts);
    *n_ops = static_cast<uint32_t>(o.size());
    if (o.size() > cap_ops) throw_invalid("distributed plan: op capacity too small");
    if (ops) std::copy(o.begin(), o.end(), ops);
    if (terms_out) std::copy(pts.begin(), pts.end(), terms_out);
    std::copy(pos.begin(), pos.end(), position_of_qubit);
  });
}

uint64_t vqf_dsv_memory_per_gpu(uint32_t n_qubits, uint32_t world, int32_t dtype, uint64_t chunk_bytes,
                                int32_t one_shard_per_process) {
  if (world == 0 || (world & (world - 1)) != 0) return 0;
  const uint32_t g = static_cast<uint32_t>(__builtin_ctz(world));
  if (n_qubits <= g) return 0;
  const uint64_t shard = (uint64_t{1} << (n_qubits - g)) * (dtype == VQF_F32 ? 8u : 16u);
  if (!one_shard_per_process) return shard * world;  // virtual ranks: all shards on one device
  const uint64_t chunk = std::min<uint64_t>(chunk_bytes ? chunk_bytes : kDefaultChunk, shard);
  return shard + 2 * chunk;
}

int vqf_dsv_create(uint32_t n_qubits, uint32_t world, int32_t dtype, int32_t device, const vqf_dsv_comm* comm,
                   uint64_t chunk_bytes, vqf_dsv* out) {
  return guarded([&] {
    if (out == nullptr) throw_invalid("null output handle");
    if (dtype != VQF_F64 && dtype != VQF_F32) throw_invalid("distributed state: unknown dtype");
    std::vector<uint32_t> ident(n_qubits);
    for (uint32_t q = 0; q < n_qubits; ++q) ident[q] = q;
    uint32_t g = 0;
    check_layout(n_qubits, world, ident.data(), g);
    auto d = std::make_unique<vqf_dsv_state>();
    d->n = n_qubits;
    d->g = g;
    d->nl = n_qubits - g;
    d->world = world;
    d->dtype = dtype;
    d->device = device;
    d->pos = ident;
    d->at = ident;
    d->virt = comm == nullptr;
    if (comm) {
      d->comm = *comm;
      if (comm->rank < 0 || static_cast<uint32_t>(comm->rank) >= world || comm->sendrecv == nullptr ||
          comm->allreduce_sum == nullptr)
        throw_invalid("distributed state: bad communicator");
      d->ranks = {static_cast<uint32_t>(comm->rank)};
    } else {
      for (uint32_t r = 0; r < world; ++r) d->ranks.push_back(r);
    }
    const uint64_t shard_bytes = (uint64_t{1} << d->nl) * (dtype == VQF_F64 ? 16u : 8u);
    d->chunk_bytes = std::min<uint64_t>(chunk_bytes ? chunk_bytes : kDefaultChunk, shard_bytes);
    struct Guard {
      vqf_dsv_state* s;
      ~Guard() {
        if (s) vqf_dsv_destroy(s);
      }
    } guard{d.get()};
    VQF_CUDA(cudaSetDevice(device));
    for (uint32_t r : d->ranks) {
      vqf_sv s = nullptr;
      if (vqf_sv_create(d->nl, 1, dtype, device, &s) != VQF_OK) throw Error(VQF_CUDA_ERROR, vqf_last_error());
      d->shards.push_back(s);
      if (r != 0) VQF_CUDA(cudaMemsetAsync(s->amps, 0, shard_bytes, s->stream));  // |0..0> lives on rank 0
      VQF_CUDA(cudaStreamSynchronize(s->stream));
    }
    if (!d->virt) {
      VQF_CUDA(cudaMalloc(&d->buf[0], d->chunk_bytes));
      VQF_CUDA(cudaMalloc(&d->buf[1], d->chunk_bytes));
    }
    VQF_CUDA(cudaMalloc(&d->part, 2 * kCrossBlocks * sizeof(double)));
    VQF_CUDA(cudaMallocHost(&d->part_host, 2 * kCrossBlocks * sizeof(double)));
    guard.s = nullptr;
    *out = d.release();
  });
}

int vqf_dsv_destroy(vqf_dsv d) {
  return guarded([&] {
    if (d == nullptr) return;
    cudaSetDevice(d->device);
    for (vqf_sv s : d->shards) vqf_sv_destroy(s);
    if (d->buf[0]) cudaFree(d->buf[0]);
    if (d->buf[1]) cudaFree(d->buf[1]);
    if (d->part) cudaFree(d->part);
    if (d->part_host) cudaFreeHost(d->part_host);
    delete d;
  });
}

int vqf_dsv_apply_circuit(vqf_dsv dd, const vqf_gate* gates, uint32_t n_gates) {
  return guarded([&] {
    vqf_dsv_state* d = checked(dd);
    if (n_gates && gates == nullptr) throw_invalid("null gates");
    vqf_statevector probe;
    probe.n_qubits = d->n;
    for (uint32_t i = 0; i < n_gates; ++i) sv_check_gate(&probe, gates[i]);  // all-or-nothing validation
    VQF_CUDA(cudaSetDevice(d->device));
    std::vector<uint32_t> pos = d->pos, at = d->at;
    Layout L{d->n, d->g, pos, at};
    std::vector<vqf_dsv_op> ops;
    std::vector<vqf_gate> mapped;
    plan_circuit(L, gates, n_gates, ops, mapped);
    Exec ex{d};
    for (const vqf_dsv_op& op : ops) {
      if (op.kind == VQF_DSV_SWAP) ex.swap(op.a, op.b);
      else ex.local(mapped.data() + op.first, op.count);
    }
    for (vqf_sv s : d->shards) VQF_CUDA(cudaStreamSynchronize(s->stream));
  });
}

int vqf_dsv_expectation(vqf_dsv dd, const vqf_hamiltonian* h, double* out) {
  return guarded([&] {
    vqf_dsv_state* d = checked(dd);
    if (h == nullptr || out == nullptr) throw_invalid("null argument");
    if (h->n_qubits != d->n) throw_invalid("expectation: qubit count mismatch");
    VQF_CUDA(cudaSetDevice(d->device));
    const auto ta = term_axes(h);
    std::vector<uint32_t> pos = d->pos, at = d->at;
    Layout L{d->n, d->g, pos, at};
    std::vector<vqf_dsv_op> ops;
    std::vector<vqf_dsv_term> pts;
    plan_expectation(L, ta, ops, pts);
    Exec ex{d};
    std::complex<double> tot = 0.0;
    for (const vqf_dsv_op& op : ops) {
      if (op.kind == VQF_DSV_SWAP) {
        ex.swap(op.a, op.b);
      } else if (op.kind == VQF_DSV_EVAL) {
        tot += ex.eval(h, pts.data() + op.first, op.count);
      } else if (op.kind == VQF_DSV_CROSS) {
        if (d->dtype == VQF_F64) tot += ex.cross<double2>(h, op.a, pts.data() + op.first, op.count);
        else tot += ex.cross<float2>(h, op.a, pts.data() + op.first, op.count);
      }
    }
    if (!d->virt) {
      double v[2] = {tot.real(), tot.imag()};
      if (d->comm.allreduce_sum(d->comm.user, v, 2) != 0) throw Error(VQF_RUNTIME_ERROR, "distributed state: allreduce failed");
      tot = std::complex<double>(v[0], v[1]);
    }
    if (std::abs(tot.imag()) >= 1e-10) throw_runtime("expectation has imaginary residue " + fstr(tot.imag()));
    out[0] = tot.real();
  });
}

int vqf_dsv_layout(vqf_dsv dd, uint32_t* position_of_qubit) {
  return guarded([&] {
    vqf_dsv_state* d = checked(dd);
    if (position_of_qubit == nullptr) throw_invalid("null argument");
    std::copy(d->pos.begin(), d->pos.end(), position_of_qubit);
  });
}

int vqf_dsv_shard_download(vqf_dsv dd, uint32_t rank, double* amps) {
  return guarded([&] {
    vqf_dsv_state* d = checked(dd);
    Exec ex{d};
    if (vqf_sv_download(ex.shard(rank), amps) != VQF_OK) throw Error(VQF_CUDA_ERROR, vqf_last_error());
  });
}

int vqf_dsv_shard_upload(vqf_dsv dd, uint32_t rank, const double* amps) {
  return guarded([&] {
    vqf_dsv_state* d = checked(dd);
    Exec ex{d};
    if (vqf_sv_upload(ex.shard(rank), amps) != VQF_OK) throw Error(VQF_CUDA_ERROR, vqf_last_error());
  });
}

int vqf_dsv_stats(vqf_dsv dd, uint64_t* swaps, uint64_t* bytes_sent, uint64_t* scratch_bytes) {
  return guarded([&] {
    vqf_dsv_state* d = checked(dd);
    if (swaps) *swaps = d->swaps;
    if (bytes_sent) *bytes_sent = d->bytes_sent;
    if (scratch_bytes) *scratch_bytes = (d->virt ? 0 : 2 * d->chunk_bytes) + 2 * kCrossBlocks * sizeof(double);
  });
}

}  // extern "C"
