// Host drivers of the VQE hot path: prepare_ansatz / energy / gradient /
// run_vqe (vqe.hpp:65-254), run_sweep (sweep.hpp:128-178) and
// run_scaling_study (sweep.hpp:265-307), over two device engines:
//   * the register-resident batched engine (vqe_small.cu) for n <= 5 — the
//     H2 PES runs there, chemistry included, one launch per worker;
//   * the HBM state-vector engine (sv.cu) for wider registers: all 2P+1
//     parameter-shift circuits of an iteration are one batched state, so each
//     gate position is one launch over every circuit.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <limits>
#include <memory>
#include <mutex>
#include <thread>

#include "adjoint.cuh"
#include "chem_host.h"
#include "pauli_host.h"
#include "sv.cuh"
#include "tile.cuh"
#include "vqe_block.cuh"
#include "vqe_small.cuh"

namespace vqf {

namespace {

constexpr double kShift = 1.5707963267948966;  // std::numbers::pi / 2 (vqe.hpp:115)

using Clock = std::chrono::steady_clock;

double seconds_since(Clock::time_point t0) {
  return std::chrono::duration<double>(Clock::now() - t0).count();
}

void check_adam(const vqf_adam_config* c) {
  if (c == nullptr) throw_invalid("null adam config");
}

std::string nonfinite_msg(int iter, const double* theta, uint32_t P) {
  std::string msg = "non-finite energy at iteration " + std::to_string(iter) + "; theta =";
  for (uint32_t k = 0; k < P; ++k) msg += " " + fstr(theta[k]);
  return msg;
}

std::string imag_msg(double v) { return "expectation has imaginary residue " + fstr(v); }

// Validates (kind, layers, n) the way prepare_ansatz does (vqe.hpp:68-75).
uint32_t ansatz_params(int32_t kind, uint32_t layers, uint32_t n) {
  if (kind != VQF_ANSATZ_H2_DOUBLE_EXCITATION && kind != VQF_ANSATZ_HARDWARE_EFFICIENT)
    throw Error(VQF_LOGIC_ERROR, "unknown ansatz kind");
  return kind == VQF_ANSATZ_H2_DOUBLE_EXCITATION ? 1u : layers * n;
}

void check_ansatz_register(int32_t kind, uint32_t n) {
  if (kind == VQF_ANSATZ_H2_DOUBLE_EXCITATION && n != 4)
    throw_invalid("H2 double-excitation ansatz requires 4 qubits");
}

// ------------------------------------------------------------------------
// Per-(thread, device) workspace: a stream, pinned staging buffers and
// device buffers that grow monotonically, so steady-state calls allocate
// nothing.
struct Workspace {
  int device = -1;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  void* dev = nullptr;
  size_t dev_cap = 0;
  void* pin = nullptr;
  size_t pin_cap = 0;
  ~Workspace() {
    if (device < 0) return;
    cudaSetDevice(device);
    if (dev) cudaFree(dev);
    if (pin) cudaFreeHost(pin);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (stream) cudaStreamDestroy(stream);
  }
  void reserve(size_t dev_bytes, size_t pin_bytes) {
    if (dev_bytes > dev_cap) {
      if (dev) VQF_CUDA(cudaFree(dev));
      VQF_CUDA(cudaMalloc(&dev, dev_bytes));
      dev_cap = dev_bytes;
    }
    if (pin_bytes > pin_cap) {
      if (pin) VQF_CUDA(cudaFreeHost(pin));
      VQF_CUDA(cudaMallocHost(&pin, pin_bytes));
      pin_cap = pin_bytes;
    }
  }
};

Workspace& workspace(int device) {
  thread_local std::vector<std::unique_ptr<Workspace>> pool;
  for (auto& w : pool)
    if (w->device == device) return *w;
  auto w = std::make_unique<Workspace>();
  VQF_CUDA(cudaSetDevice(device));
  VQF_CUDA(cudaStreamCreateWithFlags(&w->stream, cudaStreamNonBlocking));
  VQF_CUDA(cudaEventCreate(&w->ev0));
  VQF_CUDA(cudaEventCreate(&w->ev1));
  w->device = device;
  pool.push_back(std::move(w));
  return *pool.back();
}

// Carves typed slices out of one contiguous byte range (16-byte aligned).
struct Carver {
  size_t off = 0;
  template <typename T>
  size_t take(size_t count) {
    off = (off + 15) & ~size_t{15};
    const size_t at = off;
    off += count * sizeof(T);
    return at;
  }
};

// ------------------------------------------------------------------------
// Small-register batched engine: shared by run_vqe (batch 1), run_vqe_batch
// and run_sweep (PES mode).
struct SmallJob {
  uint32_t batch = 0;
  int32_t n_qubits = 4, kind = 0, layers = 0;
  uint32_t P = 1;
  vqf_adam_config adam{};
  bool pes = false;
  // inputs
  std::vector<double> bonds;          // PES
  std::vector<int32_t> status_in;     // PES: kStatusBond pre-marked
  // PES grid mode: bonds [grid_first, grid_first + batch) of
  // bond_grid(grid_min, grid_max, grid_n) are generated and range-checked on
  // the device, Adam tables come from the device cache: no H2D copy at all
  int32_t grid_n = 0, grid_first = 0;
  double grid_min = 0.0, grid_max = 0.0;
  std::vector<MaskTerm> terms;        // generic
  std::vector<uint32_t> term_off;     // generic
  std::vector<double> init_theta;     // optional, batch * P
  bool want_ham = false;
  // outputs (host)
  std::vector<double> energy, theta, traj, err_val, err_theta, ham_coeffs, hf;
  std::vector<int32_t> iters, converged, status, err_iter, ham_keys, ham_count;
  double device_seconds = 0.0;
};

// -DVQF_HOST_TIMING: host-side checkpoints of the run_sweep path (scripts/host_timing.sh)
#ifdef VQF_HOST_TIMING
struct HostMarks {
  std::chrono::steady_clock::time_point t[16];
  const char* name[16];
  int n = 0;
  void mark(const char* what) {
    if (n < 16) {
      t[n] = std::chrono::steady_clock::now();
      name[n++] = what;
    }
  }
  void dump() {
    for (int i = 1; i < n; ++i)
      std::fprintf(stderr, "HOST %-14s %8.2f us\n", name[i],
                   std::chrono::duration<double, std::micro>(t[i] - t[i - 1]).count());
    n = 0;
  }
};
static HostMarks g_marks;
#define HMARK(x) g_marks.mark(x)
#define HDUMP() g_marks.dump()
#else
#define HMARK(x)
#define HDUMP()
#endif

// Adam bias-correction tables (2T std::pow calls, ~20 us for T = 200) are a
// function of (beta1, beta2, T) only: computed once per distinct triple.
void cached_bias_tables(const vqf_adam_config& c, int32_t T, std::vector<double>& bc1, std::vector<double>& bc2) {
  struct Entry {
    double b1, b2;
    int32_t T;
    std::vector<double> bc1, bc2;
  };
  static std::mutex mu;
  static std::vector<Entry> cache;
  std::lock_guard<std::mutex> lock(mu);
  for (const Entry& e : cache)
    if (e.b1 == c.beta1 && e.b2 == c.beta2 && e.T == T) {
      bc1 = e.bc1;
      bc2 = e.bc2;
      return;
    }
  host::bias_tables(c, T, bc1, bc2);
  if (cache.size() >= 8) cache.erase(cache.begin());
  cache.push_back(Entry{c.beta1, c.beta2, T, bc1, bc2});
}

// Device-resident copy of the bias tables per (device, beta1, beta2, T),
// uploaded once; null when the cache is full (the caller stages them).
const double* device_bias_tables(int device, const vqf_adam_config& c, int32_t T) {
  struct Entry {
    int device;
    double b1, b2;
    int32_t T;
    double* ptr;
  };
  static std::mutex mu;
  static std::vector<Entry> cache;
  std::lock_guard<std::mutex> lock(mu);
  for (const Entry& e : cache)
    if (e.device == device && e.b1 == c.beta1 && e.b2 == c.beta2 && e.T == T) return e.ptr;
  if (cache.size() >= 64) return nullptr;
  std::vector<double> bc1, bc2;
  cached_bias_tables(c, T, bc1, bc2);
  const size_t n = bc1.size();
  double* d = nullptr;
  VQF_CUDA(cudaMalloc(&d, 2 * n * sizeof(double)));
  VQF_CUDA(cudaMemcpy(d, bc1.data(), n * sizeof(double), cudaMemcpyHostToDevice));
  VQF_CUDA(cudaMemcpy(d + n, bc2.data(), n * sizeof(double), cudaMemcpyHostToDevice));
  cache.push_back(Entry{device, c.beta1, c.beta2, T, d});
  return d;
}

// Device layout of one small-engine job: inputs, then fixed-size outputs,
// then the trajectories (last, so a caller that does not want them skips
// their D2H copy).  One H2D copy in, one D2H copy out.
struct SmallStage {
  size_t o_bc1, o_bc2, o_bonds, o_terms, o_toff, o_init, o_status, in_end;
  size_t o_energy, o_theta, o_iters, o_conv, o_errv, o_erri, o_errt, o_hk, o_hc, o_hn, o_hf, o_clk, o_traj, out_end, total;
  uint32_t stride = 1;
  std::vector<double> bc1, bc2;

  explicit SmallStage(const SmallJob& j) {
    const uint32_t B = j.batch, P = j.P;
    const int32_t T = j.adam.max_iterations;
    stride = static_cast<uint32_t>(std::max(T, 0)) + 1;
    cached_bias_tables(j.adam, T, bc1, bc2);
    Carver c;
    o_bc1 = c.take<double>(bc1.size());
    o_bc2 = c.take<double>(bc2.size());
    o_bonds = c.take<double>(j.pes ? B : 0);
    o_terms = c.take<MaskTerm>(j.terms.size());
    o_toff = c.take<uint32_t>(j.term_off.size());
    o_init = c.take<double>(j.init_theta.size());
    o_status = c.take<int32_t>(B);
    in_end = c.off;
    o_energy = c.take<double>(B);
    o_theta = c.take<double>((size_t)B * P);
    o_iters = c.take<int32_t>(B);
    o_conv = c.take<int32_t>(B);
    o_errv = c.take<double>(B);
    o_erri = c.take<int32_t>(B);
    o_errt = c.take<double>((size_t)B * P);
    o_hk = c.take<int32_t>(j.want_ham ? (size_t)B * 16 : 0);
    o_hc = c.take<double>(j.want_ham ? (size_t)B * 16 : 0);
    o_hn = c.take<int32_t>(j.want_ham ? B : 0);
    o_hf = c.take<double>(j.want_ham ? (size_t)B * 4 : 0);
    o_clk = c.take<uint64_t>(2 * (size_t)B);
    out_end = c.off;
    o_traj = c.take<double>((size_t)B * stride);
    total = c.off;
  }

  void pack(const SmallJob& j, unsigned char* pin) const {
    const uint32_t B = j.batch;
    std::memcpy(pin + o_bc1, bc1.data(), bc1.size() * sizeof(double));
    std::memcpy(pin + o_bc2, bc2.data(), bc2.size() * sizeof(double));
    if (j.pes) std::memcpy(pin + o_bonds, j.bonds.data(), B * sizeof(double));
    if (!j.terms.empty()) std::memcpy(pin + o_terms, j.terms.data(), j.terms.size() * sizeof(MaskTerm));
    if (!j.term_off.empty()) std::memcpy(pin + o_toff, j.term_off.data(), j.term_off.size() * sizeof(uint32_t));
    if (!j.init_theta.empty())
      std::memcpy(pin + o_init, j.init_theta.data(), j.init_theta.size() * sizeof(double));
    if (j.status_in.empty())
      std::memset(pin + o_status, 0, B * sizeof(int32_t));
    else
      std::memcpy(pin + o_status, j.status_in.data(), B * sizeof(int32_t));
  }

  // out_host: when set, the fixed-size outputs (status .. hf) are written by
  // the kernel straight into this mapped pinned buffer (zero-copy; no D2H
  // copy and its DMA latency); trajectories stay in device memory.
  SmallParams params(const SmallJob& j, unsigned char* dev, int device, unsigned char* out_host = nullptr) const {
    unsigned char* out = out_host ? out_host : dev;
    SmallParams p{};
    p.n_qubits = j.n_qubits;
    p.ansatz_kind = j.kind;
    p.layers = j.layers;
    p.n_params = static_cast<int32_t>(j.P);
    p.max_iterations = j.adam.max_iterations;
    p.has_tol = j.adam.has_gradient_tolerance;
    p.tol = j.adam.gradient_tolerance;
    p.lr = j.adam.learning_rate;
    p.beta1 = j.adam.beta1;
    p.beta2 = j.adam.beta2;
    p.eps = j.adam.epsilon;
    p.bc1 = reinterpret_cast<const double*>(dev + o_bc1);
    p.bc2 = reinterpret_cast<const double*>(dev + o_bc2);
    p.bonds = reinterpret_cast<const double*>(dev + o_bonds);
    if (j.grid_n > 0) {
      const double* tab = device_bias_tables(device, j.adam, j.adam.max_iterations);
      if (tab != nullptr) {
        p.bc1 = tab;
        p.bc2 = tab + bc1.size();
        p.grid_n = j.grid_n;
        p.grid_first = j.grid_first;
        p.grid_min = j.grid_min;
        p.grid_max = j.grid_max;
      }
    }
    p.chem = chem::consts();
    p.jw = j.pes ? chem::jw_table_device(device) : nullptr;
    p.terms = reinterpret_cast<const MaskTerm*>(dev + o_terms);
    p.term_off = reinterpret_cast<const uint32_t*>(dev + o_toff);
    p.init_theta = j.init_theta.empty() ? nullptr : reinterpret_cast<const double*>(dev + o_init);
    p.energy = reinterpret_cast<double*>(out + o_energy);
    p.theta_out = reinterpret_cast<double*>(out + o_theta);
    p.traj = reinterpret_cast<double*>(dev + o_traj);
    p.traj_stride = static_cast<int32_t>(stride);
    p.iters = reinterpret_cast<int32_t*>(out + o_iters);
    p.converged = reinterpret_cast<int32_t*>(out + o_conv);
    p.status = reinterpret_cast<int32_t*>(out + o_status);
    p.err_val = reinterpret_cast<double*>(out + o_errv);
    p.err_iter = reinterpret_cast<int32_t*>(out + o_erri);
    p.err_theta = reinterpret_cast<double*>(out + o_errt);
    if (j.want_ham) {
      p.ham_keys = reinterpret_cast<int32_t*>(out + o_hk);
      p.ham_coeffs = reinterpret_cast<double*>(out + o_hc);
      p.ham_count = reinterpret_cast<int32_t*>(out + o_hn);
      p.hf_out = reinterpret_cast<double*>(out + o_hf);
    }
    p.clk = reinterpret_cast<unsigned long long*>(out + o_clk);
    return p;
  }

  // Bytes of the D2H copy (status .. outputs [.. trajectories]).
  size_t d2h_bytes(bool traj) const { return (traj ? total : out_end) - o_status; }

  void unpack(SmallJob& j, const unsigned char* pin, bool traj) const {
    const uint32_t B = j.batch, P = j.P;
    auto grab = [&](auto& vec, size_t off, size_t count) {
      using T0 = typename std::decay_t<decltype(vec)>::value_type;
      vec.resize(count);
      if (count) std::memcpy(vec.data(), pin + off, count * sizeof(T0));
    };
    grab(j.status, o_status, B);
    grab(j.energy, o_energy, B);
    grab(j.theta, o_theta, (size_t)B * P);
    grab(j.iters, o_iters, B);
    grab(j.converged, o_conv, B);
    grab(j.err_val, o_errv, B);
    grab(j.err_iter, o_erri, B);
    grab(j.err_theta, o_errt, (size_t)B * P);
    if (j.want_ham) {
      grab(j.ham_keys, o_hk, (size_t)B * 16);
      grab(j.ham_coeffs, o_hc, (size_t)B * 16);
      grab(j.ham_count, o_hn, B);
      grab(j.hf, o_hf, (size_t)B * 4);
    }
    if (traj) grab(j.traj, o_traj, (size_t)B * stride);
  }
};

// Stage, launch and read back one job on the thread's workspace stream.
// Returns the H2D / D2H byte counts through the optional pointers.
void run_small(SmallJob& j, int device, bool want_traj = true, size_t* h2d = nullptr, size_t* d2h = nullptr) {
  Workspace& ws = workspace(device);
  VQF_CUDA(cudaSetDevice(device));
  HMARK("setdevice");
  const SmallStage st(j);
  ws.reserve(st.total, st.total);
  auto* pin = static_cast<unsigned char*>(ws.pin);
  auto* dev = static_cast<unsigned char*>(ws.dev);
  st.pack(j, pin);
  const SmallParams p = st.params(j, dev, device, pin);
  const bool staged = p.grid_n == 0;  // grid mode needs no inputs from the host
  HMARK("stage+params");
  if (staged) VQF_CUDA(cudaMemcpyAsync(dev, pin, st.in_end, cudaMemcpyHostToDevice, ws.stream));
  auto* clk = reinterpret_cast<uint64_t*>(pin + st.o_clk);  // zero-copy: the kernel stamps CTA entry / result
  std::memset(clk, 0, 2 * sizeof(uint64_t) * j.batch);
  launch_vqe_small(p, j.batch, j.pes, ws.stream);
  HMARK("launch");
  if (want_traj)  // outputs arrive zero-copy; only trajectories need a copy
    VQF_CUDA(cudaMemcpyAsync(pin + st.o_traj, dev + st.o_traj, st.total - st.o_traj, cudaMemcpyDeviceToHost,
                             ws.stream));
  HMARK("d2h issue");
  VQF_CUDA(cudaStreamSynchronize(ws.stream));
  HMARK("sync");
  // device time of the launch: first CTA entry to last result write
  uint64_t t0 = UINT64_MAX, t1 = 0;
  for (uint32_t b = 0; b < j.batch; ++b) {
    if (clk[2 * b]) t0 = std::min<uint64_t>(t0, clk[2 * b]);
    t1 = std::max<uint64_t>(t1, clk[2 * b + 1]);
  }
  j.device_seconds = (t1 > t0 && t0 != UINT64_MAX) ? (t1 - t0) * 1e-9 : 0.0;
  st.unpack(j, pin, want_traj);
  HMARK("unpack");
  if (h2d) *h2d = staged ? st.in_end : 0;
  if (d2h) *d2h = st.d2h_bytes(want_traj);
}

std::string small_error(const SmallJob& j, uint32_t b, double bond) {
  switch (j.status[b]) {
    case kStatusImag: return imag_msg(j.err_val[b]);
    case kStatusNonFinite: return nonfinite_msg(j.err_iter[b], j.err_theta.data() + (size_t)b * j.P, j.P);
    case kStatusScf: return chem::nonconvergence_msg(bond);
    case kStatusHermitian: return chem::nonhermitian_msg(j.err_val[b]);
    default: return "unknown device status " + std::to_string(j.status[b]);
  }
}

void fill_result(const SmallJob& j, uint32_t b, vqf_vqe_result* r) {
  const int32_t T = j.adam.max_iterations;
  const uint32_t stride = static_cast<uint32_t>(T) + 1;
  const int32_t it = j.iters[b];
  const bool conv = j.converged[b] != 0;
  r->energy = j.energy[b];
  if (r->theta) std::memcpy(r->theta, j.theta.data() + (size_t)b * j.P, j.P * sizeof(double));
  const uint32_t len = conv ? static_cast<uint32_t>(it) + 1 : static_cast<uint32_t>(T) + 1;
  if (r->trajectory) {
    if (r->trajectory_capacity < len) throw_invalid("vqe_result: trajectory capacity too small");
    std::memcpy(r->trajectory, j.traj.data() + (size_t)b * stride, len * sizeof(double));
  }
  r->trajectory_len = len;
  r->iterations_run = it;
  // one energy + 2P shifts per gradient iteration, +1 final when not
  // converged (vqe.hpp:215, :230, :244-247)
  const uint64_t grads = conv ? static_cast<uint64_t>(it) + 1 : static_cast<uint64_t>(T);
  r->circuit_evaluations = grads * (1 + 2 * (uint64_t)j.P) + (conv ? 0 : 1);
}

// prepare_ansatz (vqe.hpp:65-96) as a fusable gate list; parameterised gates
// take their (cos, sin) from the engine's per-entry table.
std::vector<TGate> ansatz_tgates(int32_t kind, uint32_t layers, uint32_t n) {
  std::vector<TGate> g;
  if (kind == VQF_ANSATZ_H2_DOUBLE_EXCITATION) {
    g.push_back(TGate{VQF_GATE_DOUBLE_EXCITATION, 4, {0, 1, 2, 3}, 0, 0.0, 0.0});
    return g;
  }
  int32_t k = 0;
  for (uint32_t layer = 0; layer < layers; ++layer) {
    for (uint32_t q = 0; q < n; ++q) g.push_back(TGate{VQF_GATE_RY, 1, {q, 0, 0, 0}, k++, 0.0, 0.0});
    for (uint32_t q = 0; q + 1 < n; ++q) g.push_back(TGate{VQF_GATE_CNOT, 2, {q, q + 1, 0, 0}, -1, 0.0, 0.0});
  }
  return g;
}

// ------------------------------------------------------------------------
// HBM engine: prepare every circuit of `thetas` (NC rows of P angles) into
// an NC-entry batch and evaluate <H>.  Angles go through the host libm
// (std::cos/std::sin of 0.5*angle, as apply_gate does) into per-entry tables.
struct HbmEngine {
  uint32_t n, P, layers;
  int32_t kind;
  int device;
  vqf_statevector* sv = nullptr;
  std::vector<double> cs;  // [param][entry] (cos, sin)
  HbmEngine(uint32_t n_, int32_t kind_, uint32_t layers_, uint32_t batch, int device_, int32_t dtype = VQF_F64)
      : n(n_), P(ansatz_params(kind_, layers_, n_)), layers(layers_), kind(kind_), device(device_) {
    if (vqf_sv_create(n, batch, dtype, device, &sv) != VQF_OK) throw Error(VQF_CUDA_ERROR, vqf_last_error());
  }
  ~HbmEngine() { vqf_sv_destroy(sv); }
  HbmEngine(const HbmEngine&) = delete;

  // Prepares circuits; `angle(j, e)` gives parameter j's angle in entry e.
  template <typename F>
  void prepare(F&& angle) {
    const uint32_t B = sv->batch;
    cs.resize((size_t)std::max(P, 1u) * B * 2);
    for (uint32_t j = 0; j < P; ++j)
      for (uint32_t e = 0; e < B; ++e) {
        const double a = angle(j, e);
        cs[2 * ((size_t)j * B + e)] = std::cos(0.5 * a);
        cs[2 * ((size_t)j * B + e) + 1] = std::sin(0.5 * a);
      }
    sv_ensure_cs(sv, cs.size());
    VQF_CUDA(cudaMemcpyAsync(sv->cs_dev, cs.data(), cs.size() * sizeof(double), cudaMemcpyHostToDevice,
                             sv->stream));
    sv_reset(sv, kind == VQF_ANSATZ_H2_DOUBLE_EXCITATION ? 12 : 0);  // basis_state(4, {1,1,0,0}) / |0..0>
    run_circuit_tiled(sv, ansatz_tgates(kind, layers, n), sv->cs_dev);
  }

  // Same states as prepare() for a circuit family whose entry e agrees with
  // entry 0 before tile pass join[e] (run_circuit_tiled_shared): only the
  // entries with join 0 are reset; the rest are copied from entry 0.
  template <typename F>
  void prepare_shared(F&& angle, const std::vector<uint32_t>& join) {
    const uint32_t B = sv->batch;
    cs.resize((size_t)std::max(P, 1u) * B * 2);
    for (uint32_t j = 0; j < P; ++j)
      for (uint32_t e = 0; e < B; ++e) {
        const double a = angle(j, e);
        cs[2 * ((size_t)j * B + e)] = std::cos(0.5 * a);
        cs[2 * ((size_t)j * B + e) + 1] = std::sin(0.5 * a);
      }
    sv_ensure_cs(sv, cs.size());
    VQF_CUDA(cudaMemcpyAsync(sv->cs_dev, cs.data(), cs.size() * sizeof(double), cudaMemcpyHostToDevice,
                             sv->stream));
    uint32_t k0 = 0;
    while (k0 < B && join[k0] == 0) ++k0;
    sv->batch = std::max(k0, 1u);
    try {
      sv_reset(sv, kind == VQF_ANSATZ_H2_DOUBLE_EXCITATION ? 12 : 0);
    } catch (...) {
      sv->batch = B;
      throw;
    }
    sv->batch = B;
    run_circuit_tiled_shared(sv, ansatz_tgates(kind, layers, n), sv->cs_dev, join);
  }
};

// Device memory size, queried once per device.
size_t total_device_bytes(int device) {
  static std::mutex mu;
  static std::vector<std::pair<int, size_t>> cache;
  std::lock_guard<std::mutex> lock(mu);
  for (const auto& e : cache)
    if (e.first == device) return e.second;
  cudaDeviceProp prop{};
  VQF_CUDA(cudaGetDeviceProperties(&prop, device));
  cache.emplace_back(device, prop.totalGlobalMem);
  return prop.totalGlobalMem;
}

// Memory a new state batch can take: the driver's free bytes plus what the
// device's stream-ordered pool holds reserved but unused (the pool keeps
// freed states mapped, sv.cu retain_pool, so after a wide run cudaMemGetInfo
// alone reports that memory as taken and would shrink later shift batches
// to a few entries: n = 16 shift runs went from 5 to 12-16 ms after n = 26).
size_t free_device_bytes(int device) {
  size_t fr = 0, tot = 0;
  VQF_CUDA(cudaSetDevice(device));
  VQF_CUDA(cudaMemGetInfo(&fr, &tot));
  cudaMemPool_t pool;
  uint64_t reserved = 0, used = 0;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess &&
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved) == cudaSuccess &&
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used) == cudaSuccess && reserved > used)
    fr += static_cast<size_t>(reserved - used);
  return fr;
}

// Runs all 2P+1 circuits of one parameter-shift iteration; E[c] complex.
// Uses one NC-entry batch when it fits in 60% of free memory, else NC
// sequential single-entry evaluations.
struct ShiftEvaluator {
  uint32_t n, P, NC;
  int32_t kind;
  uint32_t layers;
  int device;
  std::unique_ptr<HbmEngine> eng;
  uint32_t K;    // batch entries of the engine (<= NC; what fits 60% of free memory)
  bool batched;  // K == NC
  // shared-prefix layout of the family: position e holds circuit order[e]
  // (order[0] = 0, the base); join[e] = first tile pass using the shifted
  // parameter.  Chunks of K - 1 shifted circuits run with the base as entry 0.
  std::vector<uint32_t> order, join;
  ShiftEvaluator(uint32_t n_, int32_t kind_, uint32_t layers_, int device_, int32_t dtype = VQF_F64)
      : n(n_), P(ansatz_params(kind_, layers_, n_)), NC(2 * P + 1), kind(kind_), layers(layers_), device(device_) {
    const double entry = (double)(uint64_t{1} << n) * (dtype == VQF_F64 ? 16.0 : 8.0);
    // a family far below the device's memory needs no free-memory query
    // (cudaMemGetInfo measured 0.4-9 ms per call once many pool allocations
    // exist: it dominated the n = 16 studies' jitter)
    if ((double)NC * entry <= (double)total_device_bytes(device) / 32)
      K = NC;
    else
      K = static_cast<uint32_t>(
          std::max(1.0, std::min<double>(NC, std::floor(0.6 * (double)free_device_bytes(device) / entry))));
    if (const char* cap = std::getenv("VQF_SHIFT_MAX_BATCH")) K = std::max(1u, std::min<uint32_t>(K, std::atoi(cap)));
    batched = K == NC;
    // a chunk recomputes the base circuit: below 8 entries per chunk one
    // circuit at a time is cheaper
    if (!batched && K < 8) K = 1;
    const std::vector<int> first =
        K >= 2 ? tile_param_first_pass(n, dtype, ansatz_tgates(kind, layers, n), P) : std::vector<int>{};
    if (!first.empty() && !std::getenv("VQF_NO_SHARED_PREFIX")) {
      const auto join_of = [&](uint32_t c) -> uint32_t {
        if (c == 0) return 0;
        const int f = first[(c - 1) / 2];
        return f < 0 ? UINT32_MAX : static_cast<uint32_t>(f);
      };
      order.resize(NC);
      for (uint32_t c = 0; c < NC; ++c) order[c] = c;
      std::stable_sort(order.begin() + 1, order.end(),
                       [&](uint32_t a, uint32_t b) { return join_of(a) < join_of(b); });
      for (uint32_t e = 0; e < NC; ++e) join.push_back(join_of(order[e]));
    } else if (!batched) {
      K = 1;  // no prefix sharing: one circuit at a time
    }
    eng = std::make_unique<HbmEngine>(n, kind, layers, K, device, dtype);
  }
  // runs f with the engine's batch temporarily set to b entries
  template <typename F>
  void with_batch(uint32_t b, F&& f) {
    const uint32_t full = eng->sv->batch;
    eng->sv->batch = b;
    try {
      f();
    } catch (...) {
      eng->sv->batch = full;
      throw;
    }
    eng->sv->batch = full;
  }
  // circuits [0, c_count) of the shift family around theta
  void run(const std::vector<double>& theta, const CompiledHam& h, int c_count, std::vector<double>& E) {
    E.assign(2 * (size_t)c_count, 0.0);
    const auto angle_of = [&](uint32_t j, uint32_t c) {
      double t = theta[j];
      if (c == 2 * j + 1) t = theta[j] + kShift;
      if (c == 2 * j + 2) t = theta[j] - kShift;
      return t;
    };
    if (c_count == (int)NC && !order.empty()) {
      std::vector<uint32_t> co, cj;
      std::vector<double> tot;
      for (uint32_t i = 1; i < NC; i += K - 1) {
        const uint32_t m = std::min(K - 1, NC - i);
        co.assign(1, 0u);
        cj.assign(1, 0u);
        for (uint32_t t = 0; t < m; ++t) {
          co.push_back(order[i + t]);
          cj.push_back(join[i + t]);
        }
        tot.assign(2 * (size_t)(m + 1), 0.0);
        with_batch(m + 1, [&] {
          eng->prepare_shared([&](uint32_t j, uint32_t e) { return angle_of(j, co[e]); }, cj);
          sv_expectation(eng->sv, h, tot.data());
        });
        for (uint32_t e = i == 1 ? 0 : 1; e <= m; ++e) {
          E[2 * (size_t)co[e]] = tot[2 * (size_t)e];
          E[2 * (size_t)co[e] + 1] = tot[2 * (size_t)e + 1];
        }
      }
      return;
    }
    if (batched || (K > 1 && c_count <= (int)K)) {
      // entries are contiguous: run only the first c_count of them (the
      // final evaluation after the last Adam step needs one circuit)
      with_batch(static_cast<uint32_t>(c_count), [&] {
        eng->prepare([&](uint32_t j, uint32_t e) { return angle_of(j, e); });
        sv_expectation(eng->sv, h, E.data());
      });
      return;
    }
    for (int c = 0; c < c_count; ++c) {
      with_batch(1, [&] {
        eng->prepare([&](uint32_t j, uint32_t) { return angle_of(j, c); });
        double tot[2];
        sv_expectation(eng->sv, h, tot);
        E[2 * c] = tot[0];
        E[2 * c + 1] = tot[1];
      });
    }
  }
};

// prepare_ansatz (vqe.hpp:65-96) as a gate list for the adjoint sweep.
std::vector<AdjGate> ansatz_program(int32_t kind, uint32_t layers, uint32_t n) {
  std::vector<AdjGate> prog;
  if (kind == VQF_ANSATZ_H2_DOUBLE_EXCITATION) {
    prog.push_back(AdjGate{VQF_GATE_DOUBLE_EXCITATION, {0, 1, 2, 3}, 0});
    return prog;
  }
  int32_t k = 0;
  for (uint32_t layer = 0; layer < layers; ++layer) {
    for (uint32_t q = 0; q < n; ++q) prog.push_back(AdjGate{VQF_GATE_RY, {q, 0, 0, 0}, k++});
    for (uint32_t q = 0; q + 1 < n; ++q) prog.push_back(AdjGate{VQF_GATE_CNOT, {q, q + 1, 0, 0}, -1});
  }
  return prog;
}

// Forward state + lambda vector + adjoint plan for one register.
struct AdjointRunner {
  HbmEngine eng;
  vqf_statevector* lam = nullptr;
  AdjointPlan plan;
  std::vector<AdjGate> prog;
  AdjointRunner(uint32_t n, int32_t kind, uint32_t layers, int device, const CompiledHam& ch, int32_t dtype = VQF_F64)
      : eng(n, kind, layers, 1, device, dtype), prog(ansatz_program(kind, layers, n)) {
    if (vqf_sv_create(n, 1, dtype, device, &lam) != VQF_OK) throw Error(VQF_CUDA_ERROR, vqf_last_error());
    plan.init(eng.sv, lam, ch, eng.P);
  }
  ~AdjointRunner() { vqf_sv_destroy(lam); }
  // E(theta) (complex) and dE/dtheta.
  void run(const std::vector<double>& theta, double* e, double* grad) {
    eng.prepare([&](uint32_t j, uint32_t) { return theta[j]; });
    plan.run(prog, theta, e, grad);
  }
};

void run_vqe_hbm(const vqf_hamiltonian* h, int32_t kind, uint32_t layers, const vqf_adam_config& cfg,
                 const std::vector<double>& init, int32_t method, int device, vqf_vqe_result* r,
                 int32_t dtype = VQF_F64) {
  const uint32_t n = h->n_qubits;
  const CompiledHam ch = compile_hamiltonian(h);
  // Hamiltonians beyond the adjoint tables take parameter shift (same
  // gradient, the reference's own algorithm)
  const bool adjoint = method == VQF_GRAD_ADJOINT && AdjointPlan::supports(ch, n);
  std::unique_ptr<ShiftEvaluator> evp;
  std::unique_ptr<AdjointRunner> adj;
  if (adjoint) adj = std::make_unique<AdjointRunner>(n, kind, layers, device, ch, dtype);
  else evp = std::make_unique<ShiftEvaluator>(n, kind, layers, device, dtype);
  const uint32_t P = ansatz_params(kind, layers, n);
  std::vector<double> theta = init.empty() ? std::vector<double>(P, 0.0) : init;
  std::vector<double> m(P, 0.0), v(P, 0.0), grad(P), tn(P), mn(P), vn(P), E;
  int64_t step = 0;
  uint32_t len = 0;
  bool converged = false;
  r->iterations_run = 0;
  r->circuit_evaluations = 0;
  auto push = [&](double e) {
    if (r->trajectory) {
      if (len >= r->trajectory_capacity) throw_invalid("vqe_result: trajectory capacity too small");
      r->trajectory[len] = e;
    }
    ++len;
  };
  double last = 0.0;
  for (int iter = 0; iter < cfg.max_iterations; ++iter) {
    if (adjoint) {
      // one forward + one backward sweep; circuit_evaluations counts the
      // forward circuits actually executed
      E.assign(2, 0.0);
      adj->run(theta, E.data(), grad.data());
    } else {
      evp->run(theta, ch, static_cast<int>(evp->NC), E);
    }
    if (std::abs(E[1]) >= 1e-10) throw_runtime(imag_msg(E[1]));
    ++r->circuit_evaluations;
    if (!std::isfinite(E[0])) throw_runtime(nonfinite_msg(iter, theta.data(), P));
    push(E[0]);
    last = E[0];
    if (!adjoint) {
      for (uint32_t c = 1; c < evp->NC; ++c)
        if (std::abs(E[2 * c + 1]) >= 1e-10) throw_runtime(imag_msg(E[2 * c + 1]));
      for (uint32_t k = 0; k < P; ++k) grad[k] = 0.5 * (E[2 * (2 * k + 1)] - E[2 * (2 * k + 2)]);
      r->circuit_evaluations += 2 * (uint64_t)P;
    }
    if (cfg.has_gradient_tolerance) {
      double g_inf = 0.0;
      for (double g : grad) g_inf = std::max(g_inf, std::abs(g));
      if (g_inf < cfg.gradient_tolerance) {
        converged = true;
        break;
      }
    }
    host::adam_step(m.data(), v.data(), step, grad.data(), theta.data(), P, cfg, tn.data(), mn.data(), vn.data(),
                    &step);
    theta = tn;
    m = mn;
    v = vn;
    r->iterations_run = iter + 1;
  }
  if (!converged) {
    if (adjoint) {
      adj->eng.prepare([&](uint32_t j, uint32_t) { return theta[j]; });
      E.assign(2, 0.0);
      sv_expectation(adj->eng.sv, ch, E.data());
    } else {
      evp->run(theta, ch, 1, E);
    }
    if (std::abs(E[1]) >= 1e-10) throw_runtime(imag_msg(E[1]));
    ++r->circuit_evaluations;
    if (!std::isfinite(E[0])) throw_runtime(nonfinite_msg(cfg.max_iterations, theta.data(), P));
    push(E[0]);
    last = E[0];
  }
  r->energy = last;
  r->trajectory_len = len;
  if (r->theta) std::memcpy(r->theta, theta.data(), P * sizeof(double));
}

// One warp holds the problem with <= 16 amplitudes per lane (32 would spill:
// 5-qubit registers with >= 8 parameters take the shared-memory engine).
bool small_ok(uint32_t n, uint32_t P) {
  return n <= (uint32_t)kSmallMaxN && P <= (uint32_t)kSmallMaxP &&
         small_amps_per_lane(static_cast<int>(n), static_cast<int>(P)) <= 16;
}

// Engine override for diagnostics and cross-engine tests: VQF_ENGINE =
// warp | block | hbm (default: the fastest engine that holds the problem).
const char* engine_override() {
  const char* e = std::getenv("VQF_ENGINE");
  return (e && *e) ? e : nullptr;
}

bool block_ok(int32_t kind, uint32_t n, uint32_t P, int32_t dtype) {
  return kind == VQF_ANSATZ_HARDWARE_EFFICIENT && n >= (uint32_t)kBlockMinN && n <= (uint32_t)block_max_n(dtype) &&
         P <= (uint32_t)kBlockMaxP;
}

// 1 - beta^t for t = 1..T, interleaved (bc1, bc2), by the host libm pow as
// adam_step computes them (vqe.hpp:161-162); cached per (beta1, beta2, T).
std::vector<double> raw_bias_tables(const vqf_adam_config& c, int32_t T) {
  struct Entry {
    double b1, b2;
    int32_t T;
    std::vector<double> bc;
  };
  static std::mutex mu;
  static std::vector<std::unique_ptr<Entry>> cache;
  std::lock_guard<std::mutex> lock(mu);
  for (const auto& e : cache)
    if (e->b1 == c.beta1 && e->b2 == c.beta2 && e->T == T) return e->bc;
  auto e = std::make_unique<Entry>();
  e->b1 = c.beta1;
  e->b2 = c.beta2;
  e->T = T;
  e->bc.assign(2 * static_cast<size_t>(std::max(T, 1)), 0.0);
  for (int32_t t = 1; t <= T; ++t) {
    e->bc[2 * (t - 1)] = 1.0 - std::pow(c.beta1, static_cast<double>(t));
    e->bc[2 * (t - 1) + 1] = 1.0 - std::pow(c.beta2, static_cast<double>(t));
  }
  if (cache.size() >= 16) cache.erase(cache.begin());
  cache.push_back(std::move(e));
  return cache.back()->bc;
}

// Barrier words of the shared-memory engine, one per (thread, device):
// zeroed once, reset by the kernel's last CTA (or here after an abort).
unsigned* block_barrier(int device) {
  thread_local std::vector<std::pair<int, unsigned*>> words;
  for (const auto& w : words)
    if (w.first == device) return w.second;
  unsigned* d = nullptr;
  VQF_CUDA(cudaMalloc(&d, 4 * sizeof(unsigned)));
  VQF_CUDA(cudaMemset(d, 0, 4 * sizeof(unsigned)));
  words.emplace_back(device, d);
  return d;
}

// Shared-memory engine (vqe_block.cu): the whole run_vqe in one cooperative
// launch.  Inputs ride in the kernel parameter block when they fit
// (kBlockInline bytes), else go up in one H2D copy; results are written by
// the kernel straight into mapped pinned memory.
void run_vqe_block(const CompiledHam& ch, int32_t kind, uint32_t layers, const vqf_adam_config& cfg,
                   const std::vector<double>& init, int device, vqf_vqe_result* r, int32_t dtype) {
  const uint32_t n = ch.n_qubits;
  const uint32_t P = ansatz_params(kind, layers, n);
  const int NC = 2 * static_cast<int>(P) + 1;
  HMARK("block:enter");
  const BlockProgram prog = compile_block_program(kind, layers, n, ch, dtype);
  HMARK("compile");
  const int32_t T = cfg.max_iterations;
  const std::vector<double> bc = raw_bias_tables(cfg, T);
  Workspace& ws = workspace(device);
  VQF_CUDA(cudaSetDevice(device));
  HMARK("bias+ws");
  Carver c;  // inputs
  const size_t o_bc = c.take<double>(bc.size());
  const size_t o_pass = c.take<BlockPass>(prog.passes.size());
  const size_t o_gf = c.take<uint32_t>(prog.group_flip.size());
  const size_t o_go = c.take<uint32_t>(prog.group_off.size());
  const size_t o_terms = c.take<BlockTerm>(prog.herm ? 0 : prog.terms.size());  // complex form: non-Hermitian only
  const size_t o_rterms = c.take<BlockRTerm>(prog.rterms.size());
  const size_t o_init = c.take<double>(init.size());
  const size_t in_end = c.off;
  const bool inl = in_end <= static_cast<size_t>(kBlockInline);
  Carver oc;  // outputs (mapped pinned), after the staged inputs
  oc.off = inl ? 0 : in_end;
  const size_t o_energy = oc.take<double>(1);
  const size_t o_theta = oc.take<double>(P);
  const size_t o_traj = oc.take<double>(static_cast<size_t>(std::max(T, 0)) + 1);
  const size_t o_iters = oc.take<int32_t>(1);
  const size_t o_conv = oc.take<int32_t>(1);
  const size_t o_status = oc.take<int32_t>(1);
  const size_t o_errv = oc.take<double>(1);
  const size_t o_erri = oc.take<int32_t>(1);
  const size_t o_errt = oc.take<double>(P);
  const size_t o_clk = oc.take<uint64_t>(2);
  const size_t pin_total = oc.off;
  Carver dc;  // device scratch: staged inputs, the energy exchange, global states
  dc.off = inl ? 0 : in_end;
  const size_t o_E = dc.take<double2>(2 * static_cast<size_t>(NC));
  const int grid = block_grid(prog, dtype, NC, device);
  const size_t o_state = dc.take<double2>(prog.gmem ? static_cast<size_t>(grid) << n : 0);
  ws.reserve(dc.off, pin_total);
  auto* pin = static_cast<unsigned char*>(ws.pin);
  auto* dev = static_cast<unsigned char*>(ws.dev);
  static thread_local BlockArgs args;  // 8 KB: not on the stack
  unsigned char* in = inl ? args.blob : pin;
  auto put = [&](size_t off, const void* src, size_t bytes) {
    if (bytes) std::memcpy(in + off, src, bytes);
  };
  put(o_bc, bc.data(), bc.size() * sizeof(double));
  put(o_pass, prog.passes.data(), prog.passes.size() * sizeof(BlockPass));
  put(o_gf, prog.group_flip.data(), prog.group_flip.size() * sizeof(uint32_t));
  put(o_go, prog.group_off.data(), prog.group_off.size() * sizeof(uint32_t));
  if (!prog.herm) put(o_terms, prog.terms.data(), prog.terms.size() * sizeof(BlockTerm));
  put(o_rterms, prog.rterms.data(), prog.rterms.size() * sizeof(BlockRTerm));
  put(o_init, init.data(), init.size() * sizeof(double));
  std::memset(pin + (inl ? 0 : in_end), 0, pin_total - (inl ? 0 : in_end));
  // input addresses: device pointers (staged) or offsets into args.blob
  const auto src = [&](size_t off) -> const unsigned char* {
    return inl ? reinterpret_cast<const unsigned char*>(off) : dev + off;
  };
  BlockParams& p = args.p;
  p = BlockParams{};
  args.inl = inl ? 1 : 0;
  p.n = static_cast<int32_t>(n);
  p.P = static_cast<int32_t>(P);
  p.NC = NC;
  p.max_iterations = T;
  p.has_tol = cfg.has_gradient_tolerance;
  p.dtype = dtype;
  p.tol = cfg.gradient_tolerance;
  p.lr = cfg.learning_rate;
  p.beta1 = cfg.beta1;
  p.beta2 = cfg.beta2;
  p.eps = cfg.epsilon;
  p.bc = reinterpret_cast<const double*>(src(o_bc));
  p.passes = reinterpret_cast<const BlockPass*>(src(o_pass));
  p.n_passes = static_cast<int32_t>(prog.passes.size());
  p.init_index = prog.init_index;
  p.group_flip = reinterpret_cast<const uint32_t*>(src(o_gf));
  p.group_off = reinterpret_cast<const uint32_t*>(src(o_go));
  p.n_groups = static_cast<int32_t>(prog.group_flip.size());
  p.terms = reinterpret_cast<const BlockTerm*>(src(o_terms));
  p.herm = prog.herm ? 1 : 0;
  p.n_terms = static_cast<int32_t>(prog.terms.size());
  p.obytes = prog.obytes;
  p.team_lanes = static_cast<int32_t>(prog.lanes);
  p.gstate = prog.gmem ? static_cast<void*>(dev + o_state) : nullptr;
  p.rterms = reinterpret_cast<const BlockRTerm*>(src(o_rterms));
  p.init_theta = init.empty() ? nullptr : reinterpret_cast<const double*>(src(o_init));
  p.energies = reinterpret_cast<double2*>(dev + o_E);
  p.barrier = block_barrier(device);
  p.energy = reinterpret_cast<double*>(pin + o_energy);
  p.theta_out = reinterpret_cast<double*>(pin + o_theta);
  p.traj = reinterpret_cast<double*>(pin + o_traj);
  p.iters = reinterpret_cast<int32_t*>(pin + o_iters);
  p.converged = reinterpret_cast<int32_t*>(pin + o_conv);
  p.status = reinterpret_cast<int32_t*>(pin + o_status);
  p.err_val = reinterpret_cast<double*>(pin + o_errv);
  p.err_iter = reinterpret_cast<int32_t*>(pin + o_erri);
  p.err_theta = reinterpret_cast<double*>(pin + o_errt);
  p.clk = reinterpret_cast<unsigned long long*>(pin + o_clk);
  HMARK("stage");
  if (!inl) VQF_CUDA(cudaMemcpyAsync(dev, pin, in_end, cudaMemcpyHostToDevice, ws.stream));
  launch_vqe_block(args, in_end, prog, grid, ws.stream);
  HMARK("launch");
  VQF_CUDA(cudaStreamSynchronize(ws.stream));
  HMARK("sync");
  const int32_t st = *p.status;
  if (st == kStatusAbort) {
    VQF_CUDA(cudaMemset(p.barrier, 0, 4 * sizeof(unsigned)));
    throw Error(VQF_CUDA_ERROR, "block engine: grid barrier timed out");
  }
  if (st == kStatusImag) throw_runtime(imag_msg(*p.err_val));
  if (st == kStatusNonFinite) throw_runtime(nonfinite_msg(*p.err_iter, p.err_theta, P));
  if (st != kStatusOk) throw Error(VQF_LOGIC_ERROR, "block engine: status " + std::to_string(st));
  const int32_t it = *p.iters;
  const bool conv = *p.converged != 0;
  const uint32_t len = conv ? static_cast<uint32_t>(it) + 1 : static_cast<uint32_t>(T) + 1;
  r->energy = *p.energy;
  if (r->theta) std::memcpy(r->theta, p.theta_out, P * sizeof(double));
  if (r->trajectory) {
    if (r->trajectory_capacity < len) throw_invalid("vqe_result: trajectory capacity too small");
    std::memcpy(r->trajectory, p.traj, len * sizeof(double));
  }
  r->trajectory_len = len;
  r->iterations_run = it;
  const uint64_t grads = conv ? static_cast<uint64_t>(it) + 1 : static_cast<uint64_t>(T);
  r->circuit_evaluations = grads * (1 + 2 * (uint64_t)P) + (conv ? 0 : 1);
  HMARK("results");
  HDUMP();
}

// Storage precision of the engine's states.  complex64 (VQF_F32) runs
// fixed-iteration only: fp32 rounding cannot reproduce the reference's
// tol-mode stop decisions, so a gradient tolerance is
// refused rather than silently changing the iteration count.
void check_dtype(int32_t dtype, const vqf_adam_config* cfg) {
  if (dtype != VQF_F64 && dtype != VQF_F32) throw_invalid("unknown dtype");
  if (dtype == VQF_F32 && cfg != nullptr && cfg->has_gradient_tolerance)
    throw_invalid("fp32 (complex64) runs are fixed-iteration only: gradient_tolerance needs fp64");
}

void run_vqe_impl(const vqf_hamiltonian* h, int32_t kind, uint32_t layers, const vqf_adam_config* cfg,
                  const double* init, uint32_t n_init, int32_t method, int32_t device, vqf_vqe_result* r,
                  int32_t dtype = VQF_F64) {
  const auto t0 = Clock::now();
  check_adam(cfg);
  if (h == nullptr || r == nullptr) throw_invalid("null argument");
  const uint32_t n = h->n_qubits;
  const uint32_t P = ansatz_params(kind, layers, n);
  if (n_init != 0 && n_init != P) throw_invalid("initial parameter count mismatch");
  check_ansatz_register(kind, n);
  if (method != VQF_GRAD_PARAMETER_SHIFT && method != VQF_GRAD_ADJOINT) throw_invalid("unknown gradient method");
  check_dtype(dtype, cfg);
  std::vector<double> init_v(init, init + n_init);
  // registers that fit one warp run the whole optimisation in one launch
  // (k_vqe_warp, parameter-shift gradients); the adjoint method would equal
  // it to rounding but pays one HBM-engine launch per gate there, so small
  // registers take this path for either method (fp64 only: the register
  // engine holds complex128 amplitudes)
  const char* eng = engine_override();
  const bool want_warp = eng ? std::strcmp(eng, "warp") == 0 : true;
  const bool want_block = eng ? std::strcmp(eng, "block") == 0 : true;
  // hardware-efficient registers of >= 4 qubits: the shared-memory engine
  // (teams of lanes per circuit) beats the one-warp register engine
  const bool block_first = block_ok(kind, n, P, dtype) && !eng;
  if (dtype == VQF_F64 && small_ok(n, P) && want_warp && !block_first) {
    SmallJob j;
    j.batch = 1;
    j.n_qubits = static_cast<int32_t>(n);
    j.kind = kind;
    j.layers = static_cast<int32_t>(layers);
    j.P = P;
    j.adam = *cfg;
    const CompiledHam ch = compile_hamiltonian(h);
    j.terms = ch.terms;
    j.term_off = {0, static_cast<uint32_t>(ch.terms.size())};
    j.init_theta = init_v;
    run_small(j, device);
    if (j.status[0] != kStatusOk) throw_runtime(small_error(j, 0, 0.0));
    fill_result(j, 0, r);
  } else if (block_ok(kind, n, P, dtype) && want_block) {
    // one cooperative launch per run (parameter-shift gradients, also for
    // method = adjoint: equal to rounding, and the shifted circuits run in
    // parallel CTAs)
    HMARK("impl:enter");
    run_vqe_block(compile_hamiltonian(h), kind, layers, *cfg, init_v, device, r, dtype);
  } else {
    run_vqe_hbm(h, kind, layers, *cfg, init_v, method, device, r, dtype);
  }
  r->wall_seconds = seconds_since(t0);
}


// ------------------------------------------------------------ sweep pieces
struct SweepSlice {
  std::vector<double> grid;
  uint64_t lo = 0, hi = 0;
};

// bond_grid (sweep.hpp:68-85) and this rank's split_chunks slice of it.
SweepSlice sweep_slice(const vqf_sweep_config& cfg) {
  if (cfg.n_points < 1) throw_invalid("grid needs >= 1 point");
  if (cfg.d_max < cfg.d_min) throw_invalid("d_max < d_min");
  SweepSlice s;
  s.grid.resize(cfg.n_points);
  host::bond_grid(cfg.d_min, cfg.d_max, cfg.n_points, s.grid.data());
  s.lo = 0;
  s.hi = s.grid.size();
  if (cfg.n_chunks > 1) {
    if (cfg.chunk_index < 0 || cfg.chunk_index >= cfg.n_chunks) throw_invalid("chunk_index out of range");
    std::vector<uint64_t> be(2 * (size_t)cfg.n_chunks);
    host::split_chunks(s.grid.size(), cfg.n_chunks, be.data());
    s.lo = be[2 * cfg.chunk_index];
    s.hi = be[2 * cfg.chunk_index + 1];
  }
  return s;
}

std::vector<int32_t> sweep_devices(const vqf_sweep_config& cfg) {
  std::vector<int32_t> devices;
  if (cfg.devices != nullptr && cfg.n_devices > 0) {
    devices.assign(cfg.devices, cfg.devices + cfg.n_devices);
  } else {
    int nd = 0;
    VQF_CUDA(cudaGetDeviceCount(&nd));
    const int use = cfg.n_devices > 0 ? std::min(cfg.n_devices, nd) : nd;
    for (int d = 0; d < use; ++d) devices.push_back(d);
  }
  if (devices.empty()) throw Error(VQF_CUDA_ERROR, "CUDA: no device available");
  return devices;
}

// PES job for grid points [b0, b1): bonds outside the supported range are
// rejected on the host with the BondLengthOutOfRange text (chem.hpp:281-284)
// and skipped by the kernel.
SmallJob pes_job(const vqf_sweep_config& cfg, const std::vector<double>& grid, uint64_t b0, uint64_t b1,
                 std::vector<std::string>& errors) {
  SmallJob j;
  j.batch = static_cast<uint32_t>(b1 - b0);
  j.n_qubits = 4;
  j.kind = VQF_ANSATZ_H2_DOUBLE_EXCITATION;
  j.P = 1;
  j.adam = cfg.adam;
  j.pes = true;
  j.bonds.assign(grid.begin() + b0, grid.begin() + b1);
  j.status_in.assign(j.batch, 0);
  for (uint32_t b = 0; b < j.batch; ++b) {
    try {
      chem::check_bond(j.bonds[b]);
    } catch (const Error& e) {
      j.status_in[b] = kStatusBond;
      errors[b0 + b] = e.what();
    }
  }
  return j;
}

// Writes points [b0, b1) of the report (SweepPoint, sweep.hpp:48-56).
void pes_fill(const SmallJob& j, const vqf_sweep_config& cfg, const std::vector<double>& grid, uint64_t b0,
              uint64_t b1, std::vector<std::string>& errors, vqf_sweep_report* rep) {
  const uint32_t stride = static_cast<uint32_t>(std::max(cfg.adam.max_iterations, 0)) + 1;
  for (uint64_t i = b0; i < b1; ++i) {
    const uint32_t b = static_cast<uint32_t>(i - b0);
    rep->bond_angstrom[i] = grid[i];
    rep->energy_hartree[i] = std::numeric_limits<double>::quiet_NaN();
    rep->theta_star[i] = std::numeric_limits<double>::quiet_NaN();
    rep->iterations[i] = 0;
    rep->ok[i] = 0;
    if (rep->wall_seconds) rep->wall_seconds[i] = j.device_seconds;
    if (j.status.empty() || j.status[b] == kStatusBond) continue;
    if (j.status[b] != kStatusOk) {
      errors[i] = small_error(j, b, j.bonds[b]);
      continue;
    }
    rep->energy_hartree[i] = j.energy[b];
    rep->theta_star[i] = j.theta[b];
    rep->iterations[i] = j.iters[b];
    rep->ok[i] = 1;
    if (rep->trajectories && !j.traj.empty())
      std::memcpy(rep->trajectories + i * stride, j.traj.data() + (size_t)b * stride, stride * sizeof(double));
  }
}

void pes_finish(const SweepSlice& sl, const std::vector<std::string>& errors, vqf_sweep_report* rep) {
  int all_ok = 1;
  for (uint64_t i = sl.lo; i < sl.hi; ++i) {
    all_ok = all_ok && rep->ok[i];
    if (rep->errors && rep->error_stride) {
      char* dst = rep->errors + i * rep->error_stride;
      std::strncpy(dst, errors[i].c_str(), rep->error_stride - 1);
      dst[rep->error_stride - 1] = '\0';
    }
  }
  rep->all_ok = all_ok;
}

}  // namespace

}  // namespace vqf

// Device-resident PES plan (vqf_pes_create).
struct vqf_pes_plan {
  vqf_sweep_config cfg{};
  int device = 0;
  vqf::SweepSlice slice;
  std::vector<std::string> errors;
  vqf::SmallJob job;
  std::unique_ptr<vqf::SmallStage> stage;
  vqf::SmallParams params{};
  cudaStream_t stream = nullptr;
  cudaStream_t last_stream = nullptr;
  void* dev = nullptr;
  void* pin = nullptr;
};

using namespace vqf;

extern "C" {

int vqf_prepare_ansatz(int32_t kind, uint32_t layers, const double* theta, uint32_t n_theta, vqf_sv sv) {
  return guarded([&] {
    if (sv == nullptr) throw_invalid("null state vector");
    const uint32_t P = ansatz_params(kind, layers, sv->n_qubits);
    if (n_theta != P) throw_invalid("parameter count mismatch for ansatz");
    check_ansatz_register(kind, sv->n_qubits);
    VQF_CUDA(cudaSetDevice(sv->device));
    if (kind == VQF_ANSATZ_H2_DOUBLE_EXCITATION) {
      sv_reset(sv, 12);
      GateArgs g{VQF_GATE_DOUBLE_EXCITATION, 4, {0, 1, 2, 3}, std::cos(0.5 * theta[0]), std::sin(0.5 * theta[0]),
                 nullptr};
      sv_apply(sv, g);
    } else {
      sv_reset(sv, 0);
      std::vector<TGate> g = ansatz_tgates(kind, layers, sv->n_qubits);
      for (auto& t : g)
        if (t.param >= 0) {
          t.c = std::cos(0.5 * theta[t.param]);
          t.s = std::sin(0.5 * theta[t.param]);
          t.param = -1;
        }
      run_circuit_tiled(sv, g, nullptr);
    }
    VQF_CUDA(cudaStreamSynchronize(sv->stream));
  });
}

int vqf_energy(const double* theta, uint32_t n_theta, const vqf_hamiltonian* h, int32_t kind, uint32_t layers,
               int32_t device, double* out) {
  return vqf_energy_ex(theta, n_theta, h, kind, layers, device, VQF_F64, out);
}

int vqf_energy_ex(const double* theta, uint32_t n_theta, const vqf_hamiltonian* h, int32_t kind, uint32_t layers,
                  int32_t device, int32_t dtype, double* out) {
  return guarded([&] {
    if (h == nullptr || out == nullptr) throw_invalid("null argument");
    check_dtype(dtype, nullptr);
    const uint32_t P = ansatz_params(kind, layers, h->n_qubits);
    if (n_theta != P) throw_invalid("parameter count mismatch for ansatz");
    check_ansatz_register(kind, h->n_qubits);
    const CompiledHam ch = compile_hamiltonian(h);
    HbmEngine eng(h->n_qubits, kind, layers, 1, device, dtype);
    eng.prepare([&](uint32_t j, uint32_t) { return theta[j]; });
    double tot[2];
    sv_expectation(eng.sv, ch, tot);
    if (std::abs(tot[1]) >= 1e-10) throw_runtime(imag_msg(tot[1]));
    *out = tot[0];
  });
}

int vqf_gradient(const double* theta, uint32_t n_theta, const vqf_hamiltonian* h, int32_t kind, uint32_t layers,
                 int32_t method, int32_t device, double* grad_out) {
  return vqf_gradient_ex(theta, n_theta, h, kind, layers, method, device, VQF_F64, grad_out);
}

int vqf_gradient_ex(const double* theta, uint32_t n_theta, const vqf_hamiltonian* h, int32_t kind, uint32_t layers,
                    int32_t method, int32_t device, int32_t dtype, double* grad_out) {
  return guarded([&] {
    if (h == nullptr || grad_out == nullptr) throw_invalid("null argument");
    check_dtype(dtype, nullptr);
    const uint32_t P = ansatz_params(kind, layers, h->n_qubits);
    if (n_theta != P) throw_invalid("parameter count mismatch for ansatz");
    check_ansatz_register(kind, h->n_qubits);
    if (method != VQF_GRAD_PARAMETER_SHIFT && method != VQF_GRAD_ADJOINT) throw_invalid("unknown gradient method");
    const CompiledHam ch = compile_hamiltonian(h);
    std::vector<double> th(theta, theta + n_theta), E;
    if (method == VQF_GRAD_ADJOINT && AdjointPlan::supports(ch, h->n_qubits)) {
      AdjointRunner adj(h->n_qubits, kind, layers, device, ch, dtype);
      double e[2];
      adj.run(th, e, grad_out);
      // energy()'s check (statevector.hpp:244-247), as on the shift path
      if (std::abs(e[1]) >= 1e-10) throw_runtime(imag_msg(e[1]));
      return;
    }
    ShiftEvaluator ev(h->n_qubits, kind, layers, device, dtype);
    ev.run(th, ch, static_cast<int>(ev.NC), E);
    for (uint32_t c = 1; c < ev.NC; ++c)
      if (std::abs(E[2 * c + 1]) >= 1e-10) throw_runtime(imag_msg(E[2 * c + 1]));
    for (uint32_t k = 0; k < P; ++k) grad_out[k] = 0.5 * (E[2 * (2 * k + 1)] - E[2 * (2 * k + 2)]);
  });
}

int vqf_run_vqe(const vqf_hamiltonian* h, int32_t kind, uint32_t layers, const vqf_adam_config* config,
                const double* init, uint32_t n_init, int32_t method, int32_t device, vqf_vqe_result* result) {
  return guarded([&] { run_vqe_impl(h, kind, layers, config, init, n_init, method, device, result); });
}

int vqf_run_vqe_ex(const vqf_hamiltonian* h, int32_t kind, uint32_t layers, const vqf_adam_config* config,
                   const double* init, uint32_t n_init, int32_t method, int32_t device, int32_t dtype,
                   vqf_vqe_result* result) {
  return guarded([&] { run_vqe_impl(h, kind, layers, config, init, n_init, method, device, result, dtype); });
}

int vqf_run_vqe_batch(const vqf_hamiltonian* hs, uint32_t batch, int32_t kind, uint32_t layers,
                      const vqf_adam_config* config, int32_t device, vqf_vqe_result* results) {
  return guarded([&] {
    check_adam(config);
    if (batch == 0) return;
    if (hs == nullptr || results == nullptr) throw_invalid("null argument");
    const uint32_t n = hs[0].n_qubits;
    const uint32_t P = ansatz_params(kind, layers, n);
    check_ansatz_register(kind, n);
    for (uint32_t b = 1; b < batch; ++b)
      if (hs[b].n_qubits != n) throw_invalid("run_vqe_batch: all problems must share the register size");
    if (!small_ok(n, P)) {
      for (uint32_t b = 0; b < batch; ++b)
        run_vqe_impl(&hs[b], kind, layers, config, nullptr, 0, VQF_GRAD_PARAMETER_SHIFT, device, &results[b]);
      return;
    }
    const auto t0 = Clock::now();
    SmallJob j;
    j.batch = batch;
    j.n_qubits = static_cast<int32_t>(n);
    j.kind = kind;
    j.layers = static_cast<int32_t>(layers);
    j.P = P;
    j.adam = *config;
    j.term_off.push_back(0);
    for (uint32_t b = 0; b < batch; ++b) {
      const CompiledHam ch = compile_hamiltonian(&hs[b]);
      j.terms.insert(j.terms.end(), ch.terms.begin(), ch.terms.end());
      j.term_off.push_back(static_cast<uint32_t>(j.terms.size()));
    }
    run_small(j, device);
    for (uint32_t b = 0; b < batch; ++b)
      if (j.status[b] != kStatusOk) throw_runtime(small_error(j, b, 0.0));
    const double wall = seconds_since(t0);
    for (uint32_t b = 0; b < batch; ++b) {
      fill_result(j, b, &results[b]);
      results[b].wall_seconds = wall;
    }
  });
}

int vqf_pes_device_hamiltonians(const double* bonds, uint32_t n_bonds, int32_t device, uint32_t* n_terms,
                                int32_t* keys, double* coeffs, double* hf) {
  return guarded([&] {
    if (n_bonds == 0) return;
    if (bonds == nullptr || n_terms == nullptr || keys == nullptr || coeffs == nullptr || hf == nullptr)
      throw_invalid("null argument");
    for (uint32_t b = 0; b < n_bonds; ++b) chem::check_bond(bonds[b]);
    SmallJob j;
    j.batch = n_bonds;
    j.n_qubits = 4;
    j.kind = VQF_ANSATZ_H2_DOUBLE_EXCITATION;
    j.P = 1;
    j.adam = vqf_adam_config{0.01, 0.9, 0.999, 1e-8, 1, 0, 0.0};
    j.pes = true;
    j.want_ham = true;
    j.bonds.assign(bonds, bonds + n_bonds);
    j.status_in.assign(n_bonds, 0);
    run_small(j, device, false);
    for (uint32_t b = 0; b < n_bonds; ++b) {
      if (j.status[b] != kStatusOk) throw_runtime(small_error(j, b, bonds[b]));
      n_terms[b] = static_cast<uint32_t>(j.ham_count[b]);
      for (int t = 0; t < 16; ++t) {
        keys[16 * b + t] = t < j.ham_count[b] ? j.ham_keys[16 * b + t] : 0;
        coeffs[16 * b + t] = t < j.ham_count[b] ? j.ham_coeffs[16 * b + t] : 0.0;
      }
      for (int k = 0; k < 4; ++k) hf[4 * b + k] = j.hf[4 * b + k];
    }
  });
}

int vqf_run_sweep(const vqf_sweep_config* cfg, vqf_sweep_report* rep) {
  return guarded([&] {
    if (cfg == nullptr || rep == nullptr) throw_invalid("null argument");
    if (cfg->workers < 1) throw_invalid("workers must be >= 1");  // sweep.hpp:129
    const auto start = Clock::now();
    HMARK("enter");
    const SweepSlice sl = sweep_slice(*cfg);
    const int W = cfg->workers;
    std::vector<uint64_t> wbe(2 * (size_t)W);
    host::split_chunks(sl.hi - sl.lo, W, wbe.data());
    const std::vector<int32_t> devices = sweep_devices(*cfg);

    std::vector<std::string> errors(sl.grid.size());
    std::vector<double> dev_secs(W, 0.0);
    std::vector<size_t> h2d(W, 0), d2h(W, 0);
    std::vector<std::exception_ptr> fails(W);
    auto worker = [&](int w) {
      try {
        const auto tw = Clock::now();
        const uint64_t b0 = sl.lo + wbe[2 * w], b1 = sl.lo + wbe[2 * w + 1];
        SmallJob j = pes_job(*cfg, sl.grid, b0, b1, errors);
        j.grid_n = cfg->n_points;  // bonds generated on the device (grid mode)
        j.grid_first = static_cast<int32_t>(b0);
        j.grid_min = cfg->d_min;
        j.grid_max = cfg->d_max;
        if (j.batch > 0) {
          run_small(j, devices[w % devices.size()], rep->trajectories != nullptr, &h2d[w], &d2h[w]);
          dev_secs[w] = j.device_seconds;
        }
        pes_fill(j, *cfg, sl.grid, b0, b1, errors, rep);
        if (rep->per_worker_seconds) rep->per_worker_seconds[w] = seconds_since(tw);
      } catch (...) {
        fails[w] = std::current_exception();
      }
    };
    if (W == 1) {
      worker(0);
    } else {
      std::vector<std::thread> pool;
      pool.reserve(W);
      for (int w = 0; w < W; ++w) pool.emplace_back(worker, w);
      for (auto& t : pool) t.join();
    }
    for (auto& f : fails)
      if (f) std::rethrow_exception(f);
    HMARK("fill");
    pes_finish(sl, errors, rep);
    HMARK("finish");
    HDUMP();
    rep->device_seconds = *std::max_element(dev_secs.begin(), dev_secs.end());
    rep->h2d_bytes = 0;
    rep->d2h_bytes = 0;
    for (int w = 0; w < W; ++w) {
      rep->h2d_bytes += h2d[w];
      rep->d2h_bytes += d2h[w];
    }
    rep->total_wall_seconds = seconds_since(start);
  });
}

int vqf_pes_create(const vqf_sweep_config* cfg, int32_t device, vqf_pes* out) {
  return guarded([&] {
    if (cfg == nullptr || out == nullptr) throw_invalid("null argument");
    auto plan = std::make_unique<vqf_pes_plan>();
    plan->cfg = *cfg;
    plan->cfg.devices = nullptr;
    plan->device = device;
    plan->slice = sweep_slice(*cfg);
    plan->errors.assign(plan->slice.grid.size(), std::string());
    plan->job = pes_job(*cfg, plan->slice.grid, plan->slice.lo, plan->slice.hi, plan->errors);
    plan->stage = std::make_unique<SmallStage>(plan->job);
    VQF_CUDA(cudaSetDevice(device));
    VQF_CUDA(cudaStreamCreateWithFlags(&plan->stream, cudaStreamNonBlocking));
    VQF_CUDA(cudaMalloc(&plan->dev, std::max<size_t>(plan->stage->total, 16)));
    VQF_CUDA(cudaMallocHost(&plan->pin, std::max<size_t>(plan->stage->total, 16)));
    plan->stage->pack(plan->job, static_cast<unsigned char*>(plan->pin));
    plan->params = plan->stage->params(plan->job, static_cast<unsigned char*>(plan->dev), device);
    VQF_CUDA(cudaMemcpyAsync(plan->dev, plan->pin, plan->stage->in_end, cudaMemcpyHostToDevice, plan->stream));
    VQF_CUDA(cudaStreamSynchronize(plan->stream));
    *out = plan.release();
  });
}

int vqf_pes_launch(vqf_pes plan, void* stream) {
  return guarded([&] {
    if (plan == nullptr) throw_invalid("null plan");
    if (plan->job.batch == 0) return;
    VQF_CUDA(cudaSetDevice(plan->device));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : plan->stream;
    launch_vqe_small(plan->params, plan->job.batch, true, s);
    plan->last_stream = s;
  });
}

int vqf_pes_read(vqf_pes plan, vqf_sweep_report* rep) {
  return guarded([&] {
    if (plan == nullptr || rep == nullptr) throw_invalid("null argument");
    VQF_CUDA(cudaSetDevice(plan->device));
    auto* pin = static_cast<unsigned char*>(plan->pin);
    auto* dev = static_cast<unsigned char*>(plan->dev);
    const SmallStage& st = *plan->stage;
    const bool traj = rep->trajectories != nullptr;
    cudaStream_t s = plan->last_stream ? plan->last_stream : plan->stream;
    if (plan->job.batch > 0) {
      VQF_CUDA(cudaMemcpyAsync(pin + st.o_status, dev + st.o_status, st.d2h_bytes(traj), cudaMemcpyDeviceToHost, s));
      VQF_CUDA(cudaStreamSynchronize(s));
      st.unpack(plan->job, pin, traj);
    }
    std::vector<std::string> errors = plan->errors;
    pes_fill(plan->job, plan->cfg, plan->slice.grid, plan->slice.lo, plan->slice.hi, errors, rep);
    pes_finish(plan->slice, errors, rep);
    rep->h2d_bytes = 0;
    rep->d2h_bytes = plan->job.batch > 0 ? st.d2h_bytes(traj) : 0;
  });
}

int vqf_pes_destroy(vqf_pes plan) {
  return guarded([&] {
    if (plan == nullptr) return;
    cudaSetDevice(plan->device);
    if (plan->stream) cudaStreamSynchronize(plan->stream);
    if (plan->dev) cudaFree(plan->dev);
    if (plan->pin) cudaFreeHost(plan->pin);
    if (plan->stream) cudaStreamDestroy(plan->stream);
    delete plan;
  });
}

int vqf_run_scaling_study(const vqf_scaling_config* cfg, vqf_scaling_record* records) {
  return guarded([&] {
    if (cfg == nullptr || records == nullptr) throw_invalid("null argument");
    for (uint32_t i = 0; i < cfg->n_widths; ++i) {  // sweep.hpp:267-275
      const uint32_t n = cfg->qubits[i];
      if (n < 2) throw_invalid("scaling study needs >= 2 qubits");
      if (n > 26 && !cfg->force)
        throw_invalid("refusing " + std::to_string(n) + " qubits (> 26, state alone exceeds 1 GiB); pass force to override");
    }
    for (uint32_t i = 0; i < cfg->n_widths; ++i) {
      const uint32_t n = cfg->qubits[i];
      if (n > 22)
        std::cerr << "warning: " << n << " qubits needs " << vqf_memory_estimate(n) / (1024.0 * 1024.0 * 1024.0)
                  << " GiB of state\n";
      const auto terms = cfg->z_sum_mode ? host::build_z_sum(n) : host::build_tfim(n, cfg->coupling, cfg->field);
      std::vector<double> coeffs(2 * terms.size());
      std::vector<uint32_t> offs(terms.size() + 1), qs;
      std::vector<uint8_t> ax;
      for (size_t t = 0; t < terms.size(); ++t) {
        coeffs[2 * t] = terms[t].coeff.real();
        coeffs[2 * t + 1] = terms[t].coeff.imag();
        for (const auto& [q, a] : terms[t].axes) {
          qs.push_back(q);
          ax.push_back(a);
        }
        offs[t + 1] = static_cast<uint32_t>(qs.size());
      }
      vqf_hamiltonian h{n, static_cast<uint32_t>(terms.size()), coeffs.data(), offs.data(), qs.data(), ax.data()};
      vqf_adam_config adam{0.01, 0.9, 0.999, 1e-8, 200, 0, 0.0};
      adam.learning_rate = cfg->learning_rate;
      adam.max_iterations = cfg->iterations;
      const uint32_t P = cfg->layers * n;
      std::vector<double> init(P, cfg->theta_init), theta(P);
      vqf_vqe_result r{};
      r.theta = theta.data();
      const auto t0 = Clock::now();
      run_vqe_impl(&h, VQF_ANSATZ_HARDWARE_EFFICIENT, cfg->layers, &adam, init.data(), P, cfg->gradient_method,
                   cfg->device, &r, cfg->dtype);
      records[i].n_qubits = n;
      records[i].state_bytes = vqf_memory_estimate(n) / (cfg->dtype == VQF_F32 ? 2 : 1);
      records[i].runtime_seconds = seconds_since(t0);
      records[i].final_energy = r.energy;
      records[i].iterations_run = r.iterations_run;
    }
  });
}

}  // extern "C"
