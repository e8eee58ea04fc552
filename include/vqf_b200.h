/*
 * vqf_b200.h — C ABI of the B200-native VQE state-vector engine
 * (libvqf_b200.so, built from paper_2601_09951_b200/csrc for sm_100a).
 *
 * This is the drop-in boundary for the reference VQE Forge hot path
 * (/root/reference/proj/include/vqeforge).  The reference exposes no FFI:
 * its boundary is the header-only C++ API in namespace vqeforge.  Each entry
 * point below names the reference function it replaces (file:line); the C++
 * drop-in headers in include/vqeforge_b200/ rebuild that exact API on top of
 * these calls.
 *
 * Conventions
 *  - Plain C types, caller-owned buffers, no torch types.
 *  - Every int-returning call returns VQF_OK (0) or an error class that the
 *    C++ wrapper maps back onto the reference's exception types
 *    (SURVEY.md §8b "Error conventions"):
 *        VQF_INVALID_ARGUMENT -> std::invalid_argument
 *        VQF_RUNTIME_ERROR    -> std::runtime_error
 *        VQF_LOGIC_ERROR      -> std::logic_error
 *        VQF_DOMAIN_ERROR     -> std::domain_error (BondLengthOutOfRange)
 *        VQF_CUDA_ERROR       -> std::runtime_error ("CUDA: ...")
 *    vqf_last_error() returns the message of the calling thread's last
 *    failure (the reference's e.what() text, byte for byte where the
 *    reference defines it).
 *  - Qubit 0 is the MOST significant bit of the basis index
 *    (pauli.hpp:223-227).  Amplitudes cross the boundary as interleaved
 *    (re, im) doubles, index-ordered, one state after another for a batch.
 *  - Hamiltonians cross the boundary in sparse CSR form mirroring
 *    PauliTerm/QubitHamiltonian (pauli.hpp:65-129).
 *  - Thread safety: distinct handles may be used from distinct threads
 *    concurrently; one handle is used by one thread at a time.
 */
#ifndef VQF_B200_H
#define VQF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VQF_ABI_VERSION 1

enum {
  VQF_OK = 0,
  VQF_INVALID_ARGUMENT = 1,
  VQF_RUNTIME_ERROR = 2,
  VQF_LOGIC_ERROR = 3,
  VQF_DOMAIN_ERROR = 4,
  VQF_CUDA_ERROR = 5
};

/* PauliAxis (pauli.hpp:34): I is never stored inside a term. */
enum { VQF_AXIS_X = 1, VQF_AXIS_Y = 2, VQF_AXIS_Z = 3 };

/* GateKind (statevector.hpp:76) plus SingleExcitation (Givens on 2 wires,
 * |10> <-> |01>, same sign convention as DoubleExcitation). */
enum {
  VQF_GATE_PAULI_X = 0,
  VQF_GATE_RY = 1,
  VQF_GATE_CNOT = 2,
  VQF_GATE_DOUBLE_EXCITATION = 3,
  VQF_GATE_SINGLE_EXCITATION = 4
};

/* AnsatzKind (vqe.hpp:32-40). */
enum { VQF_ANSATZ_H2_DOUBLE_EXCITATION = 0, VQF_ANSATZ_HARDWARE_EFFICIENT = 1 };

/* Storage precision of a state vector. */
enum { VQF_F64 = 0, VQF_F32 = 1 };

/* Gradient rule: the reference's two-term parameter shift (vqe.hpp:112-127)
 * or the adjoint method (one forward + one backward sweep). */
enum { VQF_GRAD_PARAMETER_SHIFT = 0, VQF_GRAD_ADJOINT = 1 };

/* QubitHamiltonian (pauli.hpp:116-129) in CSR form. */
typedef struct vqf_hamiltonian {
  uint32_t n_qubits;
  uint32_t n_terms;
  const double* coeffs;    /* 2*n_terms: (re, im) per term */
  const uint32_t* offsets; /* n_terms + 1 */
  const uint32_t* qubits;  /* offsets[n_terms], sorted ascending per term */
  const uint8_t* axes;     /* offsets[n_terms], VQF_AXIS_* */
} vqf_hamiltonian;

/* Output buffer for Hamiltonian builders; capacities are checked. */
typedef struct vqf_hamiltonian_out {
  uint32_t n_terms; /* written */
  double* coeffs;
  uint32_t* offsets;
  uint32_t* qubits;
  uint8_t* axes;
  uint32_t cap_terms;
  uint32_t cap_axes;
} vqf_hamiltonian_out;

/* Gate (statevector.hpp:82-101). */
typedef struct vqf_gate {
  int32_t kind;
  uint32_t n_wires;
  uint32_t wires[4];
  double angle;
} vqf_gate;

/* AdamConfig (vqe.hpp:129-138). */
typedef struct vqf_adam_config {
  double learning_rate; /* 0.01 */
  double beta1;         /* 0.9 */
  double beta2;         /* 0.999 */
  double epsilon;       /* 1e-8 */
  int32_t max_iterations; /* 200 */
  int32_t has_gradient_tolerance;
  double gradient_tolerance;
} vqf_adam_config;

/* VqeResult (vqe.hpp:176-186).  theta (P) and trajectory
 * (trajectory_capacity >= max_iterations + 1) are caller-owned. */
typedef struct vqf_vqe_result {
  double energy;
  double* theta;
  double* trajectory;
  uint32_t trajectory_capacity;
  uint32_t trajectory_len; /* written: iterations_run + 1 */
  int32_t iterations_run;
  uint64_t circuit_evaluations;
  double wall_seconds;
} vqf_vqe_result;

/* SweepConfig (sweep.hpp:40-46) + device placement.
 * workers: number of parallel workers = devices used (one host thread and
 *   one CUDA stream per worker; worker w runs split_chunks(n_points,
 *   workers)[w] on devices[w % n_devices]).
 * chunk_index / n_chunks: when n_chunks > 1 only that split_chunks slice of
 *   the global grid is computed (one rank per GPU under torchrun); points
 *   outside it are left untouched.  Grid values and per-point results are
 *   bitwise independent of workers / n_chunks (test_sweep.cpp:101-129). */
typedef struct vqf_sweep_config {
  double d_min;     /* 0.1 angstrom */
  double d_max;     /* 3.0 angstrom */
  int32_t n_points; /* 100 */
  int32_t workers;  /* 1 */
  vqf_adam_config adam;
  const int32_t* devices; /* NULL => device 0.. */
  int32_t n_devices;      /* 0 => all visible devices */
  int32_t chunk_index;
  int32_t n_chunks; /* 0 or 1 => whole grid */
} vqf_sweep_config;

/* SweepReport (sweep.hpp:48-64); arrays sized n_points, caller-owned.
 * trajectories (optional, may be NULL): n_points * (max_iterations + 1)
 * doubles, row i = the VqeResult.trajectory of point i (NaN-padded).
 * errors (optional): n_points * error_stride chars. */
typedef struct vqf_sweep_report {
  double* bond_angstrom;
  double* energy_hartree;
  double* theta_star; /* one parameter per point (H2 ansatz) */
  int32_t* iterations;
  double* wall_seconds;
  int32_t* ok;
  char* errors;
  size_t error_stride;
  double* trajectories;
  double* per_worker_seconds; /* workers entries */
  double total_wall_seconds;  /* written */
  int32_t all_ok;             /* written */
  double device_seconds;      /* written: max over workers of the on-device time */
  uint64_t h2d_bytes;         /* written: host->device bytes moved by the call */
  uint64_t d2h_bytes;         /* written: device->host bytes moved by the call */
} vqf_sweep_report;

/* ScalingConfig (sweep.hpp:237-249) / ScalingRecord (:251-257). */
typedef struct vqf_scaling_config {
  const uint32_t* qubits;
  uint32_t n_widths;
  uint32_t layers;    /* 2 */
  int32_t iterations; /* 5 */
  double learning_rate; /* 0.05 */
  double coupling;      /* 1.0 */
  double field;         /* 1.0 */
  int32_t z_sum_mode;
  double theta_init; /* 0.1 */
  int32_t force;
  int32_t gradient_method; /* VQF_GRAD_* ; reference = parameter shift */
  int32_t device;
  int32_t dtype; /* VQF_F64 (reference precision) or VQF_F32 (complex64 states) */
} vqf_scaling_config;

typedef struct vqf_scaling_record {
  uint32_t n_qubits;
  uint64_t state_bytes;
  double runtime_seconds;
  double final_energy;
  int32_t iterations_run;
} vqf_scaling_record;

/* Device-resident PES plan: the inputs of one run_sweep slice (bond grid,
 * Adam bias tables; workers ignored, chunk_index / n_chunks honoured) staged
 * in HBM once.  vqf_pes_launch enqueues ONLY the fused chemistry + VQE kernel
 * on the caller's CUDA stream (NULL = the plan's own), with no host copies,
 * so throughput can be timed with inputs resident; vqf_pes_read copies the
 * results back and fills the report exactly as vqf_run_sweep would. */
typedef struct vqf_pes_plan* vqf_pes;

/* Opaque device-resident batch of state vectors (StateVector,
 * statevector.hpp:33-51, batched: `batch` independent states). */
typedef struct vqf_statevector* vqf_sv;

/* ---------------------------------------------------------------- runtime */
const char* vqf_version(void);
const char* vqf_last_error(void);
int vqf_device_count(int32_t* out);
/* Creates the CUDA context + stream pools on `device` (call outside timed
 * regions; the reference has no equivalent). */
int vqf_init(int32_t device);
/* Number of engine kernels launched by this process so far (all devices). */
uint64_t vqf_kernel_launches(void);

/* ------------------------------------------- host-only (no GPU needed) */
/* statevector.hpp:55-57 memory_estimate (x16 B per amplitude). */
uint64_t vqf_memory_estimate(uint32_t n_qubits);
/* vqe.hpp:54-62 n_parameters; returns 0 for an unknown kind. */
uint32_t vqf_n_parameters(int32_t ansatz_kind, uint32_t layers, uint32_t n_qubits);
/* sweep.hpp:68-85 bond_grid; out holds n_points doubles. */
int vqf_bond_grid(double d_min, double d_max, int32_t n_points, double* out);
/* sweep.hpp:93-107 split_chunks; begin_end holds 2*n_chunks entries. */
int vqf_split_chunks(uint64_t n_items, uint64_t n_chunks, uint64_t* begin_end);
/* sweep.hpp:111-119 effective_workers (VQE_FORGE_THREADS cap). */
int vqf_effective_workers(int32_t requested, int32_t* out);
/* vqe.hpp:152-174 adam_step (pure). */
int vqf_adam_step(const double* m, const double* v, int64_t step, const double* grad,
                  const double* theta, uint32_t n, const vqf_adam_config* config,
                  double* theta_out, double* m_out, double* v_out, int64_t* step_out);
/* pauli.hpp:180-201 canonicalize. */
int vqf_canonicalize(const vqf_hamiltonian* h, vqf_hamiltonian_out* out);
/* chem.hpp:473-482 build_h2_hamiltonian (STO-3G RHF + Jordan-Wigner), host. */
int vqf_build_h2_hamiltonian(double bond_angstrom, vqf_hamiltonian_out* out);
/* chem.hpp:280 run_hartree_fock summary: {hf_energy, electronic, nuclear,
 * scf_iterations}. */
int vqf_hartree_fock(double bond_angstrom, double* out4);
/* sweep.hpp:209-223 build_tfim, :227-235 build_z_sum. */
int vqf_build_tfim(uint32_t n_qubits, double coupling, double field, vqf_hamiltonian_out* out);
int vqf_build_z_sum(uint32_t n_qubits, vqf_hamiltonian_out* out);

/* ------------------------------------------------------ state vectors */
/* StateVector(n) ctor (statevector.hpp:39-42) for each of `batch` states. */
int vqf_sv_create(uint32_t n_qubits, uint32_t batch, int32_t dtype, int32_t device, vqf_sv* out);
int vqf_sv_destroy(vqf_sv sv);
int vqf_sv_info(vqf_sv sv, uint32_t* n_qubits, uint32_t* batch, int32_t* dtype, int32_t* device);
/* Routes all subsequent work on sv to the caller's cudaStream_t (NULL
 * restores the handle's own stream).  Calls still synchronise that stream
 * before returning host results. */
int vqf_sv_set_stream(vqf_sv sv, void* cuda_stream);
/* |0...0> (statevector.hpp:39-42). */
int vqf_sv_reset(vqf_sv sv);
/* basis_state (statevector.hpp:61-74), same bits for every batch entry. */
int vqf_sv_set_basis_state(vqf_sv sv, const int32_t* bits, uint32_t n_bits);
/* Host <-> device copies of all batch*2^n amplitudes (interleaved re, im
 * doubles; converted on the fly for VQF_F32). */
int vqf_sv_upload(vqf_sv sv, const double* amps);
int vqf_sv_download(vqf_sv sv, double* amps);
/* StateVector::norm (statevector.hpp:46-50) per batch entry. */
int vqf_sv_norm(vqf_sv sv, double* out);
/* apply_gate (statevector.hpp:148-203) / apply_circuit (:205-207) on every
 * batch entry. */
int vqf_apply_gate(vqf_sv sv, const vqf_gate* gate);
int vqf_apply_circuit(vqf_sv sv, const vqf_gate* gates, uint32_t n_gates);
/* expectation (statevector.hpp:217-249) per batch entry; throws (returns
 * VQF_RUNTIME_ERROR) on an imaginary residue >= 1e-10 in any entry. */
int vqf_expectation(vqf_sv sv, const vqf_hamiltonian* h, double* out);
/* Same sum without the residue check, as interleaved (re, im) per entry:
 * the per-shard partial of a distributed expectation (the check applies to
 * the all-reduced total). */
int vqf_expectation_complex(vqf_sv sv, const vqf_hamiltonian* h, double* out);
/* sum_t c_t (-i)^{n_y} sum_i (-1)^popc(i & yz_t) conj(a_i) b_{i ^ flip_t} for
 * two states of one register (batch entry 0), as (re, im): the shard-pair
 * term of a distributed expectation whose Pauli string flips global wires. */
int vqf_cross_expectation(vqf_sv a, vqf_sv b, const vqf_hamiltonian* h, double* out);
/* How vqf_apply_circuit would run `gates` on an n-qubit state of `dtype`
 * (host only, no device work): passes = HBM passes over the state (fused
 * shared-memory tile passes + single-gate launches), fused_ops = register
 * ops inside those passes (each one shared-memory round trip of a tile). */
int vqf_circuit_plan(uint32_t n_qubits, int32_t dtype, const vqf_gate* gates, uint32_t n_gates, uint32_t* passes,
                     uint32_t* fused_ops);
/* How vqf_expectation reads the state for h (host only, no device work):
 * state_passes = HBM passes over the state (diagonal pass + one per
 * multi-group pass + one per remaining flip group), flip_groups = distinct
 * non-zero flip masks (the reference's per-group pass count, minus the
 * diagonal), multi_passes = register-resident passes that serve several
 * flip groups each.  Any out pointer may be NULL. */
int vqf_expectation_plan(const vqf_hamiltonian* h, uint32_t* state_passes, uint32_t* flip_groups,
                         uint32_t* multi_passes);
/* The same for a state of the given dtype (VQF_F64 / VQF_F32: the tile
 * geometry and the folding of the diagonal group differ); the plain call
 * plans for VQF_F64. */
int vqf_expectation_plan_ex(const vqf_hamiltonian* h, int32_t dtype, uint32_t* state_passes, uint32_t* flip_groups,
                            uint32_t* multi_passes);
/* Raw device address and byte size of the amplitudes (for exchanging
 * shards with NCCL / peer copies; the handle keeps ownership). */
int vqf_sv_device_ptr(vqf_sv sv, void** ptr, uint64_t* bytes);

/* ---------------------------------------------------------------- VQE */
/* prepare_ansatz (vqe.hpp:65-96) into every batch entry of sv. */
int vqf_prepare_ansatz(int32_t ansatz_kind, uint32_t layers, const double* theta,
                       uint32_t n_theta, vqf_sv sv);
/* energy (vqe.hpp:99-104), on `device`. */
int vqf_energy(const double* theta, uint32_t n_theta, const vqf_hamiltonian* h,
               int32_t ansatz_kind, uint32_t layers, int32_t device, double* out);
/* gradient (vqe.hpp:112-127); method VQF_GRAD_*. */
int vqf_gradient(const double* theta, uint32_t n_theta, const vqf_hamiltonian* h,
                 int32_t ansatz_kind, uint32_t layers, int32_t method, int32_t device,
                 double* grad_out);
/* run_vqe (vqe.hpp:194-254).  init may be NULL/n_init 0 (theta0 = 0). */
int vqf_run_vqe(const vqf_hamiltonian* h, int32_t ansatz_kind, uint32_t layers,
                const vqf_adam_config* config, const double* init, uint32_t n_init,
                int32_t gradient_method, int32_t device, vqf_vqe_result* result);
/* The same three with the state precision: VQF_F64 (the reference's
 * complex128; what the entry points above use) or VQF_F32 (complex64 states,
 * fp64 angles / reductions / Adam; energies within 1e-5 of fp64).  fp32
 * run_vqe is fixed-iteration only (a gradient tolerance -> invalid_argument). */
int vqf_energy_ex(const double* theta, uint32_t n_theta, const vqf_hamiltonian* h,
                  int32_t ansatz_kind, uint32_t layers, int32_t device, int32_t dtype, double* out);
int vqf_gradient_ex(const double* theta, uint32_t n_theta, const vqf_hamiltonian* h,
                    int32_t ansatz_kind, uint32_t layers, int32_t method, int32_t device,
                    int32_t dtype, double* grad_out);
int vqf_run_vqe_ex(const vqf_hamiltonian* h, int32_t ansatz_kind, uint32_t layers,
                   const vqf_adam_config* config, const double* init, uint32_t n_init,
                   int32_t gradient_method, int32_t device, int32_t dtype, vqf_vqe_result* result);
/* Batched run_vqe: `batch` independent problems with the same ansatz and
 * register size, one on-device optimisation loop each, one launch. */
int vqf_run_vqe_batch(const vqf_hamiltonian* hs, uint32_t batch, int32_t ansatz_kind,
                      uint32_t layers, const vqf_adam_config* config, int32_t device,
                      vqf_vqe_result* results);

/* -------------------------------------------------------------- sweep */
/* run_sweep (sweep.hpp:128-178): H2 PES, Hartree-Fock + Jordan-Wigner and
 * the Adam loop for every bond on the GPU in one fused launch per worker. */
int vqf_run_sweep(const vqf_sweep_config* config, vqf_sweep_report* report);
int vqf_pes_create(const vqf_sweep_config* config, int32_t device, vqf_pes* out);
int vqf_pes_launch(vqf_pes plan, void* cuda_stream);
int vqf_pes_read(vqf_pes plan, vqf_sweep_report* report);
int vqf_pes_destroy(vqf_pes plan);

/* Diagnostic view of the PES kernel's on-device chemistry (chem.hpp:280-482
 * run_hartree_fock + jordan_wigner, built inside the fused kernel): for each
 * bond, the Hamiltonian the optimisation uses, as up to 16 terms.  Term t of
 * bond b: keys[16b + t] encodes the Pauli string with bit q = X on qubit q
 * and bit 4 + q = Z on qubit q (both set = Y); coeffs[16b + t] its (real)
 * coefficient; n_terms[b] the count (0 when the point failed).  hf[4b..4b+3]
 * = {hf_energy, electronic, nuclear_repulsion, scf_iterations}.  Bonds
 * outside chem.hpp's range fail with the BondLengthOutOfRange text. */
int vqf_pes_device_hamiltonians(const double* bonds, uint32_t n_bonds, int32_t device, uint32_t* n_terms,
                                int32_t* keys, double* coeffs, double* hf);
/* run_scaling_study (sweep.hpp:265-307). records holds n_widths entries. */
int vqf_run_scaling_study(const vqf_scaling_config* config, vqf_scaling_record* records);

/* ---------------------------------------------- distributed state vector
 * BASELINE config 5 (34-35 qubits over 8 B200).  An n-qubit state is split
 * over world = 2^g shards of 2^(n-g) amplitudes.  Every qubit sits at a
 * POSITION: positions 0..g-1 are global (position p = rank bit g-1-p),
 * positions g..n-1 are local (position p = local index bit n-1-p of every
 * shard, i.e. engine wire p-g).  The layout qubit -> position starts as the
 * identity and changes lazily: a gate or Pauli string that needs a global
 * qubit local swaps it with a local position (each rank exchanges the half
 * of its shard whose local bit differs from its own rank bit with
 * rank ^ (1 << (g-1-p))) and KEEPS the new layout (no swap back).  Circuit
 * plans evict the local qubit whose next use lies furthest ahead.
 * Shards live either all in this process on one device (comm == NULL:
 * virtual ranks, exchanges are in-place device swaps) or one per process
 * (comm set): exchanges go through comm->sendrecv in chunk_bytes pieces
 * staged through two preallocated device buffers (peak memory = shard +
 * 2 chunks), the expectation's totals through comm->allreduce_sum.
 * Reference: none (the reference caps run_scaling_study at 26 qubits,
 * sweep.hpp:36-38, 267-283); per shard the engine runs the reference's
 * apply_gate / expectation semantics (statevector.hpp:148-249). */
typedef struct vqf_dsv_comm {
  int32_t rank; /* the shard this process holds */
  /* send `bytes` device bytes at send_buf to `peer` and receive as many
   * from it into recv_buf, ordered on cuda_stream (or synchronous);
   * returns 0 on success */
  int (*sendrecv)(void* user, const void* send_buf, void* recv_buf, uint64_t bytes, int32_t peer,
                  void* cuda_stream);
  /* in-place sum of `count` host doubles over all ranks; 0 on success */
  int (*allreduce_sum)(void* user, double* values, uint32_t count);
  void* user;
} vqf_dsv_comm;

typedef struct vqf_dsv_state* vqf_dsv;

/* One step of a distributed plan.
 *  VQF_DSV_SWAP : a = global position, b = local position.
 *  VQF_DSV_LOCAL: gates [first, first + count) of the mapped gate list, on
 *                 every shard (wires are engine wires of the shard).
 *  VQF_DSV_EVAL : planned terms [first, first + count): per-shard
 *                 expectation (no global flips).
 *  VQF_DSV_CROSS: planned terms [first, first + count): rank r pairs with
 *                 rank r ^ a (terms flipping global positions that cannot be
 *                 swapped local).  */
enum { VQF_DSV_SWAP = 0, VQF_DSV_LOCAL = 1, VQF_DSV_EVAL = 2, VQF_DSV_CROSS = 3 };
typedef struct vqf_dsv_op {
  int32_t kind;
  uint32_t a, b;
  uint32_t first, count;
} vqf_dsv_op;

/* A Pauli term of the Hamiltonian under the layout at its evaluation:
 * on rank r it contributes
 *   coeff * (-i)^(l_ny + g_ny) * (-1)^popc(r & g_yz)
 *   * sum_l conj(psi_r[l]) (-1)^popc(l & l_yz) psi_{r ^ g_flip}[l ^ l_flip]. */
typedef struct vqf_dsv_term {
  uint32_t term;   /* index into the Hamiltonian */
  uint32_t g_flip; /* rank-bit mask of global X/Y */
  uint32_t g_yz;   /* rank-bit mask of global Y/Z */
  uint32_t g_ny;
  uint64_t l_flip; /* local index bits of local X/Y */
  uint64_t l_yz;   /* local index bits of local Y/Z */
  uint32_t l_ny;
  uint32_t pad;
} vqf_dsv_term;

/* Host-only planners (no GPU): position_of_qubit (n entries) is read and
 * updated; gates / terms are planned against it.  mapped_gates holds
 * n_gates entries, terms_out one entry per Hamiltonian term. */
int vqf_dsv_plan_circuit(uint32_t n_qubits, uint32_t world, uint32_t* position_of_qubit, const vqf_gate* gates,
                         uint32_t n_gates, vqf_dsv_op* ops, uint32_t cap_ops, uint32_t* n_ops,
                         vqf_gate* mapped_gates);
int vqf_dsv_plan_expectation(uint32_t n_qubits, uint32_t world, uint32_t* position_of_qubit,
                             const vqf_hamiltonian* h, vqf_dsv_op* ops, uint32_t cap_ops, uint32_t* n_ops,
                             vqf_dsv_term* terms_out);
/* Per-GPU bytes: one shard + the two exchange buffers (comm mode). */
uint64_t vqf_dsv_memory_per_gpu(uint32_t n_qubits, uint32_t world, int32_t dtype, uint64_t chunk_bytes,
                                int32_t one_shard_per_process);

/* chunk_bytes: exchange piece (0 = 256 MiB); comm NULL = virtual ranks. */
int vqf_dsv_create(uint32_t n_qubits, uint32_t world, int32_t dtype, int32_t device, const vqf_dsv_comm* comm,
                   uint64_t chunk_bytes, vqf_dsv* out);
int vqf_dsv_destroy(vqf_dsv d);
/* apply_circuit (statevector.hpp:205-207) on the distributed state. */
int vqf_dsv_apply_circuit(vqf_dsv d, const vqf_gate* gates, uint32_t n_gates);
/* expectation (statevector.hpp:217-249): the summed total; imaginary
 * residue >= 1e-10 -> VQF_RUNTIME_ERROR with the reference's message. */
int vqf_dsv_expectation(vqf_dsv d, const vqf_hamiltonian* h, double* out);
int vqf_dsv_layout(vqf_dsv d, uint32_t* position_of_qubit);
/* A shard held by this process in physical (local index) order. */
int vqf_dsv_shard_download(vqf_dsv d, uint32_t rank, double* amps);
int vqf_dsv_shard_upload(vqf_dsv d, uint32_t rank, const double* amps);
int vqf_dsv_stats(vqf_dsv d, uint64_t* swaps, uint64_t* bytes_sent, uint64_t* scratch_bytes);

#ifdef __cplusplus
}
#endif
#endif /* VQF_B200_H */
