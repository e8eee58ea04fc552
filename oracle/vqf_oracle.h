/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle restatement of the reference VQE
 * Forge hot path.  See vqf_oracle.c for the citation map and parity pin.
 */
#ifndef VQF_ORACLE_H
#define VQF_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAX_AXES 64

/* Sparse CSR Hamiltonian mirroring QubitHamiltonian (pauli.hpp:116-129). */
typedef struct {
  uint32_t n_qubits, n_terms;
  const double* coeffs;     /* 2*n_terms (re, im) */
  const uint32_t* offsets;  /* n_terms + 1 */
  const uint32_t* qubits;   /* offsets[n_terms] */
  const uint8_t* axes;      /* 1 X, 2 Y, 3 Z */
} orc_ham;

typedef struct {
  uint32_t* n_terms;
  double* coeffs;
  uint32_t* offsets;
  uint32_t* qubits;
  uint8_t* axes;
  uint32_t cap_terms, cap_axes;
} orc_ham_out;

/* ORC_SE: SingleExcitation, the engine's appended kind (not in the
 * reference's GateKind): the Givens rotation of statevector.hpp:179-200
 * restricted to two wires, |10> -> c|10> + s|01>, |01> -> c|01> - s|10>. */
enum { ORC_X = 0, ORC_RY = 1, ORC_CNOT = 2, ORC_DE = 3, ORC_SE = 4 };

typedef struct {
  int kind;
  double angle;
  uint32_t n_wires;
  uint32_t wires[4];
} orc_gate;

typedef struct {
  double learning_rate, beta1, beta2, epsilon;
  int max_iterations;
  int has_tolerance;
  double gradient_tolerance;
} orc_adam;

typedef struct {
  double energy;
  double* theta;      /* caller-owned, P */
  double* trajectory; /* caller-owned, max_iterations + 1 */
  uint32_t traj_len;
  int iterations_run;
  uint64_t circuit_evaluations;
} orc_vqe_result;

int orc_canonicalize(const orc_ham* h, orc_ham_out* out, char* err, size_t cap);
int orc_basis_state(uint32_t n, const int* bits, uint32_t n_bits, double* amps, char* err, size_t cap);
int orc_apply_gate(uint32_t n, double* amps, const orc_gate* g, char* err, size_t cap);
int orc_expectation(uint32_t n, const double* amps, const orc_ham* h, double* out, char* err, size_t cap);
uint32_t orc_n_parameters(int kind, uint32_t layers, uint32_t n);
int orc_prepare_ansatz(int kind, uint32_t layers, const double* theta, uint32_t n_theta, uint32_t n, double* amps,
                       char* err, size_t cap);
int orc_energy(int kind, uint32_t layers, const double* theta, uint32_t n_theta, const orc_ham* h, double* out,
               char* err, size_t cap);
int orc_gradient(int kind, uint32_t layers, const double* theta, uint32_t n_theta, const orc_ham* h, double* grad,
                 char* err, size_t cap);
void orc_adam_step(const double* m, const double* v, int64_t step, const double* grad, const double* theta,
                   uint32_t n, const orc_adam* cfg, double* theta_out, double* m_out, double* v_out,
                   int64_t* step_out);
int orc_run_vqe(const orc_ham* h, int kind, uint32_t layers, const orc_adam* cfg, const double* init,
                uint32_t n_init, orc_vqe_result* r, char* err, size_t cap);
int orc_bond_grid(double d_min, double d_max, int n_points, double* out, char* err, size_t cap);
int orc_split_chunks(uint64_t n_items, uint64_t n_chunks, uint64_t* begin_end, char* err, size_t cap);
int orc_build_tfim(uint32_t n, double coupling, double field, orc_ham_out* out, char* err, size_t cap);
int orc_build_z_sum(uint32_t n, orc_ham_out* out, char* err, size_t cap);
int orc_hartree_fock(double bond_angstrom, double* out4, char* err, size_t cap);
int orc_build_h2_hamiltonian(double bond_angstrom, orc_ham_out* out, char* err, size_t cap);
int orc_run_sweep(double d_min, double d_max, int n_points, const orc_adam* cfg, double* bond, double* energy,
                  double* theta_star, int* iterations, int* ok, char* errors, size_t err_stride, char* err,
                  size_t cap);

#ifdef __cplusplus
}
#endif
#endif
