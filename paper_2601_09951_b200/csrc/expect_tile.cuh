// Multi-group expectation passes over gathered TMA tiles (expect_tile.cu).
#pragma once

#include <cstdint>
#include <vector>

#include "sv.cuh"

namespace vqf {

constexpr int kExpPhases = 3;  // register phases per tile pass
constexpr int kExpSlots = 4;   // register bits (flip groups) per phase
constexpr int kExpTerms = 2;   // terms per flip group
constexpr int kExpDiag = 32;   // diagonal terms one pass can fold in (TFIM's Z Z to n = 33)

// One single-bit flip group in a register slot of a phase.
struct ExpSlot {
  uint32_t n_terms;  // 0: empty slot
  uint32_t group;    // compiled-Hamiltonian group index (partials slot)
  double cb_re[kExpTerms], cb_im[kExpTerms];
  uint64_t yz[kExpTerms];     // full Y|Z mask: thread / tile parity
  uint32_t smask[kExpTerms];  // bit r: parity of register slot pattern r against yz
  uint32_t sigma[kExpTerms];  // parity(flip & yz): the pair term is 2i Im(v), else 2 Re(v)
};

struct ExpPhase {
  uint16_t tb_s[9], rv_s[kExpSlots];  // swizzled shared-memory offsets of thread / register bits
  uint16_t tb_l[9];                   // plain local offsets of the thread bits
  ExpSlot slot[kExpSlots];
};

// A pass's tile: the B low index bits (one 128-byte row) and the window of
// k contiguous bits [h, h + k): local bit b < B is global bit b, local bit
// B + j is global bit h + j.
struct ExpTileParams {
  uint32_t n, B, k, h, n_phases, G, nb;
  ExpPhase ph[kExpPhases];
  uint8_t reg_gbit[kExpPhases][kExpSlots];  // global index bit of each register slot
  // Folded diagonal group (one pass at most; n_diag = 0 elsewhere): Z
  // strings dmask[q] with real coefficients, gathered into classes of equal
  // coefficient and equal register-slot pattern v in phase 0 (a class's
  // terms as bits q), so a class adds dc (|class| - 2 * #negative terms)
  // with two popcounts.
  // The first class of each pattern sits at index v (dq1[v] = 0: none),
  // further classes in the overflow list.
  uint32_t n_diag, v_live, n_ov;  // v_live bit v: pattern v has a class
  uint64_t dmask[kExpDiag];
  uint32_t dq1[16];
  double dc1[16];
  uint32_t ov_dq[kExpDiag], ov_v[kExpDiag];
  double ov_dc[kExpDiag];
};

// Groups whose flip is one index bit and that hold <= kExpTerms terms are read
// by tile passes: every pass covers up to kExpPhases * kExpSlots of them with
// ONE read of the state.  Returns the passes; `taken[g]` marks the groups.
std::vector<ExpTileParams> plan_expect_tiles(const CompiledHam& h, uint32_t n, int32_t dtype,
                                             std::vector<char>& taken);

// Folds the diagonal group (group 0) into the pass with the fewest register
// phases when it holds 1..kExpDiag Z strings with real coefficients, so the
// separate diagonal read of the state goes away.  Measured TFIM fp64 n = 30
// 16.7 -> 14.6 ms at introduction; fp32 folds too since the class table
// (VQF_NO_DIAG_FOLD32=1 keeps the diagonal pass: n = 26 / 28 / 30 / 32 fp32
// 0.67 / 1.94 / 8.77 / 34.0 ms unfolded vs 0.63 / 1.75 / 7.38 / 28.5 ms
// folded).  Returns whether it did.
bool fold_diag_into_tiles(std::vector<ExpTileParams>& passes, const CompiledHam& h, int32_t dtype);

// Enqueues the passes on sv's stream; each writes per-CTA complex partials
// of its groups to partials[((entry * G) + group) * nb + block].
void launch_expect_tiles(vqf_statevector* sv, std::vector<ExpTileParams> passes, double* partials, uint32_t G,
                         uint32_t nb);

}  // namespace vqf
