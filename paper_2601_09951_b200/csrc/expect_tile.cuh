// Multi-group expectation passes over gathered TMA tiles (expect_tile.cu).
#pragma once

#include <cstdint>
#include <vector>

#include "sv.cuh"

namespace vqf {

constexpr int kExpPhases = 3;  // register phases per tile pass
constexpr int kExpSlots = 4;   // register bits (flip groups) per phase
constexpr int kExpTerms = 2;   // terms per flip group

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
};

// Groups whose flip is one index bit and that hold <= kExpTerms terms are read
// by tile passes: every pass covers up to kExpPhases * kExpSlots of them with
// ONE read of the state.  Returns the passes; `taken[g]` marks the groups.
std::vector<ExpTileParams> plan_expect_tiles(const CompiledHam& h, uint32_t n, int32_t dtype,
                                             std::vector<char>& taken);

// Enqueues the passes on sv's stream; each writes per-CTA complex partials
// of its groups to partials[((entry * G) + group) * nb + block].
void launch_expect_tiles(vqf_statevector* sv, std::vector<ExpTileParams> passes, double* partials, uint32_t G,
                         uint32_t nb);

}  // namespace vqf
