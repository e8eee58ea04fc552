// Gate fusion through shared-memory tiles (see tile.cu).
#pragma once

#include <cstdint>
#include <vector>

#include "sv.cuh"

namespace vqf {

// One gate of a circuit to fuse.  param >= 0: its (cos, sin) come from the
// per-entry table cs[(param * batch + entry) * 2] (batched shift circuits);
// param < 0: uniform (c, s).
struct TGate {
  int32_t kind;
  uint32_t n_wires;
  uint32_t wires[4];
  int32_t param;
  double c, s;
};

// Applies `gates` in order (commuting gates may be regrouped) to every batch
// entry of sv with as few HBM passes as the tile budget allows.  Returns the
// number of passes issued.
int run_circuit_tiled(vqf_statevector* sv, const std::vector<TGate>& gates, const double* cs_dev);

// Circuit families sharing a prefix (the parameter-shift batch): the first
// pass of the tile schedule that uses each parameter (-1: unused); empty when
// the schedule has single-gate fallback passes (tiny registers).
std::vector<int> tile_param_first_pass(uint32_t n_qubits, int32_t dtype, const std::vector<TGate>& gates,
                                       uint32_t n_params);

// Runs `gates` on a batch whose entry e has entry 0's angles in every pass
// before join[e] (join nondecreasing; entries with join 0 and entry 0 must
// hold the initial state).  Entry e is copied from entry 0 right before pass
// join[e] instead of repeating entry 0's passes: the same operations on the
// same values, so the states are bitwise those of run_circuit_tiled.
int run_circuit_tiled_shared(vqf_statevector* sv, const std::vector<TGate>& gates, const double* cs_dev,
                             const std::vector<uint32_t>& join);

// Tile plan statistics for tests / docs: passes and gates per pass.
std::vector<int> plan_tile_passes(uint32_t n_qubits, int32_t dtype, const std::vector<TGate>& gates);

// HBM passes (fused tile passes + single-gate fallbacks) and fused register
// ops (shared-memory round trips) apply_circuit would issue.  Host only.
void plan_tile_counts(uint32_t n_qubits, int32_t dtype, const std::vector<TGate>& gates, uint32_t* passes,
                      uint32_t* fused_ops);

}  // namespace vqf
