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

// Tile plan statistics for tests / docs: passes and gates per pass.
std::vector<int> plan_tile_passes(uint32_t n_qubits, int32_t dtype, const std::vector<TGate>& gates);

// HBM passes (fused tile passes + single-gate fallbacks) and fused register
// ops (shared-memory round trips) apply_circuit would issue.  Host only.
void plan_tile_counts(uint32_t n_qubits, int32_t dtype, const std::vector<TGate>& gates, uint32_t* passes,
                      uint32_t* fused_ops);

}  // namespace vqf
