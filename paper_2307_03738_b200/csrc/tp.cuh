// Tensor-parallel one-shot all-reduce of the decode driver's row-parallel
// layers (north_star (d)): shared between the GEMV
// epilogue that pushes (gemv.cu) and the reduce / bookkeeping kernels (tp.cu).
//
// Every rank owns one device buffer, mapped into every peer's address space
// (CUDA IPC over NVLink / NVSwitch, or plain local pointers when several ranks
// are emulated on one GPU):
//   [0, 64)    flags[2 slots][8 sources]  u32 arrival counters (columns received)
//   [64, 68)   epoch                      u32 decode steps begun on this rank
//   [68, 72)   error                      u32 nonzero after a wait timed out
//   [256, ..)  inbox[2 slots][world][bmax][d] f32 partial outputs
// A row-parallel GEMV with the push epilogue stores its partial y_r (no
// residual) straight into inbox[slot][r] of EVERY rank and then adds the
// number of columns it wrote to flags[slot][r] of every rank (system-scope
// release).  Each rank then runs tp_reduce: h += sum_r inbox[slot][r] in rank
// order (bit-identical on every rank), after its flags show all d columns of
// this use from every source.  Slots alternate (o_proj / down_proj), which
// makes a rank's next write into a slot impossible before every rank has read
// that slot's previous use.  Counters only grow: the target
// of use l of step e is ((e - 1) L + l + 1) d, compared wrap-safe.
#pragma once
#include <stdint.h>

namespace qigen {

constexpr int kTpMaxWorld = 8;
constexpr int kTpHeader = 256;

struct TpPush {
  float* inbox[kTpMaxWorld];      // each rank's inbox base (peer-mapped)
  unsigned* flags[kTpMaxWorld];   // each rank's flags base (peer-mapped)
  int rank, world, slot, bmax;
  int64_t d;
};

}  // namespace qigen

struct qigen_tp_comm {
  void* base[qigen::kTpMaxWorld];  // every rank's buffer (index rank = this rank's own)
  int rank, world, bmax, layers;
  int64_t d;
};
