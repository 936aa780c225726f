// B200 extension of the drop-in API: where the device contexts of this
// process live.  The reference has no such notion (one CPU process,
// projection.cpp:106-119); here a run names its GPU and, for validation of the
// slab decomposition, a number of slab ranks emulated on that GPU (the same
// transpose-fused kernels a one-rank-per-GPU job runs, include/fftmech_b200.h
// fm_ctx_set_virtual_ranks).  One rank per GPU jobs are driven through the C
// ABI (fm_ctx_create_dist) by a launcher that owns the processes.
#pragma once

namespace fftmech {

struct Placement {
  int device = -1;            // CUDA ordinal; -1: $FFTMECH_DEVICE, else 0
  int ranks = 1;              // > 1: slab ranks emulated on `device`
  bool staged_transposes = false;  // ranks > 1: pack / all-to-all / unpack instead of fused peer stores
};

// Applies to contexts created afterwards (build_projection, models).
void set_placement(const Placement& p);
Placement placement();

}  // namespace fftmech
