// phase_api.h — host entry points of the k_phase instantiations. Each
// (signal type, mode, chain capacity, version kinds, item order) variant is
// compiled in its own translation unit (phase_inst.cu with -DINST_*), so the
// variants build in parallel and each gets its own register allocation.
#pragma once

#include <cuda_runtime.h>

#include "engine.cuh"

namespace seis {

// TM: the tile-major item order (many station tiles per warp, configs 2-4);
// otherwise proposal-major with the per-round diff-window cache (config 1)
template <typename YT, int MODE, int CAP, bool GEN, bool TM>
void phase_launch(int grid, int smem, cudaStream_t st, const Dev& d, const Samp& sp,
                  const PhaseArgs& pa, Ctl* ctl, int stamp);
template <typename YT, int MODE, int CAP, bool GEN, bool TM>
cudaError_t phase_set_smem(int bytes);

}  // namespace seis
