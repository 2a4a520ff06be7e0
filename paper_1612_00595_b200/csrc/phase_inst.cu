// phase_inst.cu — one k_phase instantiation per object file:
//   nvcc ... -DINST_YT=float -DINST_MODE=0 -DINST_CAP=64 -DINST_GEN=0 -DINST_TM=1
#include "phase.cuh"

namespace seis {
static_assert(INST_CAP == MAXOWN || INST_CAP == kSerialCap, "chain capacity: MAXOWN or kSerialCap");
template void phase_launch<INST_YT, INST_MODE, INST_CAP, (INST_GEN != 0), (INST_TM != 0)>(
    int, int, cudaStream_t, const Dev&, const Samp&, const PhaseArgs&, Ctl*, int);
template cudaError_t phase_set_smem<INST_YT, INST_MODE, INST_CAP, (INST_GEN != 0),
                                    (INST_TM != 0)>(int);
}  // namespace seis
