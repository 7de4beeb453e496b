// rasp_inst_s4.cu -- epoch-kernel instantiations for 4-byte HBM words.
#include "rasp_host.cuh"

namespace rasp {
namespace host {

template <>
int run_typed<uint32_t>(const rasp_params *p, const EpochArgs &a, const Plan &pl, const Device &dv,
                   const Workspace &ws, uint64_t d, int64_t tau_max, int64_t epoch, cudaStream_t st)
{
    if (p->w <= 16) return dispatch_flags<uint32_t, uint16_t, uint32_t>(p, a, pl, dv, ws, d, tau_max, epoch, st);
    return dispatch_flags<uint32_t, uint32_t, uint32_t>(p, a, pl, dv, ws, d, tau_max, epoch, st);
}

}  // namespace host
}  // namespace rasp
