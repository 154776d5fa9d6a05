// tcgen05 production MoL kernel (k_u = k_x = 8, d = 64, G = 64, H = 128).  Placeholder until
// the tensor-core path lands: the dispatcher falls back to the generic SIMT kernel.
#include "kernels.cuh"

namespace molr {

bool mol_tc_supported(const molr_cache*, const molr_gating*, int) { return false; }

template <class Id>
int mol_score_tc(molr_ctx*, const molr_cache*, const molr_gating*, int, const float*, const float*, float, Segs<Id>,
                 float*, int64_t, cudaStream_t) {
  MOLR_FAIL(MOLR_ERR_INVALID, "tcgen05 MoL kernel not built");
}
template int mol_score_tc<int64_t>(molr_ctx*, const molr_cache*, const molr_gating*, int, const float*, const float*,
                                   float, Segs<int64_t>, float*, int64_t, cudaStream_t);
template int mol_score_tc<int32_t>(molr_ctx*, const molr_cache*, const molr_gating*, int, const float*, const float*,
                                   float, Segs<int32_t>, float*, int64_t, cudaStream_t);
}  // namespace molr

extern "C" int molr_gating_tc_prepare(molr_gating*) { return MOLR_OK; }
