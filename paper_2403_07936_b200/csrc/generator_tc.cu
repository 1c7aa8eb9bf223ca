// Tensor-core (tcgen05) generator -- placeholder until the megakernel lands.
#include "generator.cuh"

namespace mgsr {
int tc_pack_weights(mgsr_gen *g) { (void)g; return MGSR_OK; }
size_t tc_workspace_bytes(int64_t nc) { (void)nc; return 0; }
int launch_sr_pass_tc(const mgsr_gen *, const double *, const double *, int, double, double, double *, void *,
                      size_t, cudaStream_t) {
    set_error("tensor-core generator not built");
    return MGSR_E_UNSUPPORTED;
}
}  // namespace mgsr
