// hsvd_block.cu -- block-column mode (placeholder until the DMMA path lands).
#include "hsvd_internal.cuh"

namespace hsvd {
int64_t block_workspace_size(int64_t, int64_t, const hsvd_config *) { return 256; }
int block_drive(double *, int64_t, int64_t, int64_t, double *, int64_t,
                const int8_t *, int64_t, const hsvd_config *, double *,
                double *, void *, int64_t, hsvd_result *, hsvd_telemetry *,
                cudaStream_t)
{
    set_error("block mode not built yet");
    return HSVD_ERR_UNSUPPORTED;
}
}  // namespace hsvd
