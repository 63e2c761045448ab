// wq_assemble_zhp.cu -- placeholder (replaced by the high-degree line kernel)
#include "wq_internal.cuh"
bool zhp_supported(const wq_plan_s *, int) { return false; }
wq_status launch_assemble_zhp(wq_plan_s *, int, int64_t, int64_t, double *, int32_t *, int64_t, cudaStream_t) {
    wq_set_error("ZHP kernel not built");
    return WQ_EINVAL;
}
