// tma_rate.cu -- TMA box-load throughput for the coefficient-box shapes of the line kernels
// (measurement helper, not product code).
//   z layout   [comp][q0][q1][q2] (q2 fastest), box (2 q2, QX q1, QX q0, 6 comp): 16-B inner rows
//   c layout   [q0][q1][q2][comp] (comp fastest), box (2*6, QX, QX) as 3D: 96-B inner rows
// One persistent CTA per SM, one thread issues NBUF loads in flight, walking along q2 of a line and
// then to the next line (like the line kernels).  Reports boxes/s, rows/clk/SM and GB/s.
// nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -o /tmp/tma_rate tools/tma_rate.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdint>
#include <cstdio>
#include <vector>
#include "../paper_1605_01238_b200/csrc/wq_dev.cuh"
using namespace wqdev;

__device__ __forceinline__ void tma_load_3d(void *dst, const void *tmap, uint64_t *bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

template <int NBUF, bool CL>
__global__ void k_rate(const __grid_constant__ CUtensorMap tm, int qx, int nq, int nlines, int tasks_per_line,
                       unsigned box_bytes, unsigned long long *clk) {
    extern __shared__ __align__(128) unsigned char smb[];
    uint64_t *bar = (uint64_t *)smb;
    double *buf = (double *)(smb + 128);
    const unsigned bstride = (box_bytes + 127) & ~127u;
    if (threadIdx.x == 0) {
        for (int b = 0; b < NBUF; ++b) mbar_init(&bar[b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const long long t0 = clock64();
    const int64_t ntask = (int64_t)nlines * tasks_per_line;
    int64_t issued = 0;
    auto issue = [&](int64_t T) {
        const int b = (int)(T % NBUF);
        const int line = (int)(T / tasks_per_line) * gridDim.x + blockIdx.x;
        const int tau = (int)(T % tasks_per_line);
        const int l0 = (line % 90) * 2, l1 = ((line / 90) % 90) * 2;
        mbar_arrive_tx(&bar[b], box_bytes);
        void *dst = (unsigned char *)buf + (size_t)b * bstride;
        if (CL) tma_load_3d(dst, &tm, &bar[b], 12 * tau, l1, l0);
        else tma_load_4d(dst, &tm, &bar[b], 2 * tau, l1, l0, 0);
    };
    for (; issued < NBUF && issued < ntask; ++issued) issue(issued);
    for (int64_t T = 0; T < ntask; ++T) {
        const int b = (int)(T % NBUF);
        mbar_wait(&bar[b], (unsigned)((T / NBUF) & 1));
        if (issued < ntask) { issue(issued); ++issued; }
    }
    clk[blockIdx.x] = clock64() - t0;
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    return (PFN_cuTensorMapEncodeTiled_v12000)p;
}

int main() {
    const int N = 210;  // points per direction (C4 p = 4: 209, row length padded to even)
    const size_t elems = (size_t)6 * N * N * N;
    double *d;
    cudaMalloc(&d, elems * 8);
    cudaMemset(d, 0, elems * 8);
    unsigned long long *clk;
    cudaMalloc(&clk, 148 * 8);
    auto fn = enc();
    int dev_clk_khz = 0;
    cudaDeviceGetAttribute(&dev_clk_khz, cudaDevAttrClockRate, 0);
    const int nlines = 40, tpl = 100;
    for (int qx : {9, 13, 17, 25}) {
        for (int layout = 0; layout < 2; ++layout) {
            CUtensorMap m;
            unsigned box_bytes;
            int rows;
            if (layout == 0) {
                cuuint64_t dims[4] = {(cuuint64_t)N, (cuuint64_t)N, (cuuint64_t)N, 6};
                cuuint64_t str[3] = {(cuuint64_t)N * 8, (cuuint64_t)N * N * 8, (cuuint64_t)N * N * N * 8};
                cuuint32_t box[4] = {2, (cuuint32_t)qx, (cuuint32_t)qx, 6}, es[4] = {1, 1, 1, 1};
                fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
                box_bytes = 2 * qx * qx * 6 * 8;
                rows = qx * qx * 6;
            } else {
                cuuint64_t dims[3] = {(cuuint64_t)6 * N, (cuuint64_t)N, (cuuint64_t)N};
                cuuint64_t str[2] = {(cuuint64_t)6 * N * 8, (cuuint64_t)6 * N * N * 8};
                cuuint32_t box[3] = {12, (cuuint32_t)qx, (cuuint32_t)qx}, es[3] = {1, 1, 1};
                fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
                box_bytes = 12 * qx * qx * 8;
                rows = qx * qx;
            }
            int NBUF = 8;
            while (128 + (size_t)NBUF * ((box_bytes + 127) & ~127u) > 227 * 1024) NBUF = NBUF == 8 ? 4 : 3;
            const size_t smem = 128 + (size_t)NBUF * ((box_bytes + 127) & ~127u);
            auto kern = layout == 0 ? (NBUF == 8 ? k_rate<8, false> : NBUF == 4 ? k_rate<4, false> : k_rate<3, false>)
                                    : (NBUF == 8 ? k_rate<8, true> : NBUF == 4 ? k_rate<4, true> : k_rate<3, true>);
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            kern<<<148, 32, smem>>>(m, qx, N, nlines, tpl, box_bytes, clk);
            cudaEventRecord(e0);
            kern<<<148, 32, smem>>>(m, qx, N, nlines, tpl, box_bytes, clk);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            std::vector<unsigned long long> h(148);
            cudaMemcpy(h.data(), clk, 148 * 8, cudaMemcpyDeviceToHost);
            unsigned long long mx = 0;
            for (auto v : h) mx = v > mx ? v : mx;
            const double boxes = 148.0 * nlines * tpl;
            printf("{\"qx\":%d,\"layout\":\"%s\",\"box_bytes\":%u,\"rows_per_box\":%d,\"ms\":%.3f,\"clk_per_box\":%.1f,"
                   "\"rows_per_clk_sm\":%.3f,\"GBs\":%.1f,\"nbuf\":%d,\"err\":\"%s\"}\n",
                   qx, layout == 0 ? "z(16B rows)" : "comp-inner(96B rows)", box_bytes, rows, ms,
                   (double)mx / (nlines * tpl), (double)rows * nlines * tpl / mx, boxes * box_bytes / (ms * 1e6), NBUF,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
