// tma_test.cu -- standalone check of the 4D TMA tile load used by k_ws
// (debug helper, not product code).  Tries encoding / instruction variants.
// nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o /tmp/tma_test tools/tma_test.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdint>
#include <cstdio>
#include <vector>
#include <cstdlib>
#include "../paper_1605_01238_b200/csrc/wq_dev.cuh"
using namespace wqdev;

template <int V>
__global__ void k(const __grid_constant__ CUtensorMap tm, double *out, int c0, int c1, int c2, int c3, int nbytes) {
    __shared__ __align__(128) double buf[2048];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_arrive_tx(&bar, nbytes);
        if (V == 0) {
            tma_load_4d(buf, &tm, &bar, c0, c1, c2, c3);
        } else if (V == 1) {
            asm volatile(
                "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, "
                "%6}], [%2];" ::"r"(smem_u32(buf)),
                "l"(&tm), "r"(smem_u32(&bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
                : "memory");
        } else {
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
                "[%2];" ::"r"(smem_u32(buf)),
                "l"(&tm), "r"(smem_u32(&bar)), "r"(c0), "r"(c1)
                : "memory");
        }
    }
    mbar_wait(&bar, 0);
    for (int i = threadIdx.x; i < nbytes / 8; i += blockDim.x) out[i] = buf[i];
}

PFN_cuTensorMapEncodeTiled_v12000 fn;
double *d, *o;

int run(const char *name, int V, int rank, cuuint64_t *dims, cuuint64_t *str, cuuint32_t *box, CUtensorMapDataType dt,
        CUtensorMapL2promotion l2, int c0, int c1, int c2, int c3) {
    CUtensorMap m;
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    CUresult r = fn(&m, dt, rank, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, l2,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (getenv("CLR21")) reinterpret_cast<uint64_t *>(&m)[1] &= ~(1llu << 21);
    int nb = 8;
    for (int i = 0; i < rank; ++i) nb *= box[i];
    if (V == 0) k<0><<<1, 128>>>(m, o, c0, c1, c2, c3, nb);
    if (V == 1) k<1><<<1, 128>>>(m, o, c0, c1, c2, c3, nb);
    if (V == 2) k<2><<<1, 128>>>(m, o, c0, c1, c2, c3, nb);
    cudaError_t e = cudaDeviceSynchronize();
    printf("%-40s enc %d -> %s\n", name, (int)r, cudaGetErrorString(e));
    fflush(stdout);
    return e != cudaSuccess;
}

int main(int argc, char **argv) {
    void *fnp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
    fn = (PFN_cuTensorMapEncodeTiled_v12000)fnp;
    int dv = 0;
    cudaDriverGetVersion(&dv);
    printf("driver %d\n", dv);
    const int n1 = 13, ld1 = 14, n2 = 13, n3 = 13, nc = 7;
    const size_t cs = (size_t)ld1 * n2 * n3;
    cudaMalloc(&d, cs * nc * 8 * 4);
    cudaMalloc(&o, 2048 * 8);
    int which = argc > 1 ? atoi(argv[1]) : 0;
    cuuint64_t dims[4] = {n1, n2, n3, nc};
    cuuint64_t str[3] = {(cuuint64_t)ld1 * 8, (cuuint64_t)ld1 * n2 * 8, (cuuint64_t)cs * 8};
    cuuint32_t box[4] = {4, 13, 1, 6};
    cuuint64_t d2[2] = {64, 64};
    cuuint64_t s2[1] = {64 * 8};
    cuuint32_t b2[2] = {16, 16};
    switch (which) {
    case 0: return run("2d f64 16x16 L2_256", 2, 2, d2, s2, b2, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, 0, 0, 0, 0);
    case 1: return run("2d f64 16x16 none", 2, 2, d2, s2, b2, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, CU_TENSOR_MAP_L2_PROMOTION_NONE, 0, 0, 0, 0);
    case 2: return run("2d i64 16x16 none", 2, 2, d2, s2, b2, CU_TENSOR_MAP_DATA_TYPE_INT64, CU_TENSOR_MAP_L2_PROMOTION_NONE, 0, 0, 0, 0);
    case 3: return run("4d f64 .tile L2_256", 0, 4, dims, str, box, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, 9, 1, 5, 0);
    case 4: return run("4d f64 notile L2_128", 1, 4, dims, str, box, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, 9, 1, 5, 0);
    case 5: return run("4d i64 notile none", 1, 4, dims, str, box, CU_TENSOR_MAP_DATA_TYPE_INT64, CU_TENSOR_MAP_L2_PROMOTION_NONE, 9, 1, 5, 0);
    case 6: { cuuint32_t bx[4] = {4, 13, 1, 6}; return run("4d f64 in-bounds coords", 1, 4, dims, str, bx, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, CU_TENSOR_MAP_L2_PROMOTION_NONE, 0, 0, 0, 0); }
    case 8: { cuuint32_t bx[4] = {4, 13, 1, 6}; return run("4d f64 oob dim0 only", 1, 4, dims, str, bx, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, CU_TENSOR_MAP_L2_PROMOTION_NONE, 11, 0, 0, 0); }
    case 9: { cuuint32_t bx[4] = {4, 13, 1, 6}; return run("4d f64 oob dim1 only", 1, 4, dims, str, bx, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, CU_TENSOR_MAP_L2_PROMOTION_NONE, 0, 1, 0, 0); }
    case 10: { cuuint32_t bx[2] = {16, 16}; return run("2d f64 oob", 2, 2, d2, s2, bx, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, CU_TENSOR_MAP_L2_PROMOTION_NONE, 56, 56, 0, 0); }
    case 7: { cuuint32_t bx[4] = {8, 8, 1, 1}; return run("4d f64 box 8x8x1x1", 1, 4, dims, str, bx, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, CU_TENSOR_MAP_L2_PROMOTION_NONE, 0, 0, 0, 0); }
    }
    return 0;
}
