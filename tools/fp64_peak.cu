// fp64_peak.cu -- FP64 peak microbenchmark for the roofline's FLOP term
// ("measure P_FP64 with a DFMA microbenchmark").
//   DFMA: 8 independent FMA chains per thread, 148 x k CTAs of 256 threads.
//   DMMA: mma.sync.m8n8k4.f64 back to back, 4 independent accumulators per warp.
// Prints TFLOP/s of each (2 FLOP per FMA) and the SM clock seen by nvidia-smi
// is sampled by the caller.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double *out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.678) out[0] = s;
}

__global__ void k_dmma(double *out, int iters) {
    double a = threadIdx.x * 1e-3, b = 0.999;
    double c[4][2];
#pragma unroll
    for (int k = 0; k < 4; ++k) c[k][0] = c[k][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int k = 0; k < 4; ++k)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(c[k][0]), "+d"(c[k][1])
                             : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
    if (s == 12345.678) out[0] = s;
}

// mixed: warps 0-3 of a CTA run the DFMA loop (mode bit 1), warps 4-7 the DMMA loop (mode bit 2);
// each SM sub-partition then holds one warp of each kind.  Comparing the time of mode 3 with
// modes 1 and 2 tells whether DFMA and DMMA share one FP64 pipe (time adds) or not (time = max).
__global__ void k_mixed(double *out, int iters_f, int iters_m, int mode) {
    const int w = threadIdx.x >> 5;
    if (w < 4) {
        if (!(mode & 1)) return;
        double x[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
        for (int it = 0; it < iters_f; ++it) {
#pragma unroll
            for (int r = 0; r < 16; ++r)
#pragma unroll
                for (int k = 0; k < 8; ++k) x[k] = fma(x[k], 0.999, 1e-9);
        }
        double s = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) s += x[k];
        if (s == 12345.678) out[0] = s;
    } else {
        if (!(mode & 2)) return;
        double a = threadIdx.x * 1e-3, b = 0.999;
        double c[4][2];
#pragma unroll
        for (int k = 0; k < 4; ++k) c[k][0] = c[k][1] = 0.0;
        for (int it = 0; it < iters_m; ++it) {
#pragma unroll
            for (int r = 0; r < 8; ++r)
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                                 : "+d"(c[k][0]), "+d"(c[k][1])
                                 : "d"(a), "d"(b));
        }
        double s = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
        if (s == 12345.678) out[0] = s;
    }
}

int main() {
    double *out;
    cudaMalloc(&out, 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int occ : {1, 2, 4}) {
        const int blocks = sms * occ, threads = 256, iters = 4000;
        k_dfma<<<blocks, threads>>>(out, 100, 0.999, 1e-9);
        cudaEventRecord(e0);
        k_dfma<<<blocks, threads>>>(out, iters, 0.999, 1e-9);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * blocks * threads * (double)iters * 16 * 8;
        printf("{\"kernel\":\"dfma\",\"ctas_per_sm\":%d,\"ms\":%.3f,\"tflops\":%.2f}\n", occ, ms, fl / ms / 1e9);
    }
    for (int occ : {1, 2, 4}) {
        const int blocks = sms * occ, threads = 256, iters = 2000;
        k_dmma<<<blocks, threads>>>(out, 100);
        cudaEventRecord(e0);
        k_dmma<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * 256.0 * (blocks * threads / 32) * (double)iters * 8 * 4;  // 8x8x4 FMA per mma
        printf("{\"kernel\":\"dmma_m8n8k4\",\"ctas_per_sm\":%d,\"ms\":%.3f,\"tflops\":%.2f}\n", occ, ms, fl / ms / 1e9);
    }
    for (int occ : {1, 2}) {
        const int blocks = sms * occ, threads = 256, itf = 4000, itm = 1000;
        for (int mode : {1, 2, 3}) {
            k_mixed<<<blocks, threads>>>(out, 50, 20, mode);
            cudaEventRecord(e0);
            k_mixed<<<blocks, threads>>>(out, itf, itm, mode);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double ff = (mode & 1) ? 2.0 * blocks * 128 * (double)itf * 16 * 8 : 0.0;
            double fm = (mode & 2) ? 2.0 * 256.0 * (blocks * 4) * (double)itm * 8 * 4 : 0.0;
            printf("{\"kernel\":\"mixed\",\"mode\":%d,\"ctas_per_sm\":%d,\"ms\":%.3f,\"tflops\":%.2f}\n", mode, occ, ms, (ff + fm) / ms / 1e9);
        }
    }
    cudaError_t e = cudaGetLastError();
    printf("{\"status\":\"%s\"}\n", cudaGetErrorString(e));
    return e != cudaSuccess;
}
