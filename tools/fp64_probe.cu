// fp64_probe — B200 FP64 throughput probe: DFMA (CUDA cores) vs DMMA
// (mma.sync.aligned.m8n8k4.f64, FP64 tensor cores), alone and interleaved.
// Decides whether any dense FP64 contraction on the HB-GLS path can gain from
// DMMA (north_star: "use DMMA only if ncu shows ...").  Tooling, not product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_scratch/fp64_probe tools/fp64_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

template <int MODE>  // 0 = DFMA only, 1 = DMMA only, 2 = both interleaved
__global__ void probe(double* out, int iters, double s) {
    double acc[16];
#pragma unroll
    for (int k = 0; k < 16; ++k)
        acc[k] = threadIdx.x * 1e-9 + k;
    double c[8][2];
#pragma unroll
    for (int k = 0; k < 8; ++k)
        c[k][0] = c[k][1] = 0.0;
    const double a = 1.0 + threadIdx.x * 1e-12, b = 0.999999;
    for (int it = 0; it < iters; ++it) {
        if (MODE != 1) {
#pragma unroll
            for (int k = 0; k < 16; ++k)
                acc[k] = fma(acc[k], s, 1e-9);
        }
        if (MODE != 0) {
#pragma unroll
            for (int k = 0; k < 8; ++k)
                dmma(c[k], a, b);
        }
    }
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < 16; ++k)
        t += acc[k];
#pragma unroll
    for (int k = 0; k < 8; ++k)
        t += c[k][0] + c[k][1];
    if (t == 1234.5)
        out[0] = t;
}

int main() {
    double* d;
    cudaMalloc(&d, 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 20000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int mode = 0; mode < 3; ++mode) {
        for (int warps : {8, 16, 32}) {
            const int grid = sms * 2, block = warps * 16;  // 2 CTAs/SM
            auto launch = [&]() {
                if (mode == 0) probe<0><<<grid, block>>>(d, iters, 0.9999999);
                if (mode == 1) probe<1><<<grid, block>>>(d, iters, 0.9999999);
                if (mode == 2) probe<2><<<grid, block>>>(d, iters, 0.9999999);
            };
            launch();
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            const double threads = double(grid) * block;
            const double fma_flop = mode != 1 ? threads * iters * 16 * 2.0 : 0.0;
            // one m8n8k4 per warp = 8*8*4 = 256 FMA = 512 FLOP
            const double mma_flop = mode != 0 ? threads / 32.0 * iters * 8 * 512.0 : 0.0;
            std::printf("{\"mode\": \"%s\", \"warps_per_sm\": %d, \"ms\": %.3f, \"dfma_tflops\": %.2f, "
                        "\"dmma_tflops\": %.2f, \"total_tflops\": %.2f}\n",
                        mode == 0 ? "dfma" : mode == 1 ? "dmma" : "dfma+dmma", warps * 2 / 2 * 1, ms,
                        fma_flop / (ms * 1e-3) / 1e12, mma_flop / (ms * 1e-3) / 1e12,
                        (fma_flop + mma_flop) / (ms * 1e-3) / 1e12);
        }
    }
    const cudaError_t e = cudaDeviceSynchronize();
    std::printf("{\"status\": \"%s\"}\n", cudaGetErrorString(e));
    return e == cudaSuccess ? 0 : 1;
}
