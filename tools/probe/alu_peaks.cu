// alu_peaks.cu -- measured arithmetic and issue ceilings of this B200, the
// denominators of the ALU-bound roofline rows in bench.py (C3P2, C3P12, J1S,
// N64S, N64SJ) and of the fp64 path (C2f64, C3f64):
//   ffma   FP32 FFMA throughput (8 independent chains per thread), flops = 2 per FFMA;
//   dfma   FP64 DFMA throughput, flops = 2 per DFMA;
//   issue  warp-instruction issue rate with a mix that no single pipe limits
//          (FFMA + IADD3 + LOP3 + FMUL interleaved, independent chains);
//   rsqrt  MUFU.RSQ (the XU pipe, one per functor term).
// Every kernel runs on all SMs (grid = SMs x 8 CTAs of 256 threads), long enough
// (~50-200 ms) to reach the sustained clock; the SM clock is read by the runner
// (tools/probe/alu_peaks.py, NVML during the run) to give per-clock rates too.
// Build (here or on the GPU box):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe/alu_peaks tools/probe/alu_peaks.cu
// The per-kernel SASS is checked by the runner: FFMA / DFMA / MUFU.RSQ counts.
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>

constexpr int TPB = 256;
constexpr int CH = 8;          // independent chains per thread

__global__ void __launch_bounds__(TPB) k_ffma(float *out, int iters, float a, float b) {
    float x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3f + c;
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int c = 0; c < CH; ++c) x[c] = fmaf(x[c], a, b);
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    if (s == 1.2345f) out[blockIdx.x * TPB + threadIdx.x] = s;    // keep the chains alive
}

__global__ void __launch_bounds__(TPB) k_dfma(double *out, int iters, double a, double b) {
    double x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3 + c;
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    if (s == 1.2345) out[blockIdx.x * TPB + threadIdx.x] = s;
}

// Issue rate: four independent chains on three pipes (FMA: FFMA, FMUL; ALU: IADD3,
// LOP3), each instruction independent of the previous one, so the dispatcher, not a
// pipe or a dependency, is the limit: 1 warp-instruction per cycle per SMSP at best.
__global__ void __launch_bounds__(TPB) k_issue(unsigned *out, int iters, float a, unsigned m) {
    float f0 = threadIdx.x * 1e-3f, f1 = f0 + 1.f;
    unsigned u0 = threadIdx.x, u1 = threadIdx.x * 7u;
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            f0 = fmaf(f0, a, 0.5f);
            u0 = (u0 + m) ^ (unsigned)(r * 0x01010101);
            f1 = f1 * a;
            u1 = (u1 ^ m) + (unsigned)(r * 0x00100001);
        }
    }
    if (f0 + f1 == 1.2345f || (u0 ^ u1) == 0x12345u) out[blockIdx.x * TPB + threadIdx.x] = u0 ^ u1;
}

__global__ void __launch_bounds__(TPB) k_rsqrt(float *out, int iters) {
    float x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = 1.f + threadIdx.x * 1e-3f + c;
#pragma unroll 1
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                float y;
                asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[c]));
                x[c] = y;
            }
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    if (s == 1.2345f) out[blockIdx.x * TPB + threadIdx.x] = s;
}

template <typename F>
static float time_ms(F launch, int reps) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch();                                     // warm-up
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return best;
}

int main(int argc, char **argv) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = sms * 8;
    const double threads = (double)grid * TPB;
    void *buf;
    cudaMalloc(&buf, (size_t)grid * TPB * 8);
    const int reps = argc > 1 ? atoi(argv[1]) : 5;
    const int it_f = 20000, it_d = 4000, it_i = 20000, it_r = 8000;
    float ms;
    ms = time_ms([&] { k_ffma<<<grid, TPB>>>((float *)buf, it_f, 0.999f, 1e-3f); }, reps);
    const double ffma = threads * it_f * 16 * CH;
    printf("{\"kernel\": \"ffma\", \"ms\": %.4f, \"ops\": %.6e, \"flops_per_op\": 2, \"per_s\": %.6e}\n", ms, ffma,
           ffma / (ms * 1e-3));
    ms = time_ms([&] { k_dfma<<<grid, TPB>>>((double *)buf, it_d, 0.999, 1e-3); }, reps);
    const double dfma = threads * it_d * 16 * CH;
    printf("{\"kernel\": \"dfma\", \"ms\": %.4f, \"ops\": %.6e, \"flops_per_op\": 2, \"per_s\": %.6e}\n", ms, dfma,
           dfma / (ms * 1e-3));
    ms = time_ms([&] { k_issue<<<grid, TPB>>>((unsigned *)buf, it_i, 0.999f, 0x9e3779b9u); }, reps);
    // thread-instructions executed by the loop body (SASS count per iteration, argv[2]; the runner
    // reads it from cuobjdump -sass)
    const double body = argc > 2 ? atof(argv[2]) : 64.0;
    const double iss = threads * it_i * body;
    printf("{\"kernel\": \"issue\", \"ms\": %.4f, \"ops\": %.6e, \"flops_per_op\": 0, \"per_s\": %.6e}\n", ms, iss,
           iss / (ms * 1e-3));
    ms = time_ms([&] { k_rsqrt<<<grid, TPB>>>((float *)buf, it_r); }, reps);
    const double rs = threads * it_r * 4 * CH;
    printf("{\"kernel\": \"rsqrt\", \"ms\": %.4f, \"ops\": %.6e, \"flops_per_op\": 0, \"per_s\": %.6e}\n", ms, rs,
           rs / (ms * 1e-3));
    printf("{\"sms\": %d, \"grid\": %d, \"tpb\": %d}\n", sms, grid, TPB);
    cudaFree(buf);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
