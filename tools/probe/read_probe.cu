// read_probe.cu -- achievable HBM read bandwidth on this B200 for a pure
// streaming read (the C3 kernel's access pattern without its arithmetic):
// grid-stride or tiled LDG.128 (L1::no_allocate, L2::256B) over a buffer of
// the C3 size, a few unroll depths.  Context for DESIGN.md section 7 only.
// Build and run (GPU box):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe/read_probe tools/probe/read_probe.cu
//   ./tools/probe/read_probe
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float4 ld_stream(const float4 *p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}

// 256-bit loads (sm_100: ld .v8.f32, one LDG.E.ENL2.256 per 8 floats)
struct f8 { float4 a, b; };
__device__ __forceinline__ f8 ld_stream8(const float4 *p) {
    f8 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(v.a.x), "=f"(v.a.y), "=f"(v.a.z), "=f"(v.a.w), "=f"(v.b.x), "=f"(v.b.y), "=f"(v.b.z),
                   "=f"(v.b.w) : "l"(p));
    return v;
}

// as read_soa3 with 32-byte loads: a thread's two consecutive float4 vectors per load
template <int PF, int MINB>
__global__ void __launch_bounds__(256, MINB) read_soa3_v8(const float4 *__restrict__ a, long n_vec, float *out) {
    const long np_vec = 614400 / 4;
    const long tiles_per_w = np_vec / (256 * 8 * 8);
    const long w = blockIdx.x / (tiles_per_w + 1), c = blockIdx.x % (tiles_per_w + 1);
    const float4 *px = a + w * 3 * np_vec + c * 256 * 64 + 2 * threadIdx.x;
    const float4 *py = px + np_vec, *pz = py + np_vec;
    const long lim = np_vec - c * 256 * 64 - 2 * threadIdx.x;
    float acc = 0.f;
#pragma unroll 1
    for (int sub = 0; sub < 8; ++sub) {
        f8 bx[4], by[4], bz[4];                      // 4 iterations of 8 floats per thread = 32 terms
#pragma unroll
        for (int j = 0; j < PF; ++j) {
            const long o = (long)sub * 2048 + j * 512;
            if (o < lim) { bx[j] = ld_stream8(px + o); by[j] = ld_stream8(py + o); bz[j] = ld_stream8(pz + o); }
        }
#pragma unroll
        for (int it = 0; it < 4; ++it) {
            if (it + PF < 4) {
                const long o = (long)sub * 2048 + (it + PF) * 512;
                if (o < lim) {
                    bx[it + PF] = ld_stream8(px + o); by[it + PF] = ld_stream8(py + o); bz[it + PF] = ld_stream8(pz + o);
                }
            }
            acc += bx[it].a.x * by[it].a.y + bz[it].b.z + bx[it].b.w;
        }
    }
    if (acc == 1234.5f) out[0] = acc;
}

template <int U>
__global__ void __launch_bounds__(256) read_tiled(const float4 *__restrict__ a, long n_vec, float *out) {
    // each CTA reads a contiguous tile of 256 * U * 8 vectors, U vectors in flight per thread
    const long tile = 256L * U * 8;
    const long base = (long)blockIdx.x * tile;
    float acc = 0.f;
#pragma unroll 1
    for (int it = 0; it < 8; ++it) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long i = base + ((long)it * U + u) * 256 + threadIdx.x;
            v[u] = i < n_vec ? ld_stream(a + i) : make_float4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
    }
    if (acc == 1234.5f) out[0] = acc;
}

// the C3 kernel's pattern: per walker three SoA lanes x|y|z (Np floats each);
// a CTA reads the same 8192-float window of all three, PF groups ahead
template <int PF, int MINB>
__global__ void __launch_bounds__(256, MINB) read_soa3(const float4 *__restrict__ a, long n_vec, float *out) {
    const long np_vec = 614400 / 4;                 // vectors per lane
    const long tiles_per_w = np_vec / (256 * 8 * 8);   // 65536-float tiles (8 sub-tiles of 8 iterations)
    const long w = blockIdx.x / (tiles_per_w + 1), c = blockIdx.x % (tiles_per_w + 1);
    const float4 *px = a + w * 3 * np_vec + c * 256 * 64 + threadIdx.x;
    const float4 *py = px + np_vec, *pz = py + np_vec;
    const long lim = np_vec - c * 256 * 64 - threadIdx.x;
    float acc = 0.f;
#pragma unroll 1
    for (int sub = 0; sub < 8; ++sub) {
        float4 bx[8], by[8], bz[8];
#pragma unroll
        for (int j = 0; j < PF; ++j) {
            const long o = (long)sub * 2048 + j * 256;
            bx[j] = o < lim ? ld_stream(px + o) : make_float4(0, 0, 0, 0);
            by[j] = o < lim ? ld_stream(py + o) : make_float4(0, 0, 0, 0);
            bz[j] = o < lim ? ld_stream(pz + o) : make_float4(0, 0, 0, 0);
        }
#pragma unroll
        for (int it = 0; it < 8; ++it) {
            if (it + PF < 8) {
                const long o = (long)sub * 2048 + (it + PF) * 256;
                bx[it + PF] = o < lim ? ld_stream(px + o) : make_float4(0, 0, 0, 0);
                by[it + PF] = o < lim ? ld_stream(py + o) : make_float4(0, 0, 0, 0);
                bz[it + PF] = o < lim ? ld_stream(pz + o) : make_float4(0, 0, 0, 0);
            }
            acc += bx[it].x * by[it].y + bz[it].z + bx[it].w;
        }
    }
    if (acc == 1234.5f) out[0] = acc;
}

int main() {
    const long n_vec = 1024L * 3 * 614400 / 4;             // 7.55 GB of fp32 as float4
    float4 *a; float *o;
    cudaMalloc(&a, n_vec * 16);
    cudaMalloc(&o, 16);
    cudaMemset(a, 0, n_vec * 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](const char *name, auto kern, long tile) {
        const long grid = (n_vec + tile - 1) / tile;
        for (int r = 0; r < 3; ++r) kern<<<grid, 256>>>(a, n_vec, o);
        float best = 1e9;
        for (int r = 0; r < 10; ++r) {
            cudaEventRecord(e0);
            kern<<<grid, 256>>>(a, n_vec, o);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        printf("%s: %.3f ms  %.0f GB/s\n", name, best, n_vec * 16 / best / 1e6);
    };
    run("tiled U=2", read_tiled<2>, 256L * 2 * 8);
    run("tiled U=4", read_tiled<4>, 256L * 4 * 8);
    run("tiled U=8", read_tiled<8>, 256L * 8 * 8);
    run("tiled U=16", read_tiled<16>, 256L * 16 * 8);
    auto run3 = [&](const char *name, auto kern) {
        const long tiles_per_w = (614400 / 4) / (256 * 64) + 1;
        const long grid = 1024 * tiles_per_w;
        for (int r = 0; r < 3; ++r) kern<<<grid, 256>>>(a, n_vec, o);
        float best = 1e9;
        for (int r = 0; r < 10; ++r) {
            cudaEventRecord(e0);
            kern<<<grid, 256>>>(a, n_vec, o);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        printf("%s: %.3f ms  %.0f GB/s\n", name, best, n_vec * 16 / best / 1e6);
    };
    run3("soa3 PF=2 MINB=3", read_soa3<2, 3>);
    run3("soa3 PF=3 MINB=3", read_soa3<3, 3>);
    run3("soa3 PF=2 MINB=4", read_soa3<2, 4>);
    run3("soa3 PF=4 MINB=2", read_soa3<4, 2>);
    run3("soa3 v8 PF=1 MINB=3", read_soa3_v8<1, 3>);
    run3("soa3 v8 PF=2 MINB=3", read_soa3_v8<2, 3>);
    run3("soa3 v8 PF=1 MINB=4", read_soa3_v8<1, 4>);
    run3("soa3 v8 PF=2 MINB=2", read_soa3_v8<2, 2>);
    return 0;
}
