// j2_tma.cuh -- TMA-pipelined persistent variant of the hot-path kernel
// (included by qmcj2.cu after the shared helpers).
//
// One producer warp streams the SoA lanes x|y|z of each (walker, tile) into a
// ring of NST shared-memory stages with 1-D bulk copies
// (cp.async.bulk ... mbarrier::complete_tx::bytes, SASS UBLKCP), one mbarrier
// pair (full/empty) per stage.  Eight consumer warps read one 16-byte vector
// per lane per stage from shared memory, release the stage immediately
// (registers hold the data), and run the same per-term math as the LDG kernel.
// CTAs are persistent (grid = SMs x resident CTAs) and walk the tile list
// round-robin, so the producer prefetches the next tile while the consumers
// reduce the current one.  Deterministic fp64 reduction as in j2_eval_kernel.
#pragma once

#include "bulk.cuh"

namespace qj2 {

constexpr int TMA_NCW = 8;                    // consumer warps
constexpr int TMA_THREADS = (TMA_NCW + 1) * 32;

struct TileInfo {
    int64_t w, g, c, start, end;
};

__device__ __forceinline__ TileInfo decode_tile(const EvalParams &p, uint32_t t, int64_t CH) {
    const uint32_t tpw32 = (uint32_t)p.tiles_per_walker;
    const uint32_t per_w = tpw32 * (uint32_t)p.n_groups;
    const uint32_t w32 = t / per_w;
    const uint32_t rem = t - w32 * per_w;
    const uint32_t g32 = rem / tpw32;
    TileInfo ti;
    ti.w = w32;
    ti.g = g32;
    ti.c = rem - g32 * tpw32;
    ti.start = ti.c * CH;
    ti.end = min(ti.start + CH, p.N_local);
    return ti;
}

// MINB: resident CTAs per SM (register budget), VPT: vectors per consumer
// lane per stage, TMA_NST: ring stages.
template <typename T, int PB, int MINB, int VPT, int TMA_NST>
__global__ void __launch_bounds__(TMA_THREADS, MINB)
j2_eval_tma_kernel(const __grid_constant__ EvalParams p, uint32_t n_tiles) {
    using Tr = Traits<T>;
    using V = typename Tr::V;
    constexpr int VW = Tr::VW;
    constexpr int SRC_STAGE = TPB * VW * VPT;           // sources per stage (VPT vectors per lane)
    constexpr uint32_t LANE_BYTES = SRC_STAGE * sizeof(T);
    constexpr int STAGES_PER_TILE = ITERS * SUB / VPT;  // same tile as j2_eval_kernel
    constexpr int64_t CH = (int64_t)SRC_STAGE * STAGES_PER_TILE;

    extern __shared__ __align__(128) unsigned char smem[];
    V *ring = reinterpret_cast<V *>(smem);                                   // [NST][3][VPT*TPB]
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + TMA_NST * 3 * LANE_BYTES);  // full[NST], empty[NST]
    Coef4<T> *tab = reinterpret_cast<Coef4<T> *>(bars + 2 * TMA_NST);       // [MAXTAB]
    double *red = reinterpret_cast<double *>(tab + MAXTAB);                 // [2][NCW][PB*NACC]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t bar_base = (uint32_t)__cvta_generic_to_shared(bars);
    const uint32_t ring_base = (uint32_t)__cvta_generic_to_shared(ring);
    if (threadIdx.x == 0) {
        for (int s = 0; s < TMA_NST; ++s) {
            mbar_init(bar_base + 8 * s, 1);                          // full: producer's expect_tx
            mbar_init(bar_base + 8 * (TMA_NST + s), TMA_NCW);        // empty: one arrive per consumer warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    load_table<T>(p, tab);
    __syncthreads();

    // =====================  producer warp  =====================
    if (warp == TMA_NCW) {
        if (lane == 0) {
            uint32_t n = 0;   // global stage counter
            for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
                const TileInfo ti = decode_tile(p, t, CH);
                const T *Rw = static_cast<const T *>(p.R) + ti.w * p.src_stride;
                for (int64_t s0 = ti.start; s0 < ti.end; s0 += SRC_STAGE, ++n) {
                    const uint32_t slot = n % TMA_NST, round = n / TMA_NST;
                    mbar_wait(bar_base + 8 * (TMA_NST + slot), (round & 1) ^ 1);
                    const int64_t len = min((int64_t)SRC_STAGE, ti.end - s0);
                    const uint32_t bytes = (uint32_t)(((len + VW - 1) / VW) * VW * sizeof(T));
                    const uint32_t full = bar_base + 8 * slot;
                    mbar_expect_tx(full, 3 * bytes);
#pragma unroll
                    for (int d = 0; d < 3; ++d)
                        bulk_g2s(ring_base + (slot * 3 + d) * LANE_BYTES, Rw + d * p.Np + s0, bytes, full);
                }
            }
        }
        return;
    }

    // =====================  consumer warps  =====================
    const uint32_t tab_addr = (uint32_t)__cvta_generic_to_shared(tab);
    const int tid = threadIdx.x;
    const int64_t tpw = p.tiles_per_walker;

    uint32_t n = 0;     // global stage counter (mirrors the producer's)
    uint32_t parity_tile = 0;
    for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x, parity_tile ^= 1) {
        const TileInfo ti = decode_tile(p, t, CH);
        const int32_t p0 = (int32_t)ti.g * PB;
        const int np = min(PB, p.P - p0);
        Trial<T> tr[PB];
        int kg;
        int64_t k_local;
        walker_setup<T, PB, MODE_J2>(p, ti.w, p0, np, tr, kg, k_local);
        double dacc[PB][NACC];
        T acc[PB][NACC];
#pragma unroll
        for (int q = 0; q < PB; ++q)
#pragma unroll
            for (int a = 0; a < NACC; ++a) dacc[q][a] = 0.0;

        for (int64_t s0 = ti.start; s0 < ti.end; s0 += SRC_STAGE, ++n) {
            const uint32_t slot = n % TMA_NST, round = n / TMA_NST;
            mbar_wait(bar_base + 8 * slot, round & 1);
            const V *st = ring + slot * 3 * (VPT * TPB);
            V cx[VPT], cy[VPT], cz[VPT];
#pragma unroll
            for (int u = 0; u < VPT; ++u) {
                cx[u] = st[u * TPB + tid];
                cy[u] = st[VPT * TPB + u * TPB + tid];
                cz[u] = st[2 * VPT * TPB + u * TPB + tid];
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_base + 8 * (TMA_NST + slot));   // data is in registers

            const int64_t len = min((int64_t)SRC_STAGE, ti.end - s0);
            const int64_t g0 = s0 + p.i_offset;
            const int grp = src_group(p, g0);
            const bool one_group = src_group(p, s0 + len - 1 + p.i_offset) == grp;
            const bool k_in = k_local >= s0 && k_local < s0 + len;
            const GroupC<T> gc = group_consts<T, MODE_J2>(p, grp, kg, tab_addr);
#pragma unroll
            for (int q = 0; q < PB; ++q)
#pragma unroll
                for (int a = 0; a < NACC; ++a) acc[q][a] = T(0);
#pragma unroll
            for (int u = 0; u < VPT; ++u) {
                const int rel = (u * TPB + tid) * VW;
                if (rel >= len) continue;
#pragma unroll
                for (int e = 0; e < VW; ++e) {
                    const int li = rel + e;
                    const bool dead = (li >= len) || (k_in && li == (int)(k_local - s0));
                    const GroupC<T> ge = one_group ? gc : group_consts<T, MODE_J2>(p, src_group(p, g0 + li), kg, tab_addr);
                    const T x = Tr::comp(cx[u], e), y = Tr::comp(cy[u], e), z = Tr::comp(cz[u], e);
#pragma unroll
                    for (int q = 0; q < PB; ++q) {
                        if (PB == 1 || q < np) {
                            const T dx = min_image(x, tr[q].ax);
                            const T dy = min_image(y, tr[q].ay);
                            const T dz = min_image(z, tr[q].az);
                            T r2 = fma(dz, dz, fma(dy, dy, dx * dx));
                            r2 = dead ? T(1e30) : r2;
                            accumulate<T>(dx, dy, dz, r2, gc.invd, ge.base, ge.clamp, acc[q]);
                        }
                    }
                }
            }
            flush<T, PB, MODE_J2>(acc, dacc, gc.sg, gc.sh, gc.ss);   // J2 only: raw sums
        }

        // ---- CTA (consumer) reduction, double-buffered scratch ----
        double *rb = red + parity_tile * (TMA_NCW * PB * NACC);
#pragma unroll
        for (int q = 0; q < PB; ++q)
#pragma unroll
            for (int a = 0; a < NACC; ++a) {
                const double v = warp_sum(dacc[q][a]);
                if (lane == 0) rb[warp * (PB * NACC) + q * NACC + a] = v;
            }
        named_bar(1, TPB);
        if (warp != 0) continue;

        // warp 0: tile total, publish, and (last CTA of the walker) finalize
        double tot = 0.0;
        if (lane < PB * NACC) {
#pragma unroll
            for (int wi = 0; wi < TMA_NCW; ++wi) tot += rb[wi * (PB * NACC) + lane];
        }
        const int64_t wg = ti.w * p.n_groups + ti.g;
        if (tpw > 1) {
            double *part = p.partials + (wg * tpw + ti.c) * (PB * NACC);
            if (lane < PB * NACC) part[lane] = tot;
            __threadfence();
            __syncwarp();
            unsigned last = 0;
            if (lane == 0) last = (atomicAdd(p.counters + wg, 1u) == (unsigned)(tpw - 1));
            last = __shfl_sync(0xffffffffu, last, 0);
            if (!last) continue;
            __threadfence();
            const double *pb = p.partials + wg * tpw * (PB * NACC);
            for (int v = 0; v < PB * NACC; ++v) {
                double s = 0.0;
                for (int64_t c = lane; c < tpw; c += 32) s += __ldcg(pb + c * (PB * NACC) + v);
                s = warp_sum(s);
                if (lane == v) tot = s;
            }
        }
        const double V0 = __shfl_sync(0xffffffffu, tot, 0);
#pragma unroll
        for (int q = 0; q < PB; ++q) {
            double s[NACC];
#pragma unroll
            for (int a = 0; a < NACC; ++a) s[a] = __shfl_sync(0xffffffffu, tot, q * NACC + a);
            if (lane == 0) write_out<PB, MODE_J2>(p, ti.w, p0, np, q, s, V0);
        }
    }
}

template <typename T>
constexpr size_t tma_smem_bytes(int PB, int VPT, int TMA_NST) {
    return (size_t)TMA_NST * 3 * VPT * TPB * Traits<T>::VW * sizeof(T) + 2 * TMA_NST * sizeof(uint64_t) +
           MAXTAB * sizeof(Coef4<T>) + 2 * TMA_NCW * PB * NACC * sizeof(double);
}

}  // namespace qj2
