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

namespace qj2 {

constexpr int TMA_NCW = 8;                    // consumer warps
constexpr int TMA_THREADS = (TMA_NCW + 1) * 32;

__device__ __forceinline__ void mbar_init(uint32_t addr, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(addr), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t addr, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(addr), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t addr) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(addr) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t addr, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra.uni WAIT_%=;\n}" ::"r"(addr), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t mbar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(mbar) : "memory");
}
__device__ __forceinline__ void named_bar(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

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
    Coef4<T> *tab = reinterpret_cast<Coef4<T> *>(bars + 2 * TMA_NST);       // [2][m+1]
    double *red = reinterpret_cast<double *>(tab + 2 * (QJ2_MAX_M + 1));    // [2][NCW][PB*NACC]

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
                const T *Rw = static_cast<const T *>(p.R) + ti.w * 3 * p.Np;
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
    const uint32_t magic_off = (uint32_t)(Tr::MAGIC_BITS * (typename Tr::U)sizeof(Coef4<T>));
    const uint32_t base_same = tab_addr - magic_off;
    const uint32_t base_opp = tab_addr + (uint32_t)((p.m + 1) * sizeof(Coef4<T>)) - magic_off;
    const typename Tr::U clamp_bits = Tr::MAGIC_BITS + (typename Tr::U)p.m;
    const T inv_delta = sizeof(T) == 4 ? T(p.inv_delta_f) : T(p.inv_delta);
    const T L0 = T(p.L[0]), L1 = T(p.L[1]), L2 = T(p.L[2]);
    const int tid = threadIdx.x;
    const int64_t tpw = p.tiles_per_walker;

    uint32_t n = 0;     // global stage counter (mirrors the producer's)
    uint32_t parity_tile = 0;
    for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x, parity_tile ^= 1) {
        const TileInfo ti = decode_tile(p, t, CH);
        const int32_t p0 = (int32_t)ti.g * PB;
        const int np = min(PB, p.P - p0);
        const int64_t kw = p.k[ti.w];
        const bool k_up = kw < p.N_up;
        const int64_t k_local = kw - p.i_offset;
        const int64_t nup_local = p.N_up - p.i_offset;
        Trial<T> tr[PB];
#pragma unroll
        for (int q = 0; q < PB; ++q) {
            const int qq = q < np ? q : 0;
            const T *rt = static_cast<const T *>(p.r_trial) + ((ti.w * p.P + p0 + qq) * 3);
            tr[q].ax = make_axis<T>(rt[0], L0);
            tr[q].ay = make_axis<T>(rt[1], L1);
            tr[q].az = make_axis<T>(rt[2], L2);
        }
        double dacc[PB][NACC];
        T acc[PB][NACC];
#pragma unroll
        for (int q = 0; q < PB; ++q)
#pragma unroll
            for (int a = 0; a < NACC; ++a) { dacc[q][a] = 0.0; acc[q][a] = T(0); }

        int sc = 0;
        for (int64_t s0 = ti.start; s0 < ti.end; s0 += SRC_STAGE, ++n, ++sc) {
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
            const bool k_in = k_local >= s0 && k_local < s0 + len;
            const bool clean = (len == SRC_STAGE) && !k_in && !(nup_local > s0 && nup_local < s0 + len);
#pragma unroll
            for (int u = 0; u < VPT; ++u) {
            const int rel = (u * TPB + tid) * VW;
            if (clean) {
                const uint32_t base = ((s0 < nup_local) == k_up) ? base_same : base_opp;
#pragma unroll
                for (int e = 0; e < VW; ++e) {
                    const T x = Tr::comp(cx[u], e), y = Tr::comp(cy[u], e), z = Tr::comp(cz[u], e);
#pragma unroll
                    for (int q = 0; q < PB; ++q) {
                        if (PB == 1 || q < np) {
                            const T dx = min_image(x, tr[q].ax);
                            const T dy = min_image(y, tr[q].ay);
                            const T dz = min_image(z, tr[q].az);
                            const T r2 = fma(dz, dz, fma(dy, dy, dx * dx));
                            accumulate<T>(dx, dy, dz, r2, inv_delta, base, clamp_bits, acc[q]);
                        }
                    }
                }
            } else if (rel < len) {
                const int k_rel = k_in ? (int)(k_local - s0) : -1;
                const int64_t up_rel = nup_local - s0;
#pragma unroll
                for (int e = 0; e < VW; ++e) {
                    const int li = rel + e;
                    const bool dead = (li >= len) || (li == k_rel);
                    const uint32_t base = ((li < up_rel) == k_up) ? base_same : base_opp;
                    const T x = Tr::comp(cx[u], e), y = Tr::comp(cy[u], e), z = Tr::comp(cz[u], e);
#pragma unroll
                    for (int q = 0; q < PB; ++q) {
                        if (PB == 1 || q < np) {
                            const T dx = min_image(x, tr[q].ax);
                            const T dy = min_image(y, tr[q].ay);
                            const T dz = min_image(z, tr[q].az);
                            T r2 = fma(dz, dz, fma(dy, dy, dx * dx));
                            r2 = dead ? T(1e30) : r2;
                            accumulate<T>(dx, dy, dz, r2, inv_delta, base, clamp_bits, acc[q]);
                        }
                    }
                }
            }
            }
            if ((sc & (ITERS / VPT - 1)) == ITERS / VPT - 1) {   // <= ITERS*VW = 32 terms per fp32 partial
#pragma unroll
                for (int q = 0; q < PB; ++q)
#pragma unroll
                    for (int a = 0; a < NACC; ++a) { dacc[q][a] += (double)acc[q][a]; acc[q][a] = T(0); }
            }
        }
#pragma unroll
        for (int q = 0; q < PB; ++q)
#pragma unroll
            for (int a = 0; a < NACC; ++a) dacc[q][a] += (double)acc[q][a];

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
        const double id = p.inv_delta;
        const double V0 = __shfl_sync(0xffffffffu, tot, 0);
#pragma unroll
        for (int q = 0; q < PB; ++q) {
            double s[NACC];
#pragma unroll
            for (int a = 0; a < NACC; ++a) s[a] = __shfl_sync(0xffffffffu, tot, q * NACC + a);
            if (lane == 0 && q < np) {
                const int64_t o = ti.w * p.P + p0 + q;
                p.out[o * 5 + 0] = s[0];
                p.out[o * 5 + 1] = -id * s[1];
                p.out[o * 5 + 2] = -id * s[2];
                p.out[o * 5 + 3] = -id * s[3];
                p.out[o * 5 + 4] = 2.0 * id * id * s[4] + 2.0 * id * s[5];
                if (p.ratio_out) {
                    const double dj = s[0] - (p.V_cur ? p.V_cur[ti.w] : V0);
                    p.ratio_out[o * 2 + 0] = dj;
                    p.ratio_out[o * 2 + 1] = exp(dj);
                }
            }
        }
    }
}

template <typename T>
constexpr size_t tma_smem_bytes(int PB, int VPT, int TMA_NST) {
    return (size_t)TMA_NST * 3 * VPT * TPB * Traits<T>::VW * sizeof(T) + 2 * TMA_NST * sizeof(uint64_t) +
           2 * (QJ2_MAX_M + 1) * sizeof(Coef4<T>) + 2 * TMA_NCW * PB * NACC * sizeof(double);
}

}  // namespace qj2
