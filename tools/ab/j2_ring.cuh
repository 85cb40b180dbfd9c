// j2_ring.cuh -- ARCHIVED A/B variant (not built): the J2 CTA kernel with a
// per-thread shared-memory ring filled by cp.async instead of the register
// pipeline.  Measured against the product kernel in round 2
// (profiles/r02/ab_results.txt): fp64 C3 within noise, fp32 C3 0.76x.  To
// re-measure, include it after j2_kernels.cuh and launch
// j2_eval_ring_kernel<T, D, MINB> with ring_smem_bytes<D>() of dynamic shared
// memory (cudaFuncAttributeMaxDynamicSharedMemorySize raised: the static
// buffers come on top).
#pragma once

namespace qj2 {

// ===========================================================================
// Long rows, J2 without a row output, with a shared-memory ring instead of a
// register pipeline (A/B: QJ2_RING64 / QJ2_RING32 = ring depth D): every
// thread streams its own vector groups (x|y|z, 16 B each) with cp.async into
// D ring slots of its own, D-1 groups in flight ahead of the one consumed,
// carried across the sub-tile boundaries (the register pipeline restarts at
// every sub-tile).  A thread reads back only what it copied itself, so the
// ring needs no barrier.  With D dividing ITERS every slot index is a
// compile-time constant.  Same decode, classification, masks, fp32 / fp64
// accumulation and reduction as j2_eval_kernel.
// ===========================================================================
__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src) {
    asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <bool B> struct BTag { static constexpr bool value = B; };

template <int D> constexpr size_t ring_smem_bytes() { return (size_t)D * 3 * TPB * 16; }

template <typename T, int D, int MINB>
__global__ void __launch_bounds__(TPB, MINB)
j2_eval_ring_kernel(const __grid_constant__ EvalParams p) {
    using Tr = Traits<T>;
    using V = typename Tr::V;
    static_assert(sizeof(V) == 16 && ITERS % D == 0 && D >= 2, "ring slots: 16 B vectors, D | ITERS");
    constexpr int VW = Tr::VW;
    constexpr int SCH = TPB * VW * ITERS;
    constexpr int CH = SCH * SUB;
    constexpr int ND = NACC;
    constexpr uint32_t COMP = TPB * 16;        // bytes between a slot's x, y, z planes
    constexpr uint32_t SLOT = 3 * COMP;
    __shared__ Coef4<T> tab[MAXTAB];
    __shared__ double red[TPB / 32 * ND];
    __shared__ int last_flag;
    extern __shared__ __align__(16) unsigned char ring_smem[];

    const uint32_t b = blockIdx.x;
    const uint32_t P32 = (uint32_t)p.P;
    const uint32_t per_w = (uint32_t)p.tiles_per_walker * P32;
    const uint32_t w32 = b / per_w;
    const uint32_t rem = b - w32 * per_w;
    const uint32_t c32 = rem / P32;
    const int64_t w = w32, c = c32;
    const int32_t g = (int32_t)(rem - c32 * P32);

    load_table<T>(p, tab);
    Trial<T> tr;
    int kg;
    int64_t k_local;
    walker_setup<T, MODE_J2>(p, w, g, tr, kg, k_local);
    const uint32_t tab_addr = (uint32_t)__cvta_generic_to_shared(tab);

    const int64_t start = c * CH;
    const int64_t end = min(start + (int64_t)CH, p.N_local);
    QJ2_DCHECK(w < p.W && g < p.P && c < p.tiles_per_walker && start < end && end <= p.Np);
    const T *Rw = static_cast<const T *>(p.R) + w * p.src_stride;
    const V *vx0 = reinterpret_cast<const V *>(Rw) + start / VW;
    const V *vy0 = reinterpret_cast<const V *>(Rw + p.Np) + start / VW;
    const V *vz0 = reinterpret_cast<const V *>(Rw + 2 * p.Np) + start / VW;
    const int32_t tlen = (int32_t)(end - start);
    const int32_t nvec = (tlen + VW - 1) / VW;                  // vectors of the tile (the last one in bounds: Np % VW == 0)
    const int32_t ngrp = (nvec + TPB - 1) / TPB;                // vector groups of the tile
    const uint32_t ring = (uint32_t)__cvta_generic_to_shared(ring_smem) + threadIdx.x * 16;
    const V *ring_v = reinterpret_cast<const V *>(ring_smem) + threadIdx.x;

    // group gi -> slot gi % D; groups past the tile end commit empty, vectors past it reload the last one
    auto issue = [&](int32_t gi, uint32_t slot) {
        if (gi < ngrp) {
            const int32_t v = min(gi * TPB + (int32_t)threadIdx.x, nvec - 1);
            const uint32_t d = ring + slot * SLOT;
            cp_async16(d, vx0 + v);
            cp_async16(d + COMP, vy0 + v);
            cp_async16(d + 2 * COMP, vz0 + v);
        }
        cp_async_commit();
    };
#pragma unroll
    for (int d = 0; d < D - 1; ++d) issue(d, d);

    const int32_t k_t = (k_local >= start && k_local < end) ? (int32_t)(k_local - start) : -1;
    const int64_t up64 = p.N_up - p.i_offset - start;
    const int32_t up_t = up64 <= 0 ? 0 : (up64 >= tlen ? tlen : (int32_t)up64);
    const GroupC<T> g_up = group_consts<T, MODE_J2>(p, 0, kg, tab_addr);
    const GroupC<T> g_dn = group_consts<T, MODE_J2>(p, 1, kg, tab_addr);
    __syncthreads();                                            // the functor table

    double dacc[ND];
#pragma unroll
    for (int a = 0; a < ND; ++a) dacc[a] = 0.0;

    auto run = [&](auto gen_tag, int32_t gi0, const GroupC<T> &gc, const SubMask &mk, T (&acc)[NACC]) {
        constexpr bool GEN = decltype(gen_tag)::value;
#pragma unroll
        for (int it = 0; it < ITERS; ++it) {
            cp_async_wait<D - 2>();                             // group gi0 + it has landed (this thread's copies)
            const V *sl = ring_v + (it % D) * (SLOT / 16);
            const V bx = sl[0], by = sl[COMP / 16], bz = sl[2 * COMP / 16];
            issue(gi0 + it + D - 1, (it + D - 1) % D);          // refill the slot consumed last iteration
            const int rel = (it * TPB + (int)threadIdx.x) * VW;
            if (!GEN || rel < mk.len) {
#pragma unroll
                for (int e = 0; e < VW; ++e) {
                    bool dead = false;
                    uint32_t base = gc.base;
                    if (GEN) {
                        const int li = rel + e;
                        dead = (li >= mk.len) || (li == mk.k_rel);
                        base = li < mk.up_rel ? gc.base : mk.base_hi;
                    }
                    const T dx = min_image(Tr::comp(bx, e), tr.ax);
                    const T dy = min_image(Tr::comp(by, e), tr.ay);
                    const T dz = min_image(Tr::comp(bz, e), tr.az);
                    T r2 = fma(dz, dz, fma(dy, dy, dx * dx));
                    if (GEN) r2 = dead ? T(1e30) : r2;
                    accumulate<T>(dx, dy, dz, r2, gc.invd, base, gc.clamp, acc);
                }
            }
        }
    };

#pragma unroll 1
    for (int sidx = 0; sidx < SUB; ++sidx) {
        const int32_t s0 = sidx * SCH;
        if (s0 >= tlen) break;
        const int32_t len = min(SCH, tlen - s0);
        const int32_t k_rel = k_t - s0;
        const bool k_in = k_t >= 0 && (uint32_t)k_rel < (uint32_t)len;
        const int32_t up_rel = up_t - s0;
        const bool straddle = up_rel > 0 && up_rel < len;
        const GroupC<T> &gc = up_rel > 0 ? g_up : g_dn;
        SubMask mk;
        mk.len = len;
        mk.k_rel = k_in ? k_rel : -1;
        mk.g0 = 0;
        mk.up_rel = straddle ? up_rel : len;
        mk.base_hi = straddle ? g_dn.base : gc.base;
        T acc[NACC];
#pragma unroll
        for (int a = 0; a < NACC; ++a) acc[a] = T(0);
        if (len == SCH && !k_in && !straddle) run(BTag<false>{}, sidx * ITERS, gc, mk, acc);
        else run(BTag<true>{}, sidx * ITERS, gc, mk, acc);
        flush<T, MODE_J2>(acc, dacc, gc.sg, gc.sh, gc.ss);
    }
    cp_async_wait<0>();
    cta_reduce_write<MODE_J2>(p, dacc, w, g, c, red, &last_flag);
}

}  // namespace qj2
