// device_common.cuh -- small sm_100a building blocks shared by the decoder kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace wb {

typedef unsigned long long u64;
typedef unsigned int u32;

constexpr u64 EMPTY_KEY = 0xFFFFFFFFFFFFFFFFull;
constexpr u64 SIGN64 = 0x8000000000000000ull;
constexpr u32 EPS_BIT = 0x80000000u;   // payload tag: winner came through an epsilon arc
constexpr u32 ROOT_PREV = 0xFFFFFFFFu; // trace root (decoder.py:27 ROOT_TRACE)
constexpr u32 FULL = 0xFFFFFFFFu;

// Order-preserving map from float64 cost to u64, with -0.0 folded onto +0.0 so that the two
// compare equal exactly as Python floats do (frame_costs yields -0.0 for p = 1).
__device__ __forceinline__ u64 cost_key(double c) {
    c = __dadd_rn(c, 0.0);  // -0.0 + 0.0 == +0.0 under round-to-nearest
    u64 b = (u64)__double_as_longlong(c);
    return (b & SIGN64) ? ~b : (b | SIGN64);
}
__device__ __forceinline__ double key_cost(u64 k) {
    u64 b = (k & SIGN64) ? (k & ~SIGN64) : ~k;
    return __longlong_as_double((long long)b);
}

// Recombination slot: (cost key, arc index + 1, payload).  Ordered by (key, arcp1); since arcs
// are sorted by source state, arc order == (src state, arc) order of decoder.py:131.
struct __align__(16) Slot {
    u64 key;
    u32 arcp1;
    u32 pay;
};

__device__ __forceinline__ Slot ld_slot(const Slot *p) {
    // L2-coherent read (slots are updated by L2 atomics from other warps)
    ulonglong2 v = __ldcg(reinterpret_cast<const ulonglong2 *>(p));
    Slot s;
    s.key = v.x;
    s.arcp1 = (u32)v.y;
    s.pay = (u32)(v.y >> 32);
    return s;
}
__device__ __forceinline__ void st_slot_empty(Slot *p) {
    __stcg(reinterpret_cast<ulonglong2 *>(p), make_ulonglong2(EMPTY_KEY, EMPTY_KEY));
}

// Read a slot and reset it to EMPTY in one 128-bit atomic exchange (one L2 round trip instead
// of a load plus a store).
__device__ __forceinline__ Slot xchg_slot_empty(Slot *p, bool evict_first) {
    const u64 e = EMPTY_KEY;
    u64 olo, ohi;
    if (evict_first) {  // the reset line is dead until the state's next (random) touch
        asm volatile(
            "{\n\t.reg .b128 d, o;\n\t.reg .b64 pol;\n\t"
            "createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n\t"
            "mov.b128 d, {%2, %3};\n\t"
            "atom.relaxed.gpu.global.exch.L2::cache_hint.b128 o, [%4], d, pol;\n\t"
            "mov.b128 {%0, %1}, o;\n\t}"
            : "=l"(olo), "=l"(ohi)
            : "l"(e), "l"(e), "l"(p)
            : "memory");
    } else {
        asm volatile(
            "{\n\t.reg .b128 d, o;\n\t"
            "mov.b128 d, {%2, %3};\n\t"
            "atom.relaxed.gpu.global.exch.b128 o, [%4], d;\n\t"
            "mov.b128 {%0, %1}, o;\n\t}"
            : "=l"(olo), "=l"(ohi)
            : "l"(e), "l"(e), "l"(p)
            : "memory");
    }
    Slot o;
    o.key = olo;
    o.arcp1 = (u32)ohi;
    o.pay = (u32)(ohi >> 32);
    return o;
}

// 128-bit compare-and-swap (ATOMG.E.CAS.128).  Returns the previous value.
__device__ __forceinline__ Slot cas_slot(Slot *p, const Slot &expect, const Slot &desired) {
    u64 elo = expect.key, ehi = ((u64)expect.pay << 32) | expect.arcp1;
    u64 dlo = desired.key, dhi = ((u64)desired.pay << 32) | desired.arcp1;
    u64 olo, ohi;
    asm volatile(
        "{\n\t.reg .b128 e, d, o;\n\t"
        "mov.b128 e, {%2, %3};\n\t"
        "mov.b128 d, {%4, %5};\n\t"
        "atom.relaxed.gpu.global.cas.b128 o, [%6], e, d;\n\t"
        "mov.b128 {%0, %1}, o;\n\t}"
        : "=l"(olo), "=l"(ohi)
        : "l"(elo), "l"(ehi), "l"(dlo), "l"(dhi), "l"(p)
        : "memory");
    Slot o;
    o.key = olo;
    o.arcp1 = (u32)ohi;
    o.pay = (u32)(ohi >> 32);
    return o;
}

__device__ __forceinline__ bool slot_better(u64 key, u32 arcp1, const Slot &cur) {
    return key < cur.key || (key == cur.key && arcp1 < cur.arcp1);
}

// Arc-record load.  With WB_ARC_EVICT_FIRST the line is marked evict-first in L2 (a random
// graph's arc records have little reuse; the step's candidate data should keep the L2).
__device__ __forceinline__ int4 ld_arc(const int4 *p) {
#ifdef WB_ARC_EVICT_FIRST
    int4 r;
    u64 pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("ld.global.nc.L2::cache_hint.v4.s32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p), "l"(pol));
    return r;
#else
    return __ldg(p);
#endif
}

__device__ __forceinline__ u32 lanemask_lt() {
    u32 m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ int warp_incl_scan(int v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int n = __shfl_up_sync(FULL, v, o);
        if (lane >= o) v += n;
    }
    return v;
}

// Largest lane k with excl[k] <= j (excl non-decreasing, excl[0] == 0).
__device__ __forceinline__ int warp_owner(int excl, int j) {
    int k = 0;
#pragma unroll
    for (int b = 16; b >= 1; b >>= 1) {
        int e = __shfl_sync(FULL, excl, k + b);
        if (e <= j) k += b;
    }
    return k;
}

__device__ __forceinline__ u64 warp_min_u64(u64 v) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        u64 n = __shfl_xor_sync(FULL, v, o);
        v = n < v ? n : v;
    }
    return v;
}
__device__ __forceinline__ u64 warp_max_u64(u64 v) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        u64 n = __shfl_xor_sync(FULL, v, o);
        v = n > v ? n : v;
    }
    return v;
}
__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

}  // namespace wb
