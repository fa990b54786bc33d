// prune_kernel.cuh -- lattice-beam pruning on the device (sm_100a).
//
// Stage one of prune_lattice (lattice.py:359-394) over the trimmed lattices the decode kernel
// left in its output pools: exact min-sum forward / backward costs, the arc and final cut at
// (best + lattice_beam) + 1e-9, and the re-trim to start-to-final paths (_assemble,
// lattice.py:190-237).  One CTA per utterance.  Lattices are step-layered (emitting arcs go
// from step k-1 to k, epsilon arcs stay inside a step) and the pools keep nodes in step
// order and arcs grouped by destination step (emitting first), so every sweep is a walk over
// steps; epsilon arcs inside a step are relaxed in Jacobi rounds, which reach the same
// fixpoint as the reference's topological order (min is exact).  Also rejects an epsilon
// cycle among a step's nodes (_topo_order, lattice.py:295-326).  The reference's second,
// path-exact stage (_enforce_path_soundness) runs on the host over this already-pruned lattice.
#pragma once
#include "decode_kernel.cuh"

namespace wb {

struct PruneDev {
    const int2 *node;            // decode output pools (trimmed lattices)
    const uint4 *arc;
    const double *ac;
    const u32 *fin;
    const double *finw;
    const long long *meta;       // [n][6]
    const int4 *garcs;           // graph arc records (weights)
    int n, start, T2;            // utterances, start state, step-table stride (max steps + 2)
    double lbeam;
    u64 *fw, *bw;                // scratch, indexed like the node pool
    unsigned char *nflag, *aflag;
    int *depth;
    int *nstart, *gstart, *gsplit;  // [n][T2] per-step node / arc-group / epsilon-split starts
    int2 *p_node;                // outputs
    uint4 *p_arc;
    double *p_ac;
    u32 *p_fin;
    double *p_finw;
    long long p_node_cap, p_arc_cap, p_fin_cap;
    unsigned long long *p_ctr;   // [3]
    long long *p_meta;           // [n][8]: node_off, n_nodes, arc_off, n_arcs, fin_off, n_fin,
                                 //          best (f64 bits), status
};

constexpr unsigned char PF_NS = 1, PF_F2 = 2, PF_B2 = 4, PF_K2 = 8, PF_FIN = 16;

// Forward min-sum over arcs [g0, g1) into their targets: val[to] = min((val[from] + g) + a).
__device__ __forceinline__ bool relax_fw(const PruneDev &P, size_t nb, const uint4 &e, double a,
                                         u64 *val, bool only_if_better) {
    const u64 kf = __ldcg(&val[nb + e.x]);
    if (kf == EMPTY_KEY) return false;
    const int4 r = __ldg(&P.garcs[2 * e.z]);
    const double c = __dadd_rn(__dadd_rn(key_cost(kf), __hiloint2double(r.w, r.z)), a);
    const u64 kc = cost_key(c);
    if (only_if_better && !(kc < __ldcg(&val[nb + e.y]))) return false;
    atomicMin(reinterpret_cast<unsigned long long *>(&val[nb + e.y]), kc);
    return true;
}

// Backward: val[from] = min((g + a) + val[to]).
__device__ __forceinline__ bool relax_bw(const PruneDev &P, size_t nb, const uint4 &e, double a,
                                         u64 *val, bool only_if_better) {
    const u64 kt = __ldcg(&val[nb + e.y]);
    if (kt == EMPTY_KEY) return false;
    const int4 r = __ldg(&P.garcs[2 * e.z]);
    const double c = __dadd_rn(__dadd_rn(__hiloint2double(r.w, r.z), a), key_cost(kt));
    const u64 kc = cost_key(c);
    if (only_if_better && !(kc < __ldcg(&val[nb + e.x]))) return false;
    atomicMin(reinterpret_cast<unsigned long long *>(&val[nb + e.x]), kc);
    return true;
}

template <int PB>
__global__ void __launch_bounds__(PB) prune_kernel(const __grid_constant__ PruneDev P) {
    __shared__ int s_int[4];
    __shared__ unsigned long long s_u64[2];
    const int u = blockIdx.x;
    if (u >= P.n) return;
    const long long *m = P.meta + 6 * (size_t)u;
    long long *pm = P.p_meta + 8 * (size_t)u;
    const long long nb = m[0], nn = m[1], ab = m[2], na = m[3], fb = m[4], nf = m[5];
    const int tid = threadIdx.x;
    if (nb < 0) {  // the decode failed for this utterance
        if (tid == 0) { for (int q = 0; q < 8; ++q) pm[q] = 0; pm[0] = -1; pm[7] = WB_ERR_CAPACITY; }
        return;
    }
    if (nn == 0) {  // EMPTY_LATTICE stays empty
        if (tid == 0) { for (int q = 0; q < 8; ++q) pm[q] = 0; }
        return;
    }
    const int2 *node = P.node + nb;
    const uint4 *arc = P.arc + ab;
    const double *acv = P.ac + ab;
    unsigned char *nfl = P.nflag + nb, *afl = P.aflag + ab;
    int *dep = P.depth + nb;
    int *nst = P.nstart + (size_t)u * P.T2, *gst = P.gstart + (size_t)u * P.T2,
        *gsp = P.gsplit + (size_t)u * P.T2;
    const int K = node[nn - 1].y;  // last step
    // byte flags updated with 32-bit atomics on the aligned word of the pool
    auto set_flag = [&](long long i, unsigned char f) {
        const long long gi = nb + i;
        atomicOr(reinterpret_cast<unsigned int *>(P.nflag + (gi & ~3ll)), (unsigned)f << (8 * (gi & 3)));
    };
    auto clear_flag = [&](long long i, unsigned char f) {
        const long long gi = nb + i;
        atomicAnd(reinterpret_cast<unsigned int *>(P.nflag + (gi & ~3ll)), ~((unsigned)f << (8 * (gi & 3))));
    };
    auto flag = [&](long long i) -> unsigned char { return ((volatile unsigned char *)nfl)[i]; };
    // ---- per-step tables: node starts, arc-group starts (by destination step), epsilon split
    for (int k = tid; k <= K + 1; k += PB) { nst[k] = (int)nn; gst[k] = (int)na; gsp[k] = (int)na; }
    __syncthreads();
    for (long long i = tid; i < nn; i += PB) {
        const int s = node[i].y, sp = i ? node[i - 1].y : -1;
        for (int k = sp + 1; k <= s; ++k) nst[k] = (int)i;
        P.fw[nb + i] = EMPTY_KEY;
        P.bw[nb + i] = EMPTY_KEY;
        nfl[i] = 0;
        dep[i] = 0;
    }
    for (long long e = tid; e < na; e += PB) {
        const uint4 a = arc[e];
        const int s = node[a.y].y, sf = node[a.x].y;
        const int sp = e ? node[arc[e - 1].y].y : -1;
        for (int k = sp + 1; k <= s; ++k) gst[k] = (int)e;
        // first epsilon arc of the group (emitting arcs come first)
        const bool eps = sf == s;
        const bool prev_emit = e == 0 || node[arc[e - 1].y].y != s || node[arc[e - 1].x].y != s;
        if (eps && prev_emit) gsp[s] = (int)e;
        afl[e] = 0;
    }
    __syncthreads();
    // groups without epsilon arcs: split = group end
    for (int k = tid; k <= K; k += PB) {
        const int g1 = gst[k + 1];
        if (gsp[k] > g1 || gsp[k] < gst[k]) gsp[k] = g1;
    }
    if (tid == 0) s_int[1] = -1;
    __syncthreads();
    for (int i = tid; i < nst[1]; i += PB)
        if (node[i].x == P.start) s_int[1] = i;
    for (long long q = tid; q < nf; q += PB) set_flag(P.fin[fb + q], PF_FIN);
    __syncthreads();
    const int st0 = s_int[1];
    int status = WB_OK;
    // ---- epsilon-cycle check: longest epsilon-path depth per step must converge
    for (int k = 0; k <= K; ++k) {
        const int e0 = gsp[k], e1 = gst[k + 1];
        if (e0 >= e1) continue;
        const int nk = nst[k + 1] - nst[k];
        for (int round = 0;; ++round) {
            int ch = 0;
            for (int e = e0 + tid; e < e1; e += PB) {
                const uint4 a = arc[e];
                const int d = __ldcg(&dep[a.x]) + 1;
                if (d > __ldcg(&dep[a.y])) { atomicMax(&dep[a.y], d); ch = 1; }
            }
            if (!__syncthreads_or(ch)) break;
            if (round > nk) { status = WB_ERR_LATTICE; break; }
        }
        if (status != WB_OK) break;
    }
    if (status != WB_OK || st0 < 0) {
        if (tid == 0) { for (int q = 0; q < 8; ++q) pm[q] = 0; pm[7] = status; }
        return;
    }
    // ---- forward min-sum from the start (lattice.py:329-340)
    if (tid == 0) P.fw[nb + st0] = cost_key(0.0);
    __syncthreads();
    for (int k = 0; k <= K; ++k) {
        for (int e = gst[k] + tid; e < gsp[k]; e += PB) relax_fw(P, nb, arc[e], acv[e], P.fw, false);
        __syncthreads();
        const int e0 = gsp[k], e1 = gst[k + 1];
        while (e0 < e1) {
            int ch = 0;
            for (int e = e0 + tid; e < e1; e += PB) ch |= relax_fw(P, nb, arc[e], acv[e], P.fw, true);
            if (!__syncthreads_or(ch)) break;
        }
    }
    // ---- backward min-sum from the finals (lattice.py:343-356)
    for (long long q = tid; q < nf; q += PB) P.bw[nb + P.fin[fb + q]] = cost_key(P.finw[fb + q]);
    __syncthreads();
    for (int k = K; k >= 0; --k) {
        if (k < K) {
            for (int e = gst[k + 1] + tid; e < gsp[k + 1]; e += PB) relax_bw(P, nb, arc[e], acv[e], P.bw, false);
            __syncthreads();
        }
        const int e0 = gsp[k], e1 = gst[k + 1];
        while (e0 < e1) {
            int ch = 0;
            for (int e = e0 + tid; e < e1; e += PB) ch |= relax_bw(P, nb, arc[e], acv[e], P.bw, true);
            if (!__syncthreads_or(ch)) break;
        }
    }
    const u64 kbest = __ldcg(&P.bw[nb + st0]);
    if (kbest == EMPTY_KEY) {  // best == inf: EMPTY_LATTICE
        if (tid == 0) { for (int q = 0; q < 8; ++q) pm[q] = 0; }
        return;
    }
    const double best = key_cost(kbest);
    const double cutoff = __dadd_rn(__dadd_rn(best, P.lbeam), 1e-9);  // lattice.py:380
    // ---- cut (lattice.py:382-389): arcs and finals on some path within the cutoff
    for (long long e = tid; e < na; e += PB) {
        const uint4 a = arc[e];
        const u64 kf = __ldcg(&P.fw[nb + a.x]), kt = __ldcg(&P.bw[nb + a.y]);
        bool keep = false;
        if (kf != EMPTY_KEY && kt != EMPTY_KEY) {
            const int4 r = __ldg(&P.garcs[2 * a.z]);
            const double c = __dadd_rn(__dadd_rn(__dadd_rn(key_cost(kf), __hiloint2double(r.w, r.z)), acv[e]),
                                       key_cost(kt));
            keep = c <= cutoff;
        }
        if (keep) {
            afl[e] = 1;
            set_flag(a.x, PF_NS);
            set_flag(a.y, PF_NS);
        }
    }
    __syncthreads();
    // kept finals: fw + w <= cutoff; they join the node set (PF_FIN cleared otherwise)
    for (long long q = tid; q < nf; q += PB) {
        const u32 i = P.fin[fb + q];
        const u64 kf = __ldcg(&P.fw[nb + i]);
        const bool keep = kf != EMPTY_KEY && __dadd_rn(key_cost(kf), P.finw[fb + q]) <= cutoff;
        if (keep) set_flag(i, PF_NS);
        else clear_flag(i, PF_FIN);
    }
    if (tid == 0) set_flag(st0, PF_NS | PF_F2);
    __syncthreads();
    // ---- re-trim (_assemble): forward reach over kept arcs ...
    for (int k = 0; k <= K; ++k) {
        for (int e = gst[k] + tid; e < gsp[k]; e += PB) {
            const uint4 a = arc[e];
            if (afl[e] && (flag(a.x) & PF_F2)) set_flag(a.y, PF_F2);
        }
        __syncthreads();
        const int e0 = gsp[k], e1 = gst[k + 1];
        while (e0 < e1) {
            int ch = 0;
            for (int e = e0 + tid; e < e1; e += PB) {
                const uint4 a = arc[e];
                if (afl[e] && (flag(a.x) & PF_F2) && !(flag(a.y) & PF_F2)) { set_flag(a.y, PF_F2); ch = 1; }
            }
            if (!__syncthreads_or(ch)) break;
        }
    }
    // ... live finals = kept finals reached forward; backward reach from them
    int nlive = 0;
    for (long long i = tid; i < nn; i += PB) {
        const unsigned char f = flag(i);
        if ((f & PF_FIN) && (f & PF_F2) && (f & PF_NS)) { set_flag(i, PF_B2); ++nlive; }
    }
    if (!__syncthreads_or(nlive)) {
        if (tid == 0) { for (int q = 0; q < 8; ++q) pm[q] = 0; }
        return;
    }
    for (int k = K; k >= 0; --k) {
        if (k < K) {
            for (int e = gst[k + 1] + tid; e < gsp[k + 1]; e += PB) {
                const uint4 a = arc[e];
                if (afl[e] && (flag(a.y) & PF_B2)) set_flag(a.x, PF_B2);
            }
            __syncthreads();
        }
        const int e0 = gsp[k], e1 = gst[k + 1];
        while (e0 < e1) {
            int ch = 0;
            for (int e = e0 + tid; e < e1; e += PB) {
                const uint4 a = arc[e];
                if (afl[e] && (flag(a.y) & PF_B2) && !(flag(a.x) & PF_B2)) { set_flag(a.x, PF_B2); ch = 1; }
            }
            if (!__syncthreads_or(ch)) break;
        }
    }
    // keep = (fwd & bwd | live finals) & node set; live finals carry PF_B2 already
    int kn = 0, ka = 0, kfn = 0;
    for (long long i = tid; i < nn; i += PB) {
        const unsigned char f = flag(i);
        if ((f & PF_NS) && (f & PF_F2) && (f & PF_B2)) { set_flag(i, PF_K2); ++kn; }
    }
    __syncthreads();
    for (long long e = tid; e < na; e += PB) {
        const uint4 a = arc[e];
        const bool k2 = afl[e] && (flag(a.x) & PF_K2) && (flag(a.y) & PF_K2);
        afl[e] = k2 ? 2 : 0;
        ka += k2;
    }
    for (long long q = tid; q < nf; q += PB) {
        const unsigned char f = flag(P.fin[fb + q]);
        kfn += (f & PF_FIN) && (f & PF_K2);
    }
    // ---- compact to the output pools (order left to the host's canonical pass)
    if (tid == 0) { s_int[0] = 0; s_int[2] = 0; s_int[3] = 0; }
    __syncthreads();
    atomicAdd(&s_int[0], kn);
    atomicAdd(&s_int[2], ka);
    atomicAdd(&s_int[3], kfn);
    __syncthreads();
    const int tn = s_int[0], ta = s_int[2], tf = s_int[3];
    if (tid == 0) {
        s_u64[0] = atomicAdd(&P.p_ctr[0], (unsigned long long)tn);
        s_u64[1] = atomicAdd(&P.p_ctr[1], (unsigned long long)ta);
        s_int[1] = (int)atomicAdd(&P.p_ctr[2], (unsigned long long)tf);
        s_int[0] = 0;
        s_int[2] = 0;
        s_int[3] = 0;
    }
    __syncthreads();
    const unsigned long long obn = s_u64[0], oba = s_u64[1], obf = (unsigned long long)s_int[1];
    const bool fits = obn + tn <= (unsigned long long)P.p_node_cap && oba + ta <= (unsigned long long)P.p_arc_cap &&
                      obf + tf <= (unsigned long long)P.p_fin_cap;
    if (fits) {
        // node ids: slot in the output = position among kept nodes (atomic order); remap via depth[]
        for (long long i = tid; i < nn; i += PB) {
            if (!(flag(i) & PF_K2)) continue;
            const int o = atomicAdd(&s_int[0], 1);
            dep[i] = o;
            P.p_node[obn + o] = node[i];
        }
        __syncthreads();
        for (long long e = tid; e < na; e += PB) {
            if (afl[e] != 2) continue;
            const uint4 a = arc[e];
            const int o = atomicAdd(&s_int[2], 1);
            P.p_arc[oba + o] = make_uint4((u32)dep[a.x], (u32)dep[a.y], a.z, 0u);
            P.p_ac[oba + o] = acv[e];
        }
        for (long long q = tid; q < nf; q += PB) {
            const u32 i = P.fin[fb + q];
            const unsigned char f = flag(i);
            if (!((f & PF_FIN) && (f & PF_K2))) continue;
            const int o = atomicAdd(&s_int[3], 1);
            P.p_fin[obf + o] = (u32)dep[i];
            P.p_finw[obf + o] = P.finw[fb + q];
        }
    }
    __syncthreads();
    if (tid == 0) {
        pm[0] = fits ? (long long)obn : -1;
        pm[1] = tn;
        pm[2] = (long long)oba;
        pm[3] = ta;
        pm[4] = (long long)obf;
        pm[5] = tf;
        pm[6] = __double_as_longlong(best);
        pm[7] = fits ? WB_OK : WB_ERR_CAPACITY;
    }
}

}  // namespace wb
