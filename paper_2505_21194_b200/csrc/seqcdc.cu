// seqcdc.cu -- B200 (sm_100a) SeqCDC chunking behind the C ABI in include/seqcdc.h.
//
// Pipeline for one call (all on the caller's stream, no host synchronisation):
//   0. reset       one cudaMemsetAsync of the control words + publication
//                  counters (single stream), or k_setup (batch): the segment
//                  table -- each stream cut into segments of G bytes, G a
//                  multiple of max_size.
//   1. k_walk      persistent CTAs, one warp each.  A CTA takes segments in
//                  order and walks a SPECULATIVE chain from the segment start
//                  as if a cut were there ("the next cut depends only on the
//                  previous cut"), recording cuts < segment end in its list L_s
//                  (published every 32 cuts with release semantics).  At the
//                  first cut >= segment end the chain continues (EXTENSION),
//                  each cut checked against the list of the chain that owns
//                  that region; the first common cut is a merge point: from
//                  there on both chains are identical.  Extension cuts go to X_s.
//   2. k_stitch    per stream (one CTA): follow the merges from the stream start
//                  (the only chain that is right from its start) to mark live
//                  chains and where each becomes valid; count valid cuts.  A
//                  stream whose extension overflowed its budget (pathological
//                  phase-locked data) is re-walked here by one warp, end to end.
//                  For a single stream the same CTA also scans the counts.
//   3. k_scan      (batches only) exclusive scan of per-segment counts.
//   4. k_copy      gather valid L/X cuts into d_cuts.
// The hot loop (k_walk) streams every byte HBM->SMEM once with 1-D TMA and
// classifies lazily; see seqcdc_device.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/seqcdc.h"
#include "seqcdc_device.cuh"

#define SEQCDC_API extern "C" __attribute__((visibility("default")))
#ifndef SEQCDC_MIN_BLOCKS
#define SEQCDC_MIN_BLOCKS 1
#endif

namespace seqcdc {

constexpr uint64_t DONE_BIT = 1ull << 63;
constexpr uint64_t CNT_MASK = DONE_BIT - 1;
constexpr int32_t TGT_END = -2;
constexpr int32_t TGT_OVERFLOW = -3;
constexpr int64_t ENTRY_DEAD = -2;
constexpr uint32_t K_EXT = 4;             // extension budget, in segments
constexpr uint64_t G_FLOOR_CHUNKS = 32;   // minimum segment length, in max_size units
constexpr uint64_t G_CEIL = 64ull << 20;  // keeps a chain's span (G + K_EXT*G + max) far below REL_CLAMP
constexpr uint32_t STITCH_MAX_SEGS = 8000;

enum { C_NSEG = 0, C_NEXT = 1, C_NFLAG = 2, C_BAD = 3, C_NWORDS = 8 };

struct Work {
    // inputs
    const uint8_t *in;
    const uint64_t *offs;  // [ns+1]
    uint32_t ns;
    uint32_t single;       // 1: one stream at offset 0, segment table is arithmetic
    uint32_t nseg1;        // single: number of segments
    uint32_t capL1, capX1; // single: uniform list capacities
    uint64_t G;
    uint64_t total;
    uint64_t stop;         // single: the chain ends at its first cut >= stop (= total, or a range end)
    uint64_t out_add;      // single: added to every cut written to d_cuts (range calls: global offset)
    DevParams p;
    // per stream (batch)
    uint32_t *str_first;   // [ns+1]
    uint32_t *str_flag;    // [ns]
    // per segment (batch)
    uint64_t *seg_lo, *seg_hi;
    uint32_t *seg_stream;
    uint64_t *Loff, *Xoff;
    uint32_t *Lcap, *Xcap;
    // per segment (both)
    uint64_t *Lcnt;        // published: count | DONE_BIT
    uint32_t *Xcnt;
    int32_t *target;
    int64_t *midx;
    int64_t *entry;
    uint64_t *seg_count, *seg_out;
    // lists
    uint64_t *L, *X, *FB;
    uint32_t *ctrl;
    // outputs
    uint64_t *cuts, *cut_index, *ncuts;
};

struct Seg {
    uint64_t lo, hi, S0, E;   // segment [lo,hi), stream [S0,E) -- offsets into `in`
    uint64_t Loff, Xoff;
    uint32_t Lcap, Xcap;
    uint32_t j, first, nseg;  // stream, its first segment, its segment count
    bool last;
};

__device__ __forceinline__ uint32_t nseg_total(const Work &w) { return w.single ? w.nseg1 : w.ctrl[C_NSEG]; }

__device__ __forceinline__ Seg get_seg(const Work &w, uint32_t s)
{
    Seg g;
    if (w.single) {
        g.j = 0;
        g.first = 0;
        g.nseg = w.nseg1;
        g.S0 = 0;
        g.E = w.total;
        g.last = (s + 1 == w.nseg1);
        g.lo = (uint64_t)s * w.G;
        g.hi = g.last ? w.stop : g.lo + w.G;
        g.Lcap = w.capL1;
        g.Loff = (uint64_t)s * w.capL1;
        g.Xcap = g.last ? 0 : w.capX1;
        g.Xoff = (uint64_t)s * w.capX1;
    } else {
        g.j = w.seg_stream[s];
        g.first = w.str_first[g.j];
        g.nseg = w.str_first[g.j + 1] - g.first;
        g.last = (s + 1 == g.first + g.nseg);
        g.S0 = w.offs[g.j];
        g.E = w.offs[g.j + 1];
        g.lo = w.seg_lo[s];
        g.hi = w.seg_hi[s];
        g.Lcap = w.Lcap[s];
        g.Loff = w.Loff[s];
        g.Xcap = w.Xcap[s];
        g.Xoff = w.Xoff[s];
    }
    return g;
}

__device__ __forceinline__ uint64_t seg_start(const Work &w, const Seg &g, uint32_t t)
{
    return g.S0 + (uint64_t)(t - g.first) * w.G;
}

// ------------------------------------------------------------------ block scan helper
// Exclusive scan over n items with the whole block; get(i) -> u64, put(i, excl).
template <typename Get, typename Put>
__device__ uint64_t block_scan(uint64_t n, Get get, Put put)
{
    __shared__ uint64_t warp_tot[32];
    __shared__ uint64_t carry;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) carry = 0;
    __syncthreads();
    for (uint64_t b0 = 0; b0 < n; b0 += blockDim.x) {
        const uint64_t i = b0 + tid;
        uint64_t v = i < n ? get(i) : 0, incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint64_t t = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) warp_tot[wid] = incl;
        __syncthreads();
        if (wid == 0) {
            uint64_t x = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0, xi = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint64_t t = __shfl_up_sync(FULL, xi, o);
                if (lane >= o) xi += t;
            }
            warp_tot[lane] = xi - x;
        }
        __syncthreads();
        const uint64_t base = carry;
        if (i < n) put(i, base + warp_tot[wid] + incl - v);
        __syncthreads();
        if (tid == blockDim.x - 1) carry = base + warp_tot[wid] + incl;
        __syncthreads();
    }
    return carry;
}

// ------------------------------------------------------------------ 0. setup (batches)
__global__ void __launch_bounds__(1024) k_setup(Work w)
{
    const uint64_t G = w.G, mn = w.p.mn;
    __shared__ uint32_t bad;
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < w.ns; j += blockDim.x)
        if (w.offs[j + 1] < w.offs[j]) bad = 1;
    __syncthreads();
    if (bad || w.offs[w.ns] - w.offs[0] != w.total) {
        if (threadIdx.x == 0) {
            w.ctrl[C_BAD] = 1;
            w.ctrl[C_NSEG] = 0;
        }
        return;
    }
    uint64_t nseg = block_scan(
        w.ns,
        [&](uint64_t j) -> uint64_t {
            uint64_t len = w.offs[j + 1] - w.offs[j];
            return len <= G ? 1 : (len + G - 1) / G;
        },
        [&](uint64_t j, uint64_t ex) { w.str_first[j] = (uint32_t)ex; });
    if (threadIdx.x == 0) {
        w.str_first[w.ns] = (uint32_t)nseg;
        w.ctrl[C_NSEG] = (uint32_t)nseg;
        w.ctrl[C_NEXT] = 0;
        w.ctrl[C_NFLAG] = 0;
        w.ctrl[C_BAD] = 0;
    }
    __syncthreads();
    for (uint64_t s = threadIdx.x; s < nseg; s += blockDim.x) {
        uint32_t lo = 0, hi = w.ns;  // largest j with str_first[j] <= s
        while (hi - lo > 1) {
            uint32_t mid = (lo + hi) >> 1;
            if (w.str_first[mid] <= s) lo = mid; else hi = mid;
        }
        const uint32_t j = lo;
        const uint64_t k = s - w.str_first[j];
        const uint64_t S0 = w.offs[j], E = w.offs[j + 1];
        const uint64_t a = S0 + k * G;
        const bool last = (s + 1 == w.str_first[j + 1]);
        const uint64_t b = last ? E : a + G;
        w.seg_lo[s] = a;
        w.seg_hi[s] = b;
        w.seg_stream[s] = j;
        w.Lcap[s] = (uint32_t)((b - a) / mn + 2);
        uint64_t xr = last ? 0 : E - b;
        if (xr > K_EXT * G) xr = K_EXT * G;
        w.Xcap[s] = last ? 0 : (uint32_t)(xr / mn + 2);
        w.Lcnt[s] = 0;
    }
    __syncthreads();
    block_scan(nseg, [&](uint64_t s) -> uint64_t { return w.Lcap[s]; },
               [&](uint64_t s, uint64_t ex) { w.Loff[s] = ex; });
    block_scan(nseg, [&](uint64_t s) -> uint64_t { return w.Xcap[s]; },
               [&](uint64_t s, uint64_t ex) { w.Xoff[s] = ex; });
}

// ------------------------------------------------------------------ 1. walk
struct ListBuf {  // 32 cuts buffered in lane registers, written coalesced
    uint64_t v;
    uint32_t n;   // total cuts appended
};

__device__ __forceinline__ void lb_push(ListBuf &b, uint64_t cut, uint64_t *dst, int lane)
{
    if (lane == (int)(b.n & 31)) b.v = cut;
    b.n++;
    if ((b.n & 31) == 0) dst[b.n - 32 + lane] = b.v;
}

__device__ __forceinline__ void lb_flush(ListBuf &b, uint64_t *dst, int lane)
{
    const uint32_t r = b.n & 31;
    if (lane < (int)r) dst[b.n - r + lane] = b.v;
}

// Publish the first n entries of a spec list (release), optionally final.
__device__ __forceinline__ void publish(uint64_t *cntp, uint32_t n, bool done, int lane)
{
    __threadfence();
    __syncwarp();
    if (lane == 0) st_release_u64(cntp, (uint64_t)n | (done ? DONE_BIT : 0));
}

enum { CK_MERGE = 0, CK_NO = 1, CK_UNDECIDED = 2 };

struct Cursor {
    int64_t t;     // segment whose list the window belongs to
    uint64_t j;    // list index of window entry 0
    uint32_t nv;   // valid entries in the window
    uint64_t v;    // this lane's window entry
};

// Is offset `cut` a cut of chain t (its implicit start, or an entry of L_t)?
__device__ int check_cut(const Work &w, Cursor &c, uint32_t t, uint64_t t_lo, uint64_t Loff_t, uint64_t cut,
                         int64_t &idx, int lane)
{
    if ((int64_t)t != c.t) {
        c.t = t;
        c.j = 0;
        c.nv = 0;
    }
    if (cut == t_lo) {
        idx = -1;
        return CK_MERGE;
    }
    const uint64_t *Lt = w.L + Loff_t;
#pragma unroll 1
    for (;;) {
        if (c.nv > 0) {
            const uint32_t hit = __ballot_sync(FULL, lane < (int)c.nv && c.v == cut);
            if (hit) {
                idx = (int64_t)(c.j + __ffs(hit) - 1);
                return CK_MERGE;
            }
            const uint64_t last = __shfl_sync(FULL, c.v, c.nv - 1);
            if (last > cut) return CK_NO;
            if (c.nv == 32) {
                c.j += 32;
                c.nv = 0;
            } else {
                const uint64_t word = ld_acquire_u64(w.Lcnt + t);
                const uint64_t cnt = word & CNT_MASK;
                if (cnt > c.j + c.nv) {
                    c.nv = (uint32_t)(cnt - c.j < 32 ? cnt - c.j : 32);
                    c.v = lane < (int)c.nv ? __ldcg(Lt + c.j + lane) : 0;
                    continue;
                }
                return (word & DONE_BIT) ? CK_NO : CK_UNDECIDED;
            }
        }
        const uint64_t word = ld_acquire_u64(w.Lcnt + t);
        const uint64_t cnt = word & CNT_MASK;
        if (cnt > c.j) {
            c.nv = (uint32_t)(cnt - c.j < 32 ? cnt - c.j : 32);
            c.v = lane < (int)c.nv ? __ldcg(Lt + c.j + lane) : 0;
            continue;
        }
        return (word & DONE_BIT) ? CK_NO : CK_UNDECIDED;
    }
}

template <int MODE, int MSPEC>
__device__ void walk_segment(const Work &w, Walker &wk, uint32_t s, int lane)
{
    const uint64_t abase = (uint64_t)(uintptr_t)w.in;
    const Seg g = get_seg(w, s);
    uint32_t base = walker_begin(wk, abase + g.lo, abase + g.E);
    const uint64_t off = wk.rb - abase;                      // relative position -> offset into `in`
    const uint32_t end_rel = wk.end_rel;
    const uint32_t hi_rel = g.last ? FULL : base + (uint32_t)(g.hi - g.lo);
    // the chain of the stream's last segment ends at its first cut >= stop
    // (the stream end, or for range calls the range end: the overhang)
    const uint64_t stop_abs = w.single ? w.stop : g.E;
    const uint32_t stop_rel = (uint32_t)(stop_abs - off);
    uint64_t *Ls = w.L + g.Loff;
    ListBuf lb{0, 0};
    uint32_t c = base;
    bool extend = false;
    // spec phase: cuts < hi belong to L_s
#pragma unroll 1
    while (base < end_rel) {
        c = resolve<MODE, MSPEC>(wk, w.p, base, lane);
        if (c >= hi_rel) {
            extend = true;
            break;
        }
        lb_push(lb, off + c, Ls, lane);
        if ((lb.n & 31) == 0) publish(w.Lcnt + s, lb.n, false, lane);
        if (c >= stop_rel) break;
        base = c;
    }
    lb_flush(lb, Ls, lane);
    publish(w.Lcnt + s, lb.n, true, lane);
    if (!extend) {                       // the stream's last segment: no extension
        if (lane == 0) {
            w.Xcnt[s] = 0;
            w.target[s] = TGT_END;
            w.midx[s] = -1;
        }
        return;
    }

    // ---- extension: walk on until a cut coincides with the chain owning it
    uint64_t *Xs = w.X + g.Xoff;
    ListBuf xb{0, 0};
    Cursor cur{-1, 0, 0, 0};
    int32_t tgt = TGT_OVERFLOW;
    int64_t mi = -1;
    uint64_t t_lo = 0, t_Loff = 0;
    const uint32_t ext_end = hi_rel + (uint32_t)(K_EXT * w.G);  // byte budget (REL_CLAMP safety)
#pragma unroll 1
    for (;;) {
        if (xb.n == g.Xcap || c > ext_end) {
            tgt = TGT_OVERFLOW;
            break;
        }
        const uint64_t cut = off + c;
        lb_push(xb, cut, Xs, lane);
        if (cut >= stop_abs) {                 // the stream end / the range's overhang
            tgt = TGT_END;
            break;
        }
        const uint32_t t = g.first + (uint32_t)((cut - g.S0) / w.G);
        if ((int64_t)t != cur.t) {
            t_lo = seg_start(w, g, t);
            t_Loff = w.single ? (uint64_t)t * w.capL1 : w.Loff[t];
        }
        int64_t idx;
        if (check_cut(w, cur, t, t_lo, t_Loff, cut, idx, lane) == CK_MERGE) {
            tgt = (int32_t)t;
            mi = idx;
            break;
        }
        base = c;
        c = resolve<MODE, MSPEC>(wk, w.p, base, lane);
    }
    lb_flush(xb, Xs, lane);
    if (lane == 0) {
        w.Xcnt[s] = xb.n;
        w.target[s] = tgt;
        w.midx[s] = mi;
    }
}

template <int MODE, int MSPEC>
__global__ void __launch_bounds__(32, SEQCDC_MIN_BLOCKS) k_walk(Work w)
{
    extern __shared__ __align__(128) uint8_t smem[];
    const int lane = threadIdx.x;
    Walker wk;
    walker_init(wk, smem);
    const uint32_t nseg = w.ctrl[C_BAD] ? 0u : nseg_total(w);
#pragma unroll 1
    for (;;) {
        uint32_t s = 0;
        if (lane == 0) s = atomicAdd(w.ctrl + C_NEXT, 1u);
        s = __shfl_sync(FULL, s, 0);
        if (s >= nseg) break;
        walk_segment<MODE, MSPEC>(w, wk, s, lane);
    }
    walker_finish(wk);
}

// ------------------------------------------------------------------ 2. stitch (+fallback, +scan for one stream)
// One warp re-walks a whole stream (only when an extension overflowed), in
// jobs of <= 1 GiB so relative positions stay 32-bit.
template <int MODE, int MSPEC>
__device__ uint32_t fallback_stream(const Work &w, Walker &wk, uint64_t S0, uint64_t E, uint64_t stop, uint64_t *dst,
                                    int lane)
{
    const uint64_t abase = (uint64_t)(uintptr_t)w.in;
    ListBuf lb{0, 0};
    uint64_t pos = S0;                   // offset of the current chunk start
#pragma unroll 1
    while (pos < stop) {
        uint32_t base = walker_begin(wk, abase + pos, abase + E);
        const uint64_t off = wk.rb - abase;
        const uint32_t stop_at = base + JOB_SPAN;
        const uint32_t stop_rel = (uint32_t)(stop - off < (uint64_t)FULL ? stop - off : FULL);
#pragma unroll 1
        while (base < wk.end_rel && base < stop_at && base < stop_rel) {
            const uint32_t c = resolve<MODE, MSPEC>(wk, w.p, base, lane);
            lb_push(lb, off + c, dst, lane);
            base = c;
        }
        pos = off + base;
    }
    lb_flush(lb, dst, lane);
    walker_finish(wk);
    return lb.n;
}

template <int MODE, int MSPEC>
__global__ void __launch_bounds__(1024) k_stitch(Work w)
{
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ uint32_t flag;
    if (w.ctrl[C_BAD]) return;
    // layout: [ring | barriers | tg[K] | mi[K] | en[K]]
    int32_t *tg = (int32_t *)(sm + SMEM_WALK);
    const uint32_t kmax = STITCH_MAX_SEGS;
    int64_t *mi = (int64_t *)(sm + SMEM_WALK + 4 * kmax);
    int64_t *en = (int64_t *)(sm + SMEM_WALK + 12 * kmax);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (uint32_t j = blockIdx.x; j < w.ns; j += gridDim.x) {
        const uint32_t f = w.single ? 0 : w.str_first[j];
        const uint32_t k = w.single ? w.nseg1 : w.str_first[j + 1] - f;
        if (k == 1) {
            if (threadIdx.x == 0) {
                w.entry[f] = -1;
                w.seg_count[f] = w.Lcnt[f] & CNT_MASK;
                if (!w.single) w.str_flag[j] = 0;
            }
            continue;
        }
        for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) {
            const int32_t t = w.target[f + i];
            tg[i] = t >= 0 ? t - (int32_t)f : t;
            mi[i] = w.midx[f + i];
            en[i] = ENTRY_DEAD;
        }
        if (threadIdx.x == 0) flag = 0;
        __syncthreads();
        if (wid == 0) {
            uint32_t cur = 0;
            int64_t ent = -1;
#pragma unroll 1
            for (;;) {
                const uint32_t i = cur + lane;
                const int32_t t = i < k ? tg[i] : 0;
                const bool pass = (i + 1 < k) && t == (int32_t)(i + 1);
                const uint32_t nb = __ballot_sync(FULL, !pass);
                const int js = nb ? __ffs(nb) - 1 : 32;
                if (lane <= js && i < k) en[i] = lane == 0 ? ent : mi[i - 1];
                if (js == 32) {
                    ent = mi[cur + 31];
                    cur += 32;
                    continue;
                }
                const uint32_t ic = cur + js;
                if (ic + 1 == k) break;               // the stream's last segment ends at E
                const int32_t tj = tg[ic];
                if (tj == TGT_END) break;
                if (tj < 0) {                         // overflow (or never set)
                    if (lane == 0) flag = 1;
                    break;
                }
                ent = mi[ic];
                cur = (uint32_t)tj;
            }
        }
        __syncthreads();
        if (flag) {
            // pathological stream: one warp re-walks it end to end into FB
            for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) {
                w.seg_count[f + i] = 0;
                w.entry[f + i] = ENTRY_DEAD;
            }
            __syncthreads();
            if (wid == 0) {
                Walker wk;
                walker_init(wk, sm);
                const uint64_t S0 = w.single ? 0 : w.offs[j], E = w.single ? w.total : w.offs[j + 1];
                const uint64_t o0 = w.single ? 0 : w.offs[0];
                const uint32_t n = fallback_stream<MODE, MSPEC>(w, wk, S0, E, w.single ? w.stop : E,
                                                                w.FB + (S0 - o0) / w.p.mn + j, lane);
                if (lane == 0) {
                    w.seg_count[f] = n;
                    w.entry[f] = ENTRY_DEAD;
                }
            }
            if (threadIdx.x == 0 && !w.single) w.str_flag[j] = 1;
            if (threadIdx.x == 0 && w.single) w.ctrl[C_NFLAG] = 1;
        } else {
            for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) {
                const int64_t e = en[i];
                uint64_t c = 0;
                if (e != ENTRY_DEAD) c = (w.Lcnt[f + i] & CNT_MASK) - (uint64_t)(e + 1) + w.Xcnt[f + i];
                w.seg_count[f + i] = c;
                w.entry[f + i] = e;
            }
            if (threadIdx.x == 0 && !w.single) w.str_flag[j] = 0;
        }
        __syncthreads();
    }
    if (w.single && blockIdx.x == 0) {
        __syncthreads();
        const uint64_t total = block_scan(
            w.nseg1, [&](uint64_t s) -> uint64_t { return w.seg_count[s]; },
            [&](uint64_t s, uint64_t ex) { w.seg_out[s] = ex; });
        if (threadIdx.x == 0) {
            w.cut_index[0] = 0;
            w.cut_index[1] = total;
            *w.ncuts = total;
        }
    }
}

// ------------------------------------------------------------------ 3. scan (batches), 4. copy
__global__ void __launch_bounds__(1024) k_scan(Work w)
{
    if (w.ctrl[C_BAD]) {
        if (threadIdx.x == 0) *w.ncuts = SEQCDC_NCUTS_BAD_INPUT;
        return;
    }
    const uint32_t nseg = w.ctrl[C_NSEG];
    const uint64_t total = block_scan(
        nseg, [&](uint64_t s) -> uint64_t { return w.seg_count[s]; },
        [&](uint64_t s, uint64_t ex) { w.seg_out[s] = ex; });
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < w.ns; j += blockDim.x) w.cut_index[j] = w.seg_out[w.str_first[j]];
    if (threadIdx.x == 0) {
        w.cut_index[w.ns] = total;
        *w.ncuts = total;
    }
}

__global__ void __launch_bounds__(256) k_copy(Work w)
{
    if (w.ctrl[C_BAD]) return;
    const uint32_t nseg = nseg_total(w);
    const int lane = threadIdx.x & 31;
    const uint32_t warps = gridDim.x * (blockDim.x >> 5);
    for (uint32_t s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); s < nseg; s += warps) {
        const int64_t e = w.entry[s];
        const uint64_t lc = w.Lcnt[s] & CNT_MASK, nx = w.Xcnt[s], o = w.seg_out[s], cnt = w.seg_count[s];
        uint64_t *out = w.cuts + o;
        const Seg g = get_seg(w, s);
        const bool flagged = w.single ? (w.ctrl[C_NFLAG] != 0) : (w.str_flag[g.j] != 0);
        if (flagged) {
            if (s != g.first) continue;
            const uint64_t o0 = w.single ? 0 : w.offs[0];
            const uint64_t *src = w.FB + (g.S0 - o0) / w.p.mn + g.j;
            for (uint64_t i = lane; i < cnt; i += 32) out[i] = src[i] + w.out_add;
            continue;
        }
        if (e == ENTRY_DEAD) continue;
        const uint64_t nl = lc - (uint64_t)(e + 1);
        const uint64_t *Ls = w.L + g.Loff + (e + 1);
        for (uint64_t i = lane; i < nl; i += 32) out[i] = __ldcg(Ls + i) + w.out_add;
        const uint64_t *Xs = w.X + g.Xoff;
        for (uint64_t i = lane; i < nx; i += 32) out[nl + i] = __ldcg(Xs + i) + w.out_add;
    }
}

__global__ void k_empty(uint64_t *cut_index, uint64_t *ncuts)
{
    cut_index[0] = 0;
    *ncuts = 0;
}

__global__ void k_single_offsets(uint64_t *offs, uint64_t n)
{
    offs[0] = 0;
    offs[1] = n;
}

// ------------------------------------------------------------------ host side
struct Plan {
    uint64_t G, nseg_max, L_items, X_items, FB_items;
    uint32_t nseg1, capL1, capX1;
    size_t bytes;
    size_t o_ctrl, o_Lcnt, o_str_first, o_str_flag, o_seg_lo, o_seg_hi, o_seg_stream, o_Loff, o_Xoff,
        o_Lcap, o_Xcap, o_Xcnt, o_target, o_midx, o_entry, o_seg_count, o_seg_out, o_L, o_X, o_FB;
    uint32_t walk_grid;
};

static int g_sms = 0, g_occ = 0;
static uint64_t g_force_G = 0;
static std::mutex g_mu;
static cudaMemPool_t g_pool[64];
static bool g_pool_ok[64];

template <int MODE, int MSPEC>
static void set_attrs()
{
    cudaFuncSetAttribute((const void *)k_walk<MODE, MSPEC>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_WALK);
    cudaFuncSetAttribute((const void *)k_stitch<MODE, MSPEC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         SMEM_WALK + 20 * STITCH_MAX_SEGS);
}

static int device_info(int &sms, int &occ)
{
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_sms) {
        int dev;
        if (cudaGetDevice(&dev) != cudaSuccess) return SEQCDC_ECUDA;
        int nsm = 0;
        if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return SEQCDC_ECUDA;
        set_attrs<0, 4>();
        set_attrs<0, 0>();
        set_attrs<0, -1>();
        set_attrs<1, 4>();
        set_attrs<1, 0>();
        set_attrs<1, -1>();
        int occ_ = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_, k_walk<0, 4>, 32, SMEM_WALK) != cudaSuccess)
            return SEQCDC_ECUDA;
        if (const char *e = getenv("SEQCDC_WALKERS_PER_SM")) {
            int v = atoi(e);
            if (v > 0 && v < occ_) occ_ = v;
        }
        g_occ = occ_ > 0 ? occ_ : 1;
        g_sms = nsm;
    }
    sms = g_sms;
    occ = g_occ;
    return SEQCDC_OK;
}

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

static void make_plan(uint64_t total, uint32_t ns, const seqcdc_params_t *p, int sms, int occ, Plan &pl,
                      bool single, uint64_t stop)
{
    const uint64_t walkers = (uint64_t)sms * occ;
    const uint64_t mx = p->max_size, mn = p->min_size;
    uint64_t denom = walkers > 2ull * ns ? walkers - ns : std::max<uint64_t>(walkers / 2, 1);
    uint64_t G = (total + denom - 1) / denom;
    G = std::max<uint64_t>(G, G_FLOOR_CHUNKS * mx);
    if (g_force_G) G = std::max<uint64_t>(g_force_G, mx);
    G = std::min<uint64_t>(G, std::max<uint64_t>(G_CEIL, mx));
    G = (G + mx - 1) / mx * mx;
    pl.G = G;
    if (single) {
        pl.nseg1 = (uint32_t)(stop <= G ? 1 : (stop + G - 1) / G);
        pl.nseg_max = pl.nseg1;
        pl.capL1 = (uint32_t)(G / mn + 2);
        pl.capX1 = (uint32_t)(std::min<uint64_t>(K_EXT * G, total) / mn + 2);
        pl.L_items = (uint64_t)pl.nseg1 * pl.capL1;
        pl.X_items = (uint64_t)pl.nseg1 * pl.capX1;
    } else {
        pl.nseg1 = pl.capL1 = pl.capX1 = 0;
        pl.nseg_max = (uint64_t)ns + total / G + 1;
        pl.L_items = total / mn + 2 * pl.nseg_max + 2;
        pl.X_items = K_EXT * (total / mn) + 2 * pl.nseg_max + 2;
    }
    pl.FB_items = total / mn + ns + 2;
    pl.walk_grid = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(pl.nseg_max, walkers));
    size_t o = 0;
    auto take = [&](size_t bytes) {
        size_t r = o;
        o = align_up(o + bytes, 256);
        return r;
    };
    const uint64_t S = pl.nseg_max;
    pl.o_ctrl = take(C_NWORDS * 4);
    pl.o_Lcnt = o;  // contiguous with ctrl: one memset resets both
    o = align_up(o + 8 * S, 256);
    pl.o_str_first = take(4ull * (ns + 1));
    pl.o_str_flag = take(4ull * ns);
    pl.o_seg_lo = take(single ? 0 : 8 * S);
    pl.o_seg_hi = take(single ? 0 : 8 * S);
    pl.o_seg_stream = take(single ? 0 : 4 * S);
    pl.o_Loff = take(single ? 0 : 8 * S);
    pl.o_Xoff = take(single ? 0 : 8 * S);
    pl.o_Lcap = take(single ? 0 : 4 * S);
    pl.o_Xcap = take(single ? 0 : 4 * S);
    pl.o_Xcnt = take(4 * S);
    pl.o_target = take(4 * S);
    pl.o_midx = take(8 * S);
    pl.o_entry = take(8 * S);
    pl.o_seg_count = take(8 * S);
    pl.o_seg_out = take(8 * S);
    pl.o_L = take(8 * pl.L_items);
    pl.o_X = take(8 * pl.X_items);
    pl.o_FB = take(8 * pl.FB_items);
    pl.bytes = o;
}

static int get_pool(cudaMemPool_t &pool)
{
    int dev;
    if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return SEQCDC_ECUDA;
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_pool_ok[dev]) {
        cudaMemPoolProps props;
        memset(&props, 0, sizeof(props));
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        if (cudaMemPoolCreate(&g_pool[dev], &props) != cudaSuccess) return SEQCDC_ECUDA;
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(g_pool[dev], cudaMemPoolAttrReleaseThreshold, &thr);
        g_pool_ok[dev] = true;
    }
    pool = g_pool[dev];
    return SEQCDC_OK;
}

// ------------------------------------------------------------------ profiling (bench only)
// When enabled, every call records 4 events on its stream: before the reset,
// before the walk, after the walk, after the copy.  collect() sums elapsed times.
struct ProfRec { cudaEvent_t e[4]; };
static bool g_prof = false;
static std::vector<ProfRec> g_prof_recs;

static void prof_mark(ProfRec *r, int i, cudaStream_t st)
{
    if (r) cudaEventRecord(r->e[i], st);
}

template <int MODE, int MSPEC>
static void launch_all(const Work &w, const Plan &pl, int sms, cudaStream_t st, ProfRec *pr)
{
    prof_mark(pr, 1, st);
    k_walk<MODE, MSPEC><<<pl.walk_grid, 32, SMEM_WALK, st>>>(w);
    prof_mark(pr, 2, st);
    const uint32_t sgrid = w.single ? 1u : (uint32_t)std::min<uint64_t>(w.ns, 2ull * sms);
    k_stitch<MODE, MSPEC><<<sgrid, 1024, SMEM_WALK + 20 * STITCH_MAX_SEGS, st>>>(w);
    if (!w.single) k_scan<<<1, 1024, 0, st>>>(w);
    k_copy<<<std::max(1, sms * 4), 256, 0, st>>>(w);
}

static int run(const uint8_t *d_in, const uint64_t *d_offsets, uint32_t ns, uint64_t total, uint64_t stop,
               uint64_t out_add, const seqcdc_params_t *p, uint64_t *d_cuts, uint64_t *d_cut_index,
               uint64_t *d_ncuts, uint8_t *ws, size_t ws_bytes, const Plan &pl, int sms, cudaStream_t st,
               bool single)
{
    if (ws_bytes < pl.bytes) return SEQCDC_ENOMEM;
    if (total / pl.G + 2 > STITCH_MAX_SEGS) return SEQCDC_EINVAL;  // one stream's segments fit the stitch smem
    Work w;
    memset(&w, 0, sizeof(w));
    w.in = d_in;
    w.offs = d_offsets;
    w.ns = ns;
    w.single = single ? 1u : 0u;
    w.nseg1 = pl.nseg1;
    w.capL1 = pl.capL1;
    w.capX1 = pl.capX1;
    w.G = pl.G;
    w.total = total;
    w.stop = stop;
    w.out_add = out_add;
    w.p.L = p->seq_length;
    w.p.T = p->skip_trigger;
    w.p.S = p->skip_size;
    w.p.M = p->seq_length - 1;
    w.p.mn = (uint32_t)p->min_size;
    w.p.mx = (uint32_t)p->max_size;
    w.p.mnL = (uint32_t)p->min_size - p->seq_length;
    w.ctrl = (uint32_t *)(ws + pl.o_ctrl);
    w.Lcnt = (uint64_t *)(ws + pl.o_Lcnt);
    w.str_first = (uint32_t *)(ws + pl.o_str_first);
    w.str_flag = (uint32_t *)(ws + pl.o_str_flag);
    w.seg_lo = (uint64_t *)(ws + pl.o_seg_lo);
    w.seg_hi = (uint64_t *)(ws + pl.o_seg_hi);
    w.seg_stream = (uint32_t *)(ws + pl.o_seg_stream);
    w.Loff = (uint64_t *)(ws + pl.o_Loff);
    w.Xoff = (uint64_t *)(ws + pl.o_Xoff);
    w.Lcap = (uint32_t *)(ws + pl.o_Lcap);
    w.Xcap = (uint32_t *)(ws + pl.o_Xcap);
    w.Xcnt = (uint32_t *)(ws + pl.o_Xcnt);
    w.target = (int32_t *)(ws + pl.o_target);
    w.midx = (int64_t *)(ws + pl.o_midx);
    w.entry = (int64_t *)(ws + pl.o_entry);
    w.seg_count = (uint64_t *)(ws + pl.o_seg_count);
    w.seg_out = (uint64_t *)(ws + pl.o_seg_out);
    w.L = (uint64_t *)(ws + pl.o_L);
    w.X = (uint64_t *)(ws + pl.o_X);
    w.FB = (uint64_t *)(ws + pl.o_FB);
    w.cuts = d_cuts;
    w.cut_index = d_cut_index;
    w.ncuts = d_ncuts;

    ProfRec rec, *pr = nullptr;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if (g_prof) {
            for (int i = 0; i < 4; i++) cudaEventCreate(&rec.e[i]);
            pr = &rec;
        }
    }
    prof_mark(pr, 0, st);
    if (w.single) {
        if (cudaMemsetAsync(ws + pl.o_ctrl, 0, pl.o_Lcnt - pl.o_ctrl + 8 * pl.nseg1, st) != cudaSuccess)
            return SEQCDC_ECUDA;
    } else {
        k_setup<<<1, 1024, 0, st>>>(w);
    }
    const int ms = p->seq_length == 5 ? 4 : (p->seq_length < 5 ? 0 : -1);
    if (p->mode == SEQCDC_INCREASING) {
        if (ms == 4) launch_all<0, 4>(w, pl, sms, st, pr);
        else if (ms == 0) launch_all<0, 0>(w, pl, sms, st, pr);
        else launch_all<0, -1>(w, pl, sms, st, pr);
    } else {
        if (ms == 4) launch_all<1, 4>(w, pl, sms, st, pr);
        else if (ms == 0) launch_all<1, 0>(w, pl, sms, st, pr);
        else launch_all<1, -1>(w, pl, sms, st, pr);
    }
    prof_mark(pr, 3, st);
    if (pr) {
        std::lock_guard<std::mutex> lk(g_mu);
        g_prof_recs.push_back(rec);
    }
    return cudaGetLastError() == cudaSuccess ? SEQCDC_OK : SEQCDC_ECUDA;
}

// single-stream calls keep their [0, n] offsets and cut index in front of the workspace
constexpr size_t SINGLE_EXTRA = 256;

static int enqueue(const uint8_t *d_in, const uint64_t *d_offsets, uint32_t ns, uint64_t total, uint64_t stop,
                   uint64_t out_add, const seqcdc_params_t *p, uint64_t *d_cuts, uint64_t *d_cut_index,
                   uint64_t *d_ncuts, void *d_ws, size_t ws_bytes, cudaStream_t st, bool single_api)
{
    int sms, occ;
    int rc = device_info(sms, occ);
    if (rc) return rc;
    Plan pl;
    make_plan(total, ns, p, sms, occ, pl, single_api, stop);
    const size_t extra = single_api ? SINGLE_EXTRA : 0;
    uint8_t *ws = (uint8_t *)d_ws;
    bool owned = false;
    if (ws) {
        if (ws_bytes < pl.bytes + extra) return SEQCDC_ENOMEM;
    } else {
        cudaMemPool_t pool;
        if ((rc = get_pool(pool))) return rc;
        if (cudaMallocFromPoolAsync((void **)&ws, pl.bytes + extra, pool, st) != cudaSuccess) return SEQCDC_ENOMEM;
        owned = true;
    }
    if (single_api) {
        uint64_t *offs = (uint64_t *)ws;
        d_offsets = offs;
        d_cut_index = offs + 2;
        k_single_offsets<<<1, 1, 0, st>>>(offs, total);
    }
    rc = run(d_in, d_offsets, ns, total, stop, out_add, p, d_cuts, d_cut_index, d_ncuts, ws + extra, pl.bytes, pl,
             sms, st, single_api);
    if (owned) cudaFreeAsync(ws, st);
    return rc;
}

}  // namespace seqcdc

using namespace seqcdc;

SEQCDC_API int seqcdc_validate_params(const seqcdc_params_t *p)
{
    if (!p) return SEQCDC_EINVAL;
    if (p->mode > 1) return SEQCDC_EINVAL;
    if (p->seq_length < 2 || p->seq_length > SEQCDC_MAX_SEQ_LENGTH) return SEQCDC_EINVAL;
    if (p->skip_trigger < 1) return SEQCDC_EINVAL;
    if (p->min_size < p->seq_length) return SEQCDC_EINVAL;
    if (p->max_size < p->min_size) return SEQCDC_EINVAL;
    if (p->max_size > (1ull << 28)) return SEQCDC_EINVAL;  // implementation limit: 256 MiB chunks
    if (p->flags || p->reserved) return SEQCDC_EINVAL;
    return SEQCDC_OK;
}

SEQCDC_API int seqcdc_default_params(uint32_t avg_kib, uint32_t mode, seqcdc_params_t *out)
{
    if (!out || mode > 1) return SEQCDC_EINVAL;
    uint32_t T, S;
    if (avg_kib == 4) { T = 55; S = 256; }
    else if (avg_kib == 8) { T = 50; S = 256; }
    else if (avg_kib == 16) { T = 50; S = 512; }
    else return SEQCDC_EINVAL;
    memset(out, 0, sizeof(*out));
    out->mode = mode;
    out->seq_length = 5;
    out->skip_trigger = T;
    out->skip_size = S;
    out->min_size = (uint64_t)avg_kib * 512;
    out->max_size = (uint64_t)avg_kib * 2048;
    return SEQCDC_OK;
}

SEQCDC_API uint64_t seqcdc_max_cuts(uint64_t n, const seqcdc_params_t *p)
{
    if (!p || !p->min_size || n == 0) return 0;
    return (n + p->min_size - 1) / p->min_size;
}

SEQCDC_API uint64_t seqcdc_max_cuts_batch(uint64_t total, uint32_t ns, const seqcdc_params_t *p)
{
    if (!p || !p->min_size) return 0;
    return total / p->min_size + ns;
}

SEQCDC_API size_t seqcdc_workspace_size(uint64_t total, uint32_t ns, const seqcdc_params_t *p)
{
    if (seqcdc_validate_params(p)) return 0;
    int sms, occ;
    if (device_info(sms, occ)) {
        sms = 148;
        occ = 32;
    }
    Plan pl;
    Plan pb;
    make_plan(total, ns ? ns : 1, p, sms, occ, pl, ns <= 1, total);
    make_plan(total, ns ? ns : 1, p, sms, occ, pb, false, total);
    return std::max(pl.bytes, pb.bytes) + SINGLE_EXTRA;
}

SEQCDC_API int seqcdc_chunk_batch(const uint8_t *d_in, const uint64_t *d_offsets, uint32_t ns, uint64_t total,
                                  const seqcdc_params_t *p, uint64_t *d_cuts, uint64_t *d_cut_index,
                                  uint64_t *d_ncuts, void *d_ws, size_t ws_bytes, void *stream)
{
    if (seqcdc_validate_params(p)) return SEQCDC_EINVAL;
    if (!d_offsets || !d_cut_index || !d_ncuts) return SEQCDC_EINVAL;
    if (total && (!d_in || !d_cuts)) return SEQCDC_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    if (ns == 0) {
        k_empty<<<1, 1, 0, st>>>(d_cut_index, d_ncuts);
        return cudaGetLastError() == cudaSuccess ? SEQCDC_OK : SEQCDC_ECUDA;
    }
    return enqueue(d_in, d_offsets, ns, total, total, 0, p, d_cuts, d_cut_index, d_ncuts, d_ws, ws_bytes, st,
                   false);
}

SEQCDC_API int seqcdc_chunk(const uint8_t *d_in, uint64_t n, const seqcdc_params_t *p, uint64_t *d_cuts,
                            uint64_t *d_ncuts, void *d_ws, size_t ws_bytes, void *stream)
{
    if (seqcdc_validate_params(p)) return SEQCDC_EINVAL;
    if (!d_ncuts) return SEQCDC_EINVAL;
    if (n && (!d_in || !d_cuts)) return SEQCDC_EINVAL;
    return enqueue(d_in, nullptr, 1, n, n, 0, p, d_cuts, nullptr, d_ncuts, d_ws, ws_bytes, (cudaStream_t)stream,
                   true);
}

SEQCDC_API uint64_t seqcdc_range_max_cuts(uint64_t buf_len, uint64_t range_len, const seqcdc_params_t *p)
{
    if (!p || !p->min_size) return 0;
    const uint64_t span = std::min<uint64_t>(buf_len, range_len + p->max_size);
    return span / p->min_size + 2;
}

SEQCDC_API int seqcdc_range_chunk(const uint8_t *d_buf, uint64_t buf_len, uint64_t range_len, uint64_t entry,
                                  uint64_t global_offset, const seqcdc_params_t *p, uint64_t *d_cuts,
                                  uint64_t *d_ncuts, void *d_ws, size_t ws_bytes, void *stream)
{
    if (seqcdc_validate_params(p)) return SEQCDC_EINVAL;
    if (!d_ncuts || range_len > buf_len || entry > range_len) return SEQCDC_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    if (entry >= range_len) {     // no chunk starts inside the range
        if (cudaMemsetAsync(d_ncuts, 0, 8, st) != cudaSuccess) return SEQCDC_ECUDA;
        return SEQCDC_OK;
    }
    if (!d_buf || !d_cuts) return SEQCDC_EINVAL;
    return enqueue(d_buf + entry, nullptr, 1, buf_len - entry, range_len - entry, global_offset + entry, p, d_cuts,
                   nullptr, d_ncuts, d_ws, ws_bytes, st, true);
}

SEQCDC_API int seqcdc_profile_enable(int on)
{
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto &r : g_prof_recs)
        for (int i = 0; i < 4; i++) cudaEventDestroy(r.e[i]);
    g_prof_recs.clear();
    g_prof = on != 0;
    return SEQCDC_OK;
}

SEQCDC_API int seqcdc_profile_collect(double *ms, uint64_t *ncalls)
{
    std::lock_guard<std::mutex> lk(g_mu);
    double acc[4] = {0, 0, 0, 0};
    for (auto &r : g_prof_recs) {
        if (cudaEventSynchronize(r.e[3]) != cudaSuccess) return SEQCDC_ECUDA;
        float t;
        cudaEventElapsedTime(&t, r.e[0], r.e[1]);
        acc[0] += t;
        cudaEventElapsedTime(&t, r.e[1], r.e[2]);
        acc[1] += t;
        cudaEventElapsedTime(&t, r.e[2], r.e[3]);
        acc[2] += t;
        cudaEventElapsedTime(&t, r.e[0], r.e[3]);
        acc[3] += t;
        for (int i = 0; i < 4; i++) cudaEventDestroy(r.e[i]);
    }
    if (ms)
        for (int i = 0; i < 4; i++) ms[i] = acc[i];
    if (ncalls) *ncalls = g_prof_recs.size();
    g_prof_recs.clear();
    return SEQCDC_OK;
}

SEQCDC_API int seqcdc_set_segment_bytes(uint64_t g)
{
    std::lock_guard<std::mutex> lk(g_mu);
    g_force_G = g;
    return SEQCDC_OK;
}

SEQCDC_API const char *seqcdc_strerror(int code)
{
    switch (code) {
    case SEQCDC_OK: return "ok";
    case SEQCDC_EINVAL: return "invalid argument";
    case SEQCDC_ENOMEM: return "out of memory / workspace too small";
    case SEQCDC_ECUDA: return "CUDA error while enqueuing";
    default: return "unknown error";
    }
}

SEQCDC_API const char *seqcdc_build_info(void)
{
    static char buf[192];
    int sms = 0, occ = 0;
    device_info(sms, occ);
    snprintf(buf, sizeof(buf), "seqcdc sm_100a blk=%u nblk=%u ahead=%u ring=%u win_pairs=%u k_ext=%u walkers=%dx%d",
             BLK, NBLK, AHEAD, RING, WIN_PAIRS, K_EXT, sms, occ);
    return buf;
}
