// seqcdc.cu -- B200 (sm_100a) SeqCDC chunking behind the C ABI in include/seqcdc.h.
//
// Pipeline for one call (all on the caller's stream, no host synchronisation):
//   0. reset       one cudaMemsetAsync of the control words + publication
//                  counters (single stream), or k_setup (batch): the segment
//                  table -- each stream cut into segments of G bytes (G a
//                  multiple of max_size, except the shortened last segment of a
//                  range call with a tail).
//   1. the walk    speculative chains, one per segment, each started at its
//                  segment start as if a cut were there ("the next cut depends
//                  only on the previous cut"), recording cuts < segment end in
//                  L_s and publishing them with release semantics; at the first
//                  cut >= segment end the chain continues (EXTENSION), each cut
//                  checked against the list of the chain owning that region; the
//                  first common cut is a merge point (from there on both chains
//                  are identical).  Extension cuts go to X_s.
//                  k_walk  (default): persistent one-warp CTAs, each warp one
//                          chain; bytes stream HBM->SMEM through a cp.async
//                          (LDGSTS) ring and are classified lazily, one 128-pair
//                          window per round (seqcdc_device.cuh).
//                  k_lwalk (SEQCDC_WALKER=lane): one chain per LANE with sparse
//                          128-B line fills (seqcdc_lane.cuh).
//   2. post        single stream, k_walk: one k_post launch (every CTA follows
//                  the merges and scans the counts itself, then copies its share);
//                  k_lwalk: k_lpost (valid path over the jumper segments, counts,
//                  scan) + k_lcopy; batches: k_stitch (per stream: follow merges,
//                  continue overflowed extensions), k_scan, k_copy.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
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
constexpr uint64_t HANDED_BIT = 1ull << 62;   // lane walker: count of a speculative part a late lane handed to a warp
constexpr int32_t TGT_END = -2;
constexpr int32_t TGT_OVERFLOW = -3;
constexpr int64_t ENTRY_DEAD = -2;
constexpr int64_t ENTRY_UNSET = -3;   // k_lpost -> k_lscan: the entry follows from midx[s-1]
constexpr uint32_t K_EXT = 8;             // extension budget, in segments
constexpr uint64_t G_FLOOR_CHUNKS = 32;   // minimum segment length, in max_size units
constexpr uint64_t G_CEIL = 64ull << 20;  // keeps a chain's span (G + K_EXT*G + max) far below REL_CLAMP
constexpr uint32_t STITCH_MAX_SEGS = 8000;

enum { C_NSEG = 0, C_NEXT = 1, C_BAD = 3, C_DONE = 4, C_OVF = 5, C_HAND = 6, C_HNEXT = 7, C_FIN = 8, C_SPECDONE = 9, C_SERVED = 10,
       C_NWORDS = 16 };

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
    uint32_t *cont_cnt;    // cuts of the continuation walk appended after X_s (stitch)
    // lists
    uint64_t *L, *X, *FB;
    uint32_t *ctrl;
    // outputs
    uint64_t *cuts, *cut_index, *ncuts;
    // range calls: the chain continued past its overhang for up to tail_max cuts
    // (only chunks wholly inside the buffer), for the next rank's local merge
    uint64_t *tail;        // [tail_max] global offsets: tail[0] = the overhang
    uint64_t *tail_n;      // count written (0 = none / invalid)
    uint32_t tail_max;
    uint64_t *summary;     // range calls (optional): [overhang, number of cuts], written by k_post
    // range calls (optional): push the exchange block [overhang, count, tail_n, tail...]
    // into the next range's mailbox (peer memory), then release push_value to *push_flag
    uint64_t *push_blk, *push_flag;
    uint64_t push_value;
    // lane walker: extensions longer than lw_ext_cap cuts (and a range call's
    // tail) are handed to warps (task list, zeroed with the control words)
    uint32_t *hand;
    uint64_t *lstat;       // k_lscan tile status (look-back), zeroed with the control words
    uint32_t *lclaim;      // per segment: a handed-off speculative part claimed by a warp (zeroed too)
    uint32_t lw_ext_cap;
    uint32_t lw_late;      // lane walker: once this many lanes finished their speculative part, a lane
                           // still in it hands the rest of its segment to a warp (0: never)
    uint32_t lw_late_ext;  // ... and a lane in its extension hands that to a warp at its next cut
    // extension budget in segments (<= K_EXT, the list capacity); a testing knob
    // (SEQCDC_EXT_SEGS) that forces the overflow / continuation paths
    uint32_t ext_segs;
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
// Debug timeline (variant builds with -DSEQCDC_TIMELINE): per segment the
// globaltimer at walk start, end of the speculative part, end of the extension
// and the SM id.  Set with seqcdc_debug_timeline().
#ifdef SEQCDC_TIMELINE
__device__ uint64_t *g_tl;
__device__ uint64_t g_tl_cap;
__device__ __forceinline__ void tl_mark(uint32_t s, int k)
{
    if (g_tl && s < g_tl_cap && threadIdx.x == 0) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        uint32_t smid, wid;
        asm("mov.u32 %0, %%smid;" : "=r"(smid));
        asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
        g_tl[4 * s + k] = t;
        g_tl[4 * s + 3] = smid | ((uint64_t)wid << 32);
    }
}
#define TL_MARK(s, k) tl_mark((s), (k))
#else
#define TL_MARK(s, k)
#endif

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
// The entries were written by all lanes; the warp barrier orders them before
// lane 0's (cumulative) release store of the count.
__device__ __forceinline__ void publish(uint64_t *cntp, uint32_t n, bool done, int lane)
{
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

// BR: the decision used for the speculative bulk (resolve's RED).  Measured:
// the warp min-reduction is faster on single streams (config 2 +3%, 4 GiB
// Markov +3%), the ballot decision on batches of mixed streams (config 3 4 KiB
// row +6%, 8 KiB +2%); extensions and re-walks always use the min-reduction.
template <int MODE, int MSPEC, bool BR>
__device__ void walk_segment(const Work &w, Walker &wk, uint32_t s, int lane)
{
    TL_MARK(s, 0);
    const uint64_t abase = (uint64_t)(uintptr_t)w.in;
    const Seg g = get_seg(w, s);
    uint32_t base = walker_begin(wk, abase + g.lo, abase + g.E);
    const uint64_t off = wk.rb - abase;                      // relative position -> offset into `in`
    const uint32_t end_rel = wk.end_rel;
    const uint32_t hi_rel = g.last ? FULL : base + (uint32_t)(g.hi - g.lo);
    // the chain of the stream's last segment ends at its first cut >= stop
    // (the stream end, or for range calls the range end: the overhang)
    const uint64_t stop_abs = w.single ? w.stop : g.E;
    const uint32_t stop_rel = stop_abs - off < (uint64_t)FULL ? (uint32_t)(stop_abs - off) : FULL;
    uint64_t *Ls = w.L + g.Loff;
    ListBuf lb{0, 0};
    uint32_t c = base;
    bool extend = false;
    // spec phase: cuts < hi belong to L_s
#pragma unroll 1
    while (base < end_rel) {
        c = resolve<MODE, MSPEC, BR>(wk, w.p, base, lane);
        SEQCDC_ASSERT_CUT(base, c, w.p, end_rel);
        if (c >= hi_rel) {
            extend = true;
            break;
        }
        SEQCDC_ASSERT(lb.n < g.Lcap);
        lb_push(lb, off + c, Ls, lane);
        if ((lb.n & 31) == 0) publish(w.Lcnt + s, lb.n, false, lane);
        if (c >= stop_rel) break;
        base = c;
    }
    lb_flush(lb, Ls, lane);
    publish(w.Lcnt + s, lb.n, true, lane);
    TL_MARK(s, 1);
    if (!extend) {                       // the stream's last segment: no extension
        if (w.single && w.tail_max) {    // range call: continue past the overhang (next rank's merge)
            ListBuf tb{0, 0};
            if (c >= stop_rel && c < end_rel) {
                lb_push(tb, off + c + w.out_add, w.tail, lane);
                base = c;
#pragma unroll 1
                while (tb.n < w.tail_max && base + w.p.mx <= end_rel) {
                    c = resolve<MODE, MSPEC>(wk, w.p, base, lane);
                    SEQCDC_ASSERT_CUT(base, c, w.p, end_rel);
                    lb_push(tb, off + c + w.out_add, w.tail, lane);
                    base = c;
                }
            }
            lb_flush(tb, w.tail, lane);
            if (lane == 0) *w.tail_n = tb.n;
        }
        if (lane == 0) {
            w.Xcnt[s] = 0;
            w.target[s] = TGT_END;
            w.midx[s] = -1;
            w.cont_cnt[s] = 0;
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
    const uint32_t ext_end = hi_rel + (uint32_t)(w.ext_segs * w.G);  // byte budget (REL_CLAMP safety)
    // segment owning the current cut, tracked incrementally (segments are uniform
    // within a stream: segment t starts at S0 + (t - first) * G)
    uint32_t t = s;
    uint64_t t_next = seg_start(w, g, s + 1);
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
#pragma unroll 1
        while (cut >= t_next) {
            t++;
            t_next += w.G;
        }
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
        SEQCDC_ASSERT_CUT(base, c, w.p, end_rel);
    }
    lb_flush(xb, Xs, lane);
    TL_MARK(s, 2);
    if (lane == 0) {
        w.Xcnt[s] = xb.n;
        w.target[s] = tgt;
        w.midx[s] = mi;
        w.cont_cnt[s] = 0;
        if (tgt == TGT_OVERFLOW) atomicOr(w.ctrl + C_OVF, 1u);
    }
}

// ------------------------------------------------------------------ 2. stitch (+continuation, +scan for one stream)
// FB slot of the continuation of segment s that starts at offset `from`: on the
// valid path continuations cover disjoint, increasing position ranges, and a
// chain covering [a, b] has at most (b-a)/min + 1 cuts, so `from/min + s` never
// overlaps the next one.
__device__ __forceinline__ uint64_t *cont_slot(const Work &w, uint32_t s, uint64_t from)
{
    return w.FB + (from - (w.single ? 0 : w.offs[0])) / w.p.mn + s;
}

// Continue the valid chain of segment s past its exhausted extension budget:
// walk from `from` (its last extension cut, a true cut) until a cut coincides
// with the chain owning its region (all lists are complete now) or the stream
// (range) ends.  One warp; positions re-based every JOB_SPAN bytes.
template <int MODE, int MSPEC>
__device__ uint32_t continue_chain(const Work &w, Walker &wk, const Seg &g, uint32_t s, uint64_t from,
                                   int32_t &tgt, int64_t &mi, int lane)
{
    const uint64_t abase = (uint64_t)(uintptr_t)w.in;
    const uint64_t stop = w.single ? w.stop : g.E;
    uint64_t *dst = cont_slot(w, s, from);
    ListBuf lb{0, 0};
    Cursor cur{-1, 0, 0, 0};
    uint64_t t_lo = 0, t_Loff = 0;
    tgt = TGT_END;
    mi = -1;
    uint64_t pos = from;
    bool done = false;
    uint32_t t = g.first + (uint32_t)((from - g.S0) / w.G);     // segment owning `from`, then incremental
    uint64_t t_next = seg_start(w, g, t + 1);
#pragma unroll 1
    while (!done && pos < stop) {
        uint32_t base = walker_begin(wk, abase + pos, abase + g.E);
        const uint64_t off = wk.rb - abase;
        const uint32_t stop_at = base + JOB_SPAN;
#pragma unroll 1
        while (base < wk.end_rel && base < stop_at) {
            const uint32_t c = resolve<MODE, MSPEC>(wk, w.p, base, lane);
            SEQCDC_ASSERT_CUT(base, c, w.p, wk.end_rel);
            const uint64_t cut = off + c;
            lb_push(lb, cut, dst, lane);
            base = c;
            if (cut >= stop) {
                done = true;
                break;
            }
#pragma unroll 1
            while (cut >= t_next) {
                t++;
                t_next += w.G;
            }
            if ((int64_t)t != cur.t) {
                t_lo = seg_start(w, g, t);
                t_Loff = w.single ? (uint64_t)t * w.capL1 : w.Loff[t];
            }
            int64_t idx;
            if (check_cut(w, cur, t, t_lo, t_Loff, cut, idx, lane) == CK_MERGE) {
                tgt = (int32_t)t;
                mi = idx;
                done = true;
                break;
            }
        }
        pos = off + base;
    }
    lb_flush(lb, dst, lane);
    return lb.n;
}

// Single stream: follow merges from the stream start (32 segments per step)
// and continue every valid extension that exhausted its budget; the result
// is written back as that segment's target / merge index.  One warp.
template <int MODE, int MSPEC>
__device__ void fix_overflows(const Work &w, Walker &wk, int lane)
{
    const uint32_t k = w.nseg1;
    uint32_t cur = 0;
#pragma unroll 1
    while (cur + 1 < k) {
        const uint32_t i = cur + lane;
        const int32_t t = i + 1 < k ? __ldcg(w.target + i) : 0;
        const uint32_t nb = __ballot_sync(FULL, i + 1 < k && t != (int32_t)(i + 1));
        if (!nb) {
            cur += 32;
            continue;
        }
        const uint32_t ic = cur + __ffs(nb) - 1;
        int32_t tj = __ldcg(w.target + ic);
        if (tj == TGT_OVERFLOW) {
            const Seg g = get_seg(w, ic);
            const uint64_t from = __ldcg(w.X + g.Xoff + __ldcg(w.Xcnt + ic) - 1);
            int64_t mj;
            const uint32_t n = continue_chain<MODE, MSPEC>(w, wk, g, ic, from, tj, mj, lane);
            if (lane == 0) {
                w.cont_cnt[ic] = n;
                w.target[ic] = tj;
                w.midx[ic] = mj;
            }
            __syncwarp();
        }
        if (tj < 0) break;                 // the stream (range) ends on this path
        cur = (uint32_t)tj;
    }
}

template <int MODE, int MSPEC, bool BR>
__global__ void __launch_bounds__(32, SEQCDC_MIN_BLOCKS) k_walk(Work w)
{
    __shared__ __align__(128) uint8_t ring[RING];
    const int lane = threadIdx.x;
    asm volatile("griddepcontrol.launch_dependents;");   // let k_post's CTAs queue for the tail
    Walker wk;
    walker_init(wk, ring, w.p, lane);
    const uint32_t nseg = w.ctrl[C_BAD] ? 0u : nseg_total(w);
#pragma unroll 1
    for (;;) {
        uint32_t s = 0;
        if (lane == 0) s = atomicAdd(w.ctrl + C_NEXT, 1u);
        s = __shfl_sync(FULL, s, 0);
        if (s >= nseg) break;
        walk_segment<MODE, MSPEC, BR>(w, wk, s, lane);
    }
    if (w.single) {
        // the last walker to finish continues any extension on the valid path
        // that ran out of budget (rare: phase-locked data), so k_post only
        // has to follow merges
        __syncwarp();
        uint32_t last = 0;
        if (lane == 0) {
            __threadfence();
            last = atomicAdd(w.ctrl + C_DONE, 1u) == gridDim.x - 1;
        }
        if (__shfl_sync(FULL, last, 0)) {
            __threadfence();
            if (*(volatile uint32_t *)(w.ctrl + C_OVF)) fix_overflows<MODE, MSPEC>(w, wk, lane);
        }
    }
    walker_finish(wk);
}

}  // namespace seqcdc
#include "seqcdc_lane.cuh"
namespace seqcdc {

// ------------------------------------------------------------------ 2. stitch (batches)
template <int MODE, int MSPEC>
__global__ void __launch_bounds__(1024) k_stitch(Work w)
{
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(128) uint8_t ring[RING];
    if (w.ctrl[C_BAD]) return;
    // layout: [tg[K] | mi[K] | en[K]]
    int32_t *tg = (int32_t *)sm;
    const uint32_t kmax = STITCH_MAX_SEGS;
    int64_t *mi = (int64_t *)(sm + 4 * kmax);
    int64_t *en = (int64_t *)(sm + 12 * kmax);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (uint32_t j = blockIdx.x; j < w.ns; j += gridDim.x) {
        const uint32_t f = w.single ? 0 : w.str_first[j];
        const uint32_t k = w.single ? w.nseg1 : w.str_first[j + 1] - f;
        if (k == 1) {
            if (threadIdx.x == 0) {
                w.entry[f] = -1;
                w.seg_count[f] = w.Lcnt[f] & CNT_MASK;
                w.cont_cnt[f] = 0;
            }
            continue;
        }
        for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) {
            const int32_t t = w.target[f + i];
            tg[i] = t >= 0 ? t - (int32_t)f : t;
            mi[i] = w.midx[f + i];
            en[i] = ENTRY_DEAD;
            w.cont_cnt[f + i] = 0;
        }
        __syncthreads();
        if (wid == 0) {
            // follow merges from the stream start (the only chain right from its start)
            Walker wk;
            walker_init(wk, ring, w.p, lane);
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
                int32_t tj = tg[ic];
                int64_t mj = mi[ic];
                if (tj == TGT_OVERFLOW) {             // extension budget exhausted: continue it here
                    const Seg g = get_seg(w, f + ic);
                    const uint32_t nx = w.Xcnt[f + ic];
                    const uint64_t from = __ldcg(w.X + g.Xoff + nx - 1);
                    int32_t t2;
                    const uint32_t n = continue_chain<MODE, MSPEC>(w, wk, g, f + ic, from, t2, mj, lane);
                    if (lane == 0) w.cont_cnt[f + ic] = n;
                    tj = t2 >= 0 ? t2 - (int32_t)f : t2;
                }
                if (tj < 0) break;                    // reached the end of the stream / range
                ent = mj;
                cur = (uint32_t)tj;
            }
            walker_finish(wk);
        }
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) {
            const int64_t e = en[i];
            uint64_t c = 0;
            if (e != ENTRY_DEAD)
                c = (w.Lcnt[f + i] & CNT_MASK) - (uint64_t)(e + 1) + w.Xcnt[f + i] + w.cont_cnt[f + i];
            w.seg_count[f + i] = c;
            w.entry[f + i] = e;
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
        if (e == ENTRY_DEAD) continue;
        const Seg g = get_seg(w, s);
        const uint64_t nl = lc - (uint64_t)(e + 1);
        const uint64_t *Ls = w.L + g.Loff + (e + 1);
        for (uint64_t i = lane; i < nl; i += 32) out[i] = __ldcg(Ls + i) + w.out_add;
        const uint64_t *Xs = w.X + g.Xoff;
        for (uint64_t i = lane; i < nx; i += 32) out[nl + i] = __ldcg(Xs + i) + w.out_add;
        const uint64_t nc = cnt - nl - nx;   // continuation (stitch) cuts
        if (nc) {
            const uint64_t *Cs = cont_slot(w, s, __ldcg(Xs + nx - 1));
            for (uint64_t i = lane; i < nc; i += 32) out[nl + nx + i] = __ldcg(Cs + i) + w.out_add;
        }
    }
}

// ------------------------------------------------------------------ single stream: stitch + scan + copy in one launch
// Every CTA follows the merges from the stream start and scans the per-segment
// valid counts itself (a few KB of L2 reads each: no grid-wide barrier), then
// copies its share of the segments' valid cuts to d_cuts.
__device__ void smem_scan_excl(uint64_t *a, uint32_t n)
{
    __shared__ uint64_t wsum[32];
    const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nt = blockDim.x;
    const uint32_t per = (n + nt - 1) / nt;
    const uint32_t b0 = tid * per, b1 = min(n, b0 + per);
    uint64_t loc = 0;
    for (uint32_t i = b0; i < b1; i++) loc += a[i];
    uint64_t inc = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t t = __shfl_up_sync(FULL, inc, o);
        if ((int)lane >= o) inc += t;
    }
    if (lane == 31) wsum[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        const uint64_t x = lane < nt / 32 ? wsum[lane] : 0;
        uint64_t xi = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t t = __shfl_up_sync(FULL, xi, o);
            if ((int)lane >= o) xi += t;
        }
        wsum[lane] = xi - x;
    }
    __syncthreads();
    uint64_t run = wsum[wid] + inc - loc;
    for (uint32_t i = b0; i < b1; i++) {
        const uint64_t v = a[i];
        a[i] = run;
        run += v;
    }
    __syncthreads();
}

__global__ void __launch_bounds__(1024) k_post(Work w)
{
    extern __shared__ __align__(128) uint8_t sm[];
    asm volatile("griddepcontrol.wait;" ::: "memory");   // k_walk complete and its writes visible
    const uint32_t k = w.nseg1;
    int32_t *tg = (int32_t *)sm;                          // [K]
    int64_t *en = (int64_t *)(sm + 4 * STITCH_MAX_SEGS);  // [K] entry index (-1: from the start)
    uint64_t *cnt = (uint64_t *)(sm + 12 * STITCH_MAX_SEGS);  // [K] merge index, then count, then offset
    const uint32_t tid = threadIdx.x;
    const int lane = tid & 31, wid = tid >> 5;
    int ok = 1;
    // one round of loads for everything per segment: the targets/merge indices go
    // to shared memory, the list counts stay in registers for the count pass
    // (launched with exactly 1024 threads; PER strides cover STITCH_MAX_SEGS)
    constexpr int PER = (STITCH_MAX_SEGS + 1023) / 1024;
    uint32_t lcv[PER], xcv[PER];
#pragma unroll
    for (int u = 0; u < PER; u++) {
        const uint32_t i = tid + 1024u * u;
        lcv[u] = xcv[u] = 0;
        if (i < k) {
            const int32_t t = __ldcg(w.target + i);
            const int64_t m = __ldcg(w.midx + i);
            lcv[u] = (uint32_t)(__ldcg(w.Lcnt + i) & CNT_MASK);
            xcv[u] = __ldcg(w.Xcnt + i) + __ldcg(w.cont_cnt + i);
            tg[i] = t;
            cnt[i] = (uint64_t)m;
            en[i] = ENTRY_DEAD;
            if (i + 1 < k && t != (int32_t)(i + 1)) ok = 0;
        }
    }
    ok = __syncthreads_and(ok);
    if (ok) {                                   // every extension merged into its successor
        for (uint32_t i = tid; i < k; i += blockDim.x) en[i] = i ? (int64_t)cnt[i - 1] : -1;
    } else if (wid == 0) {                      // follow the merges (some chain skipped a segment)
        uint32_t cur = 0;
        int64_t ent = -1;
#pragma unroll 1
        for (;;) {
            const uint32_t i = cur + lane;
            const int32_t t = i < k ? tg[i] : 0;
            const bool pass = (i + 1 < k) && t == (int32_t)(i + 1);
            const uint32_t nb = __ballot_sync(FULL, !pass);
            const int js = nb ? __ffs(nb) - 1 : 32;
            if (lane <= js && i < k) en[i] = lane == 0 ? ent : (int64_t)cnt[i - 1];
            if (js == 32) {
                ent = (int64_t)cnt[cur + 31];
                cur += 32;
                continue;
            }
            const uint32_t ic = cur + js;
            if (ic + 1 == k) break;
            const int32_t tj = tg[ic];
            if (tj < 0) break;                  // end of stream / range (overflows were fixed in k_walk)
            ent = (int64_t)cnt[ic];
            cur = (uint32_t)tj;
        }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < PER; u++) {
        const uint32_t i = tid + 1024u * u;
        if (i < k) {
            const int64_t e = en[i];
            SEQCDC_ASSERT(e == ENTRY_DEAD || (uint64_t)(e + 1) <= (uint64_t)lcv[u]);
            cnt[i] = e == ENTRY_DEAD ? 0 : (uint64_t)lcv[u] - (uint64_t)(e + 1) + xcv[u];
        }
    }
    __syncthreads();
    const uint64_t last = cnt[k - 1];
    smem_scan_excl(cnt, k);
    if (blockIdx.x == 0 && tid == 0) {
        if (w.tail_n && en[k - 1] == ENTRY_DEAD) *w.tail_n = 0;   // its chain is not the valid one
        const uint64_t total = cnt[k - 1] + last;
        if (w.summary) {                        // the overhang = the last valid cut (k_copy is not needed)
            uint64_t ov = w.out_add;
            for (int32_t s3 = (int32_t)k - 1; s3 >= 0; s3--) {
                const int64_t e = en[s3];
                if (e == ENTRY_DEAD) continue;
                const uint64_t nc = __ldcg(w.cont_cnt + s3), nx = __ldcg(w.Xcnt + s3);
                const uint64_t lc = __ldcg(w.Lcnt + s3) & CNT_MASK;
                const Seg g = get_seg(w, s3);
                if (nc) ov = __ldcg(cont_slot(w, s3, __ldcg(w.X + g.Xoff + nx - 1)) + nc - 1) + w.out_add;
                else if (nx) ov = __ldcg(w.X + g.Xoff + nx - 1) + w.out_add;
                else if (lc > (uint64_t)(e + 1)) ov = __ldcg(w.L + g.Loff + lc - 1) + w.out_add;
                else continue;
                break;
            }
            w.summary[0] = ov;
            w.summary[1] = total;
        }
        w.cut_index[0] = 0;
        w.cut_index[1] = total;
        *w.ncuts = total;
    }
    if (blockIdx.x == 0 && w.push_blk) {
        // fused exchange: this range's block goes straight into the next range's
        // mailbox over peer memory (NVLink), then the flag is released at system
        // scope; the next range's merge kernel acquires it (SURVEY 8(e) fused form)
        __syncthreads();                        // thread 0's summary / tail_n writes
        const uint64_t tn = w.tail_n ? min(*(volatile uint64_t *)w.tail_n, (uint64_t)w.tail_max) : 0;
        for (uint32_t i = tid; i < 3 + tn; i += blockDim.x)
            w.push_blk[i] = i == 0 ? w.summary[0] : i == 1 ? w.summary[1] : i == 2 ? tn : __ldcg(w.tail + (i - 3));
        __syncthreads();
        if (tid == 0) {
            __threadfence_system();
            asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(w.push_flag), "l"(w.push_value) : "memory");
        }
    }
    // copy: one warp per segment
    const uint32_t nw = gridDim.x * (blockDim.x >> 5);
    for (uint32_t s2 = blockIdx.x * (blockDim.x >> 5) + wid; s2 < k; s2 += nw) {
        const int64_t e = en[s2];
        if (e == ENTRY_DEAD) continue;
        const Seg g = get_seg(w, s2);
        uint64_t *out = w.cuts + cnt[s2];
        const uint64_t lc = __ldcg(w.Lcnt + s2) & CNT_MASK, nx = __ldcg(w.Xcnt + s2), nc = __ldcg(w.cont_cnt + s2);
        const uint64_t nl = lc - (uint64_t)(e + 1);
        const uint64_t *Ls = w.L + g.Loff + (e + 1);
        const uint64_t add = w.out_add;
        // speculative list then extension list, 8 loads in flight per lane before
        // their stores (one memory round trip per 256 cuts instead of per 32)
        const uint64_t *Xs = w.X + g.Xoff;
#pragma unroll 1
        for (uint64_t i0 = 0; i0 < nl + nx; i0 += 256) {
            uint64_t v[8];
#pragma unroll
            for (int u = 0; u < 8; u++) {
                const uint64_t i = i0 + 32 * u + lane;
                v[u] = i < nl ? __ldcg(Ls + i) : (i < nl + nx ? __ldcg(Xs + (i - nl)) : 0);
            }
#pragma unroll
            for (int u = 0; u < 8; u++) {
                const uint64_t i = i0 + 32 * u + lane;
                if (i < nl + nx) out[i] = v[u] + add;
            }
        }
        if (nc) {
            const uint64_t *Cs = cont_slot(w, s2, __ldcg(Xs + nx - 1));
            for (uint64_t i = lane; i < nc; i += 32) out[nl + nx + i] = __ldcg(Cs + i) + add;
        }
    }
}

// ------------------------------------------------------------------ many segments (lane walker): post in two launches
// k_lpost (one CTA): which segments lie on the valid chain, each one's entry and
// valid count, the exclusive scan of the counts; k_lcopy (grid): the copy.
// A segment's extension merges into the next segment's chain except when it ran
// through it without meeting a common cut (a "jumper": target != s+1); the
// valid path from segment 0 only changes at jumpers, so it is followed over the
// (few) jumpers alone: jumper j is on the path iff the path has not already
// jumped past it; a live jumper kills the segments strictly between it and its
// target and gives its target the entry midx[j].  Everything else is parallel.
constexpr uint32_t LP_JCAP = 8192;                 // jumpers followed from shared memory
constexpr uint32_t LP_MAX_SEGS = 180000;           // (planning cap on lane-walker segments)
constexpr uint32_t LP_SMEM = 4 * LP_JCAP;
constexpr uint32_t LS_MAX_TILES = 64;              // >= LP_MAX_SEGS / (512 * 8)

__device__ __forceinline__ uint32_t tgt_of(const Work &w, uint32_t i, uint32_t k)
{
    const int32_t t = __ldcg(w.target + i);
    return t >= 0 ? (uint32_t)t : k;               // the stream (range) end
}

// Block-wide exclusive scan of one value per thread (512 threads = 16 warps);
// returns the exclusive prefix, *tot the block total.
template <typename T>
__device__ __forceinline__ T block_excl(T v, T *ws, T &tot)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    T inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T t = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) ws[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        const T x = lane < nw ? ws[lane] : 0;
        T xi = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const T t = __shfl_up_sync(FULL, xi, o);
            if (lane >= o) xi += t;
        }
        ws[lane] = xi - x;
        if (lane == 31) ws[32] = xi;
    }
    __syncthreads();
    const T r = ws[wid] + inc - v;
    tot = ws[32];
    __syncthreads();
    return r;
}

constexpr uint32_t LP_TILE = 512, LP_BATCH = 8;   // one segment per thread per tile, 8 tiles per load round


// Exclusive scan of LP_BATCH values per thread taken tile by tile (value u of
// thread t is element u * blockDim + t): warp scans per tile, one combine of
// the LP_BATCH x 16 warp totals (tile-major) by warp 0, two barriers in all.
// Returns the prefixes in ex[], the batch total in tot.
template <typename T>
__device__ __forceinline__ void batch_excl(const T (&v)[LP_BATCH], T (&ex)[LP_BATCH], T *wt, T &tot)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    T inc[LP_BATCH];
#pragma unroll
    for (uint32_t u = 0; u < LP_BATCH; u++) {
        T x = v[u];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const T t = __shfl_up_sync(FULL, x, o);
            if (lane >= o) x += t;
        }
        inc[u] = x;
        if (lane == 31) wt[u * nw + wid] = x;
    }
    __syncthreads();
    if (wid == 0) {                                 // tile-major exclusive scan of the warp totals
        const uint32_t m = LP_BATCH * nw;           // <= 8 x 32
        T carry = 0;
        for (uint32_t b = 0; b < m; b += 32) {
            const T x = b + lane < m ? wt[b + lane] : 0;
            T xi = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const T t = __shfl_up_sync(FULL, xi, o);
                if (lane >= o) xi += t;
            }
            if (b + lane < m) wt[b + lane] = carry + xi - x;
            carry += __shfl_sync(FULL, xi, 31);
        }
        if (lane == 0) wt[m] = carry;
    }
    __syncthreads();
#pragma unroll
    for (uint32_t u = 0; u < LP_BATCH; u++) ex[u] = wt[u * nw + wid] + inc[u] - v[u];
    tot = wt[LP_BATCH * nw];
    __syncthreads();
}

__global__ void __launch_bounds__(512) k_lpost(Work w)
{
    extern __shared__ __align__(128) uint8_t sm[];
    asm volatile("griddepcontrol.wait;" ::: "memory");   // the walk complete and its writes visible
    const uint32_t k = w.nseg1;
    uint32_t *jl = (uint32_t *)sm;                 // [LP_JCAP] jumpers in ascending order
    __shared__ uint32_t ws32[LP_BATCH * 16 + 1];
    const uint32_t tid = threadIdx.x;
    const int lane = tid & 31, wid = tid >> 5;
    // A. jumpers (target != s + 1), in ascending order: coalesced tiles, order-
    // preserving compaction per tile; every entry reset to "from midx[s-1]"
    uint32_t nj = 0;
    for (uint32_t base = 0; base < k; base += LP_TILE * LP_BATCH) {
        int32_t t8[LP_BATCH];
#pragma unroll
        for (uint32_t u = 0; u < LP_BATCH; u++) {
            const uint32_t i = base + u * LP_TILE + tid;
            t8[u] = i < k ? __ldcg(w.target + i) : 0;
        }
        uint32_t jp[LP_BATCH], ex[LP_BATCH], tot;
#pragma unroll
        for (uint32_t u = 0; u < LP_BATCH; u++) {
            const uint32_t i = base + u * LP_TILE + tid;
            const uint32_t t = t8[u] >= 0 ? (uint32_t)t8[u] : k;
            jp[u] = i + 1 < k && t != i + 1;
            if (i < k) w.entry[i] = ENTRY_UNSET;
        }
        batch_excl<uint32_t>(jp, ex, ws32, tot);
#pragma unroll
        for (uint32_t u = 0; u < LP_BATCH; u++)
            if (jp[u] && nj + ex[u] < LP_JCAP) jl[nj + ex[u]] = base + u * LP_TILE + tid;
        nj += tot;
    }
    __syncthreads();
    // B. follow the valid path over the jumpers (one warp): a live jumper's
    // target takes its entry from the jumper, the segments in between are dead
    if (wid == 0) {
        uint32_t state = 0;                        // the next segment on the path
        if (nj <= LP_JCAP) {
            for (uint32_t base = 0; base < nj; base += 32) {
                const uint32_t idx = base + lane;
                const uint32_t j = idx < nj ? jl[idx] : FULL;
                const uint32_t t = idx < nj ? tgt_of(w, j, k) : k;
                uint32_t livem = 0;
                const uint32_t m = min(32u, nj - base);
                for (uint32_t l = 0; l < m; l++) {
                    const uint32_t jj = __shfl_sync(FULL, j, l), tt = __shfl_sync(FULL, t, l);
                    if (state <= jj) {             // the path reaches jumper jj: it is live
                        state = tt;
                        livem |= 1u << l;
                    }
                }
                if ((livem >> lane) & 1u) {
                    for (uint32_t i = j + 1; i < t && i < k; i++) w.entry[i] = ENTRY_DEAD;
                    if (t < k) w.entry[t] = __ldcg(w.midx + j);
                }
                __syncwarp();
            }
        } else {                                   // many jumpers: follow segment by segment
            uint32_t cur = 0;
            while (cur + 1 < k) {
                const uint32_t i = cur + lane;
                const bool pass = i + 1 < k && tgt_of(w, i, k) == i + 1;
                const uint32_t nb = __ballot_sync(FULL, !pass);
                if (!nb) {
                    cur += 32;
                    continue;
                }
                const uint32_t ic = cur + __ffs(nb) - 1;
                if (ic + 1 >= k) break;
                const uint32_t t = tgt_of(w, ic, k);
                for (uint32_t x = ic + 1 + lane; x < t && x < k; x += 32) w.entry[x] = ENTRY_DEAD;
                if (lane == 0 && t < k) w.entry[t] = __ldcg(w.midx + ic);
                __syncwarp();
                if (t >= k) break;
                cur = t;
            }
        }
    }
}

// C. entries, valid counts and their exclusive scan, in tiles of LS_TILE
// segments (one CTA each, all resident), chained by a decoupled look-back over
// the tile status words (value << 2 | 1: tile total, | 2: inclusive prefix).
// The last tile also writes the totals, the range summary and the tail check.
constexpr uint32_t LS_TILE = LP_TILE * LP_BATCH;

__global__ void __launch_bounds__(512) k_lscan(Work w)
{
    __shared__ uint64_t ws64[LP_BATCH * 16 + 1];
    __shared__ uint64_t s_pre;
    const uint32_t k = w.nseg1, tid = threadIdx.x, tile = blockIdx.x;
    const uint32_t base = tile * LS_TILE;
    int64_t e8[LP_BATCH], m8[LP_BATCH];
    uint64_t l8[LP_BATCH];
    uint32_t x8[LP_BATCH], c8[LP_BATCH];
#pragma unroll
    for (uint32_t u = 0; u < LP_BATCH; u++) {
        const uint32_t i = base + u * LP_TILE + tid;
        const bool in = i < k;
        e8[u] = in ? __ldcg(w.entry + i) : ENTRY_DEAD;
        m8[u] = in && i > 0 ? __ldcg(w.midx + i - 1) : -1;
        l8[u] = in ? __ldcg(w.Lcnt + i) & CNT_MASK : 0;
        x8[u] = in ? __ldcg(w.Xcnt + i) : 0;
        c8[u] = in ? __ldcg(w.cont_cnt + i) : 0;
    }
    uint64_t cv[LP_BATCH], ex[LP_BATCH], tot;
#pragma unroll
    for (uint32_t u = 0; u < LP_BATCH; u++) {
        const uint32_t i = base + u * LP_TILE + tid;
        uint64_t c = 0;
        if (i < k) {
            int64_t e = e8[u];
            if (e == ENTRY_UNSET) e = i == 0 ? -1 : m8[u];
            if (e != ENTRY_DEAD) {
                SEQCDC_ASSERT((uint64_t)(e + 1) <= l8[u]);
                c = l8[u] - (uint64_t)(e + 1) + x8[u] + c8[u];
            }
            w.entry[i] = e;
            w.seg_count[i] = c;
        }
        cv[u] = c;
    }
    batch_excl<uint64_t>(cv, ex, ws64, tot);       // (its barriers order the writes above before the publish)
    if (tid == 0) {
        __threadfence();
        uint64_t pre = 0;
        if (tile == 0) {
            st_release_u64(w.lstat, (tot << 2) | 2u);
        } else {
            st_release_u64(w.lstat + tile, (tot << 2) | 1u);
#pragma unroll 1
            for (int32_t j = (int32_t)tile - 1; j >= 0; j--) {
                uint64_t v;
#pragma unroll 1
                while (((v = ld_acquire_u64(w.lstat + j)) & 3u) == 0) __nanosleep(32);
                pre += v >> 2;
                if (v & 2u) break;
            }
            st_release_u64(w.lstat + tile, ((pre + tot) << 2) | 2u);
        }
        s_pre = pre;
    }
    __syncthreads();
    const uint64_t pre = s_pre;
#pragma unroll
    for (uint32_t u = 0; u < LP_BATCH; u++) {
        const uint32_t i = base + u * LP_TILE + tid;
        if (i < k) w.seg_out[i] = pre + ex[u];
    }
    if (tile == gridDim.x - 1 && tid == 0) {
        const uint64_t total = pre + tot;
        if (w.tail_n && k && __ldcg(w.entry + k - 1) == ENTRY_DEAD) *w.tail_n = 0;   // the last chain is not the valid one
        if (w.summary) {                                      // the overhang = the last valid cut
            uint64_t ov = w.out_add;
            for (int32_t s3 = (int32_t)k - 1; s3 >= 0; s3--) {
                const int64_t e = __ldcg(w.entry + s3);
                if (e == ENTRY_DEAD) continue;
                const uint64_t nc = __ldcg(w.cont_cnt + s3), nx = __ldcg(w.Xcnt + s3);
                const uint64_t lc = __ldcg(w.Lcnt + s3) & CNT_MASK;
                const Seg g = get_seg(w, s3);
                if (nc) ov = __ldcg(cont_slot(w, s3, __ldcg(w.X + g.Xoff + nx - 1)) + nc - 1) + w.out_add;
                else if (nx) ov = __ldcg(w.X + g.Xoff + nx - 1) + w.out_add;
                else if (lc > (uint64_t)(e + 1)) ov = __ldcg(w.L + g.Loff + lc - 1) + w.out_add;
                else continue;
                break;
            }
            w.summary[0] = ov;
            w.summary[1] = total;
        }
        w.cut_index[0] = 0;
        w.cut_index[1] = total;
        *w.ncuts = total;
    }
}

// one warp per segment, 8 loads in flight per lane before their stores
__global__ void __launch_bounds__(256) k_lcopy(Work w)
{
    const uint32_t k = w.nseg1;
    const int lane = threadIdx.x & 31;
    const uint32_t nw = gridDim.x * (blockDim.x >> 5);
    for (uint32_t s2 = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); s2 < k; s2 += nw) {
        const int64_t e = __ldcg(w.entry + s2);
        if (e == ENTRY_DEAD) continue;
        const Seg g = get_seg(w, s2);
        uint64_t *out = w.cuts + __ldcg(w.seg_out + s2);
        const uint64_t lc = __ldcg(w.Lcnt + s2) & CNT_MASK, nx = __ldcg(w.Xcnt + s2), nc = __ldcg(w.cont_cnt + s2);
        const uint64_t nl = lc - (uint64_t)(e + 1);
        const uint64_t *Ls = w.L + g.Loff + (e + 1);
        const uint64_t *Xs = w.X + g.Xoff;
        const uint64_t add = w.out_add;
#pragma unroll 1
        for (uint64_t i0 = 0; i0 < nl + nx; i0 += 256) {
            uint64_t v[8];
#pragma unroll
            for (int u = 0; u < 8; u++) {
                const uint64_t i = i0 + 32 * u + lane;
                v[u] = i < nl ? __ldcg(Ls + i) : (i < nl + nx ? __ldcg(Xs + (i - nl)) : 0);
            }
#pragma unroll
            for (int u = 0; u < 8; u++) {
                const uint64_t i = i0 + 32 * u + lane;
                if (i < nl + nx) out[i] = v[u] + add;
            }
        }
        if (nc) {
            const uint64_t *Cs = cont_slot(w, s2, __ldcg(Xs + nx - 1));
            for (uint64_t i = lane; i < nc; i += 32) out[nl + nx + i] = __ldcg(Cs + i) + add;
        }
    }
}

// an empty range's exchange block (no walk ran): [overhang, 0, 0] + flag
__global__ void k_push_empty(uint64_t *blk, uint64_t *flag, uint64_t ov, uint64_t value)
{
    blk[0] = ov;
    blk[1] = 0;
    blk[2] = 0;
    __threadfence_system();
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(value) : "memory");
}

#ifdef SEQCDC_DEBUG
// debug builds: the finished cut list is strictly increasing and positive
__global__ void k_debug_sorted(const uint64_t *cuts, const uint64_t *ncuts)
{
    const uint64_t k = *ncuts;
    if (k == SEQCDC_NCUTS_BAD_INPUT) return;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k; i += (uint64_t)gridDim.x * blockDim.x)
        SEQCDC_ASSERT(cuts[i] > 0 && (i == 0 || cuts[i] > cuts[i - 1]));
}
#endif

__global__ void k_set2(uint64_t *p, uint64_t a, uint64_t b)
{
    p[0] = a;
    p[1] = b;
}

__global__ void k_empty(uint64_t *cut_index, uint64_t *ncuts)
{
    cut_index[0] = 0;
    *ncuts = 0;
}


// ------------------------------------------------------------------ host side
struct Plan {
    uint64_t G, nseg_max, L_items, X_items, FB_items;
    uint32_t nseg1, capL1, capX1;
    size_t bytes;
    size_t o_ctrl, o_Lcnt, o_str_first, o_cont_cnt, o_seg_lo, o_seg_hi, o_seg_stream, o_Loff, o_Xoff,
        o_Lcap, o_Xcap, o_Xcnt, o_target, o_midx, o_entry, o_seg_count, o_seg_out, o_L, o_X, o_FB, o_hand;
    uint32_t walk_grid;
    bool lane;             // single stream on the lane walker (k_lwalk + k_lpost + k_lscan + k_lcopy)
    uint64_t lane_slots;   // lanes the lane walker could run (SMs x CTAs x threads)
};

static std::atomic<uint64_t> g_launches{0};   // kernels this library has launched (process-wide)
static uint64_t g_force_G = 0;
static std::mutex g_mu;
static cudaMemPool_t g_pool[64];
static bool g_pool_ok[64];

constexpr uint32_t STITCH_SMEM = 20 * STITCH_MAX_SEGS;

template <int MODE, int MSPEC>
static void set_attrs()
{
    cudaFuncSetAttribute((const void *)k_stitch<MODE, MSPEC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         STITCH_SMEM);
}

template <int MODE>
static void set_attrs_mode()
{
    set_attrs<MODE, 4>();
    set_attrs<MODE, 0>();
    set_attrs<MODE, -1>();
}

static int env_int(const char *name, int dflt)
{
    const char *e = getenv(name);
    return e ? atoi(e) : dflt;
}

// Ring geometry of the warp walker (fixed in this build; reported by build_info).
static void ring_geometry(const seqcdc_params_t *, DevParams &d)
{
    d.bs = BLK_SHIFT;
    d.nb = NBLK;
    d.ah = AHEAD;
}

// Per device: SM count, occupancies, and the function attributes (dynamic
// shared memory opt-ins are per device context, so they are set once for every
// device a process uses).
struct DevInfo {
    int sms = 0;
    int occ_warp = 0;      // warp-walker CTAs (one warp each) per SM
    int occ_lane = 0;      // lane-walker CTAs per SM
};
static DevInfo g_dev[64];
static int g_last_occ;
static int g_last_lane;            // the last single-stream call used the lane walker
static uint32_t g_last_nseg;       // ... with this many segments

static int device_info(int &sms, int &occ, int *occ_lane = nullptr)
{
    int dev;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return SEQCDC_ECUDA;
    std::lock_guard<std::mutex> lk(g_mu);
    DevInfo &d = g_dev[dev];
    if (!d.sms) {
        int nsm = 0;
        if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return SEQCDC_ECUDA;
        set_attrs_mode<0>();
        set_attrs_mode<1>();
        set_attrs_mode<2>();
        set_attrs_mode<3>();
        cudaFuncSetAttribute((const void *)k_post, cudaFuncAttributeMaxDynamicSharedMemorySize, STITCH_SMEM);
        cudaFuncSetAttribute((const void *)k_lpost, cudaFuncAttributeMaxDynamicSharedMemorySize, LP_SMEM);
        int o = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_walk<0, 4, true>, 32, 0) != cudaSuccess)
            return SEQCDC_ECUDA;
        // 24 walkers per SM measured best (25 -- the smem limit -- leaves almost no L1
        // and runs ~25% slower on config 2; profiles/r01/sweeps.md)
        d.occ_warp = std::max(1, std::min(o, 24));
        int ol = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ol, k_lwalk<0, true>, lw::THREADS, 0) != cudaSuccess)
            return SEQCDC_ECUDA;
        d.occ_lane = std::max(1, ol);
        d.sms = nsm;
    }
    sms = d.sms;
    occ = d.occ_warp;
    const int v = env_int("SEQCDC_WALKERS_PER_SM", 0);
    if (v > 0 && v < occ) occ = v;
    if (occ_lane) *occ_lane = d.occ_lane;
    return SEQCDC_OK;
}

// Which walker a single-stream call uses: the lane walker (skip-aware sparse
// reads) for long streams with M <= 4 favourable pairs per run (every Table I
// row), the warp walker otherwise.  SEQCDC_WALKER=warp|lane forces one (tests).
static bool use_lane_walker(uint64_t total, const seqcdc_params_t *p, bool single)
{
    if (!single) return false;
    const uint32_t M = p->seq_length - ((p->flags & SEQCDC_FLAG_PAIRS) ? 0u : 1u);
    if (M > 4) return false;
    const char *e = getenv("SEQCDC_WALKER");
    if (e && !strcmp(e, "lane")) return true;
    if (e && !strcmp(e, "warp")) return false;
    // long chunks (max > 16 KiB) merge only after ~65+ chunks: segments would
    // have to be far longer than the lanes allow (config 4: 4x slower)
    if (p->max_size > 16384) return false;
    if (e && !strcmp(e, "warp")) return false;
    if (e && !strcmp(e, "lane")) return true;
    // it needs ~75k lanes with segments several merge distances long, i.e. a
    // stream of >= 16 GiB, to beat the warp walker (profiles/r02/lane_ab_v10.jsonl:
    // 16 GiB ramp mix 2.48 vs 2.82 ms, 8 GiB 2.21 vs 1.51 ms)
    const int mib = env_int("SEQCDC_LW_MIN_MIB", 16 << 10);
    return mib >= 0 && total >= ((uint64_t)mib << 20);
}

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
// lane walker: the hand-off task list (<= 2 tasks per segment), k_lscan's tile
// status words, the claim words of handed-off speculative parts -- all zeroed
static size_t lstat_off(uint64_t S) { return align_up(4 * (2 * S + S / 32 + 8), 8); }
static size_t lclaim_off(uint64_t S) { return lstat_off(S) + 8 * LS_MAX_TILES; }
static size_t lzero_end(uint64_t S) { return lclaim_off(S) + 4 * S; }

static void make_plan(uint64_t total, uint32_t ns, const seqcdc_params_t *p, int sms, int occ, Plan &pl,
                      bool single, uint64_t stop, bool short_tail = false, int occ_lane = 0)
{
    pl.lane = occ_lane > 0;
    // up to ~1.5 GiB the run ends with the longest seam extension, and 22 walkers
    // per SM (longer segments, less contention on the tail) measured ~4% faster
    // than 24 on config 2; larger inputs are throughput-bound (profiles/r01/sweeps.md)
    const int occ_eff = (total <= (3ull << 29) && occ > 22 && !getenv("SEQCDC_WALKERS_PER_SM")) ? 22 : occ;
    const uint64_t walkers = (uint64_t)sms * occ_eff;
    const uint64_t mx = p->max_size, mn = p->min_size;
    // segments per walker (x100; tuning knob) and the segment floor in max_size units
    // Batches of streams: two segments per walker for the 4 and 8 KiB rows (the
    // second wave is claimed by whichever walkers finish first, which evens out
    // the warp-slot unfairness: config 3 4 KiB row +15%, 8 KiB +10%); one for
    // larger rows, whose long merge distances make the extra seams cost more
    // (16 KiB row -8% at two).  A single stream keeps one: its overflowing
    // extensions are continued by one warp (profiles/r01/sweeps.md).
    const int spw_default = (!single && p->min_size <= 4096) ? 200 : 100;
    const uint64_t spw = (uint64_t)std::max(1, env_int("SEQCDC_SEGS_PER_WALKER_X100", spw_default));
    const uint64_t floor_chunks = (uint64_t)std::max(1, env_int("SEQCDC_G_FLOOR_CHUNKS", (int)G_FLOOR_CHUNKS));
    uint64_t denom = walkers > 2ull * ns ? walkers - ns : std::max<uint64_t>(walkers / 2, 1);
    denom = std::max<uint64_t>(1, denom * spw / 100);
    uint64_t G = (total + denom - 1) / denom;
    G = std::max<uint64_t>(G, floor_chunks * mx);
    if (pl.lane) {
        // lane walker: one segment per lane, all lanes resident at once; the floor
        // keeps a segment several merge distances long (SURVEY.md [MC-3])
        const uint64_t ctas = (uint64_t)std::max(1, std::min(occ_lane, env_int("SEQCDC_LW_CTAS_PER_SM", 5)));
        const uint64_t lanes = (uint64_t)sms * ctas * lw::THREADS;
        pl.lane_slots = lanes;
        G = std::max<uint64_t>((total + lanes - 1) / lanes,
                               (uint64_t)std::max(1, env_int("SEQCDC_LW_G_FLOOR_CHUNKS", 24)) * mx);
        G = std::max<uint64_t>(G, (total + LP_MAX_SEGS - 3) / (LP_MAX_SEGS - 2));
    }
    if (g_force_G) G = std::max<uint64_t>(g_force_G, mx);
    G = std::min<uint64_t>(G, std::max<uint64_t>(G_CEIL, mx));
    G = (G + mx - 1) / mx * mx;
    if (single && short_tail) {
        // range call with a tail: the last segment's walker also continues the
        // chain past the range end (~96 chunks), so give it a third of a segment
        const uint64_t ns1 = stop <= G ? 1 : (stop + G - 1) / G;
        if (ns1 >= 3) {
            const uint64_t Gt = (stop - G / 3 + (ns1 - 1) - 1) / (ns1 - 1);
            if (Gt * (ns1 - 1) < stop && Gt >= mx) G = Gt;
        }
    }
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
    pl.FB_items = total / mn + ns + pl.nseg_max + 2;
    pl.walk_grid = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(pl.nseg_max, walkers));
    if (pl.lane) pl.walk_grid = (uint32_t)((pl.nseg1 + lw::THREADS - 1) / lw::THREADS);
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
    pl.o_hand = o;  // lane walker task list, also reset by that memset
    o = align_up(o + (pl.lane ? lzero_end(S) : 0), 256);
    pl.o_str_first = take(4ull * (ns + 1));
    pl.o_cont_cnt = take(4 * S);
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

static void launch_pdl(const void *fn, dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl, const Work &w)
{
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    void *args[] = {(void *)&w};
    cudaLaunchKernelExC(&cfg, fn, args);
}

template <int MODE>
static void launch_lane(const Work &w, const Plan &pl, int sms, cudaStream_t st, ProfRec *pr)
{
    prof_mark(pr, 1, st);
    if (w.p.M == 4) k_lwalk<MODE, true><<<pl.walk_grid, lw::THREADS, 0, st>>>(w);
    else k_lwalk<MODE, false><<<pl.walk_grid, lw::THREADS, 0, st>>>(w);
    // handed-off extensions / tail on warps, then the post; both wait on the
    // device (griddepcontrol.wait) for their predecessor: launched early
    prof_mark(pr, 2, st);
    const void *hand = w.p.M == 4 ? (const void *)k_lhand<MODE, 4> : (const void *)k_lhand<MODE, 0>;
    const bool pdl = pr == nullptr && !getenv("SEQCDC_NO_PDL");     // (debug knob: plain launches)
    launch_pdl(hand, dim3(std::max(1, sms * 16)), dim3(32), 0, st, pdl, w);
    launch_pdl((const void *)k_lpost, dim3(1), dim3(512), LP_SMEM, st, pdl, w);
    k_lscan<<<std::max<uint32_t>(1, (pl.nseg1 + LS_TILE - 1) / LS_TILE), 512, 0, st>>>(w);
    g_launches++;
    if (w.tail_max || w.push_blk) {            // range calls: the tail from the true overhang, the push
        const void *tl = w.p.M == 4 ? (const void *)k_ltail<MODE, 4> : (const void *)k_ltail<MODE, 0>;
        launch_pdl(tl, dim3(1), dim3(32), 0, st, pdl, w);
        g_launches++;
    }
    k_lcopy<<<std::max(1, sms * 8), 256, 0, st>>>(w);
    g_launches += 4;
}

template <int MODE, int MSPEC>
static void launch_all(const Work &w, const Plan &pl, int sms, cudaStream_t st, ProfRec *pr)
{
    if (pl.lane) {
        launch_lane<MODE>(w, pl, sms, st, pr);
        return;
    }
    prof_mark(pr, 1, st);
    if (w.single) k_walk<MODE, MSPEC, true><<<pl.walk_grid, 32, walker_smem(w.p), st>>>(w);
    else k_walk<MODE, MSPEC, false><<<pl.walk_grid, 32, walker_smem(w.p), st>>>(w);
    g_launches++;
    prof_mark(pr, 2, st);
    if (w.single) {
        // programmatic dependent launch: k_post's CTAs become resident on SMs the
        // walk's tail leaves idle and wait (griddepcontrol.wait) for its completion
        const uint32_t pgrid = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(sms, (w.nseg1 + 31) / 32));
        cudaLaunchConfig_t cfg;
        memset(&cfg, 0, sizeof(cfg));
        cfg.gridDim = dim3(pgrid);
        cfg.blockDim = dim3(1024);
        cfg.dynamicSmemBytes = 20 * STITCH_MAX_SEGS;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = pr ? 0 : 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, k_post, w);
        g_launches++;
        return;
    }
    const uint32_t sgrid = (uint32_t)std::min<uint64_t>(w.ns, 2ull * sms);
    k_stitch<MODE, MSPEC><<<sgrid, 1024, STITCH_SMEM, st>>>(w);
    k_scan<<<1, 1024, 0, st>>>(w);
    k_copy<<<std::max(1, sms * 4), 256, 0, st>>>(w);
    g_launches += 3;
}

struct TailReq {
    uint64_t *tail = nullptr, *tail_n = nullptr;
    uint32_t max = 0;
    uint64_t *summary = nullptr;
    uint64_t *push_blk = nullptr, *push_flag = nullptr;
    uint64_t push_value = 0;
};

template <int MODE>
static void launch_ms(int ms, const Work &w, const Plan &pl, int sms, cudaStream_t st, ProfRec *pr)
{
    if (ms == 4) launch_all<MODE, 4>(w, pl, sms, st, pr);
    else if (ms == 0) launch_all<MODE, 0>(w, pl, sms, st, pr);
    else launch_all<MODE, -1>(w, pl, sms, st, pr);
}

static int run(const uint8_t *d_in, const uint64_t *d_offsets, uint32_t ns, uint64_t total, uint64_t stop,
               uint64_t out_add, const seqcdc_params_t *p, const DevParams &geo, uint64_t *d_cuts, uint64_t *d_cut_index,
               uint64_t *d_ncuts, uint8_t *ws, size_t ws_bytes, const Plan &pl, int sms, cudaStream_t st,
               bool single, const TailReq &tail)
{
    if (ws_bytes < pl.bytes) return SEQCDC_ENOMEM;
    if (total / pl.G + 2 > (pl.lane ? LP_MAX_SEGS : STITCH_MAX_SEGS)) return SEQCDC_EINVAL;  // post smem limits
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
    w.p.M = p->seq_length - ((p->flags & SEQCDC_FLAG_PAIRS) ? 0u : 1u);   // favourable pairs per run (c1)
    w.p.mn = (uint32_t)p->min_size;
    w.p.mx = (uint32_t)p->max_size;
    w.p.mnL = (uint32_t)p->min_size - p->seq_length;
    w.p.bs = geo.bs;
    w.p.nb = geo.nb;
    w.p.ah = geo.ah;
    w.ctrl = (uint32_t *)(ws + pl.o_ctrl);
    w.Lcnt = (uint64_t *)(ws + pl.o_Lcnt);
    w.str_first = (uint32_t *)(ws + pl.o_str_first);
    w.cont_cnt = (uint32_t *)(ws + pl.o_cont_cnt);
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
    w.hand = pl.lane ? (uint32_t *)(ws + pl.o_hand) : nullptr;
    w.lstat = pl.lane ? (uint64_t *)(ws + pl.o_hand + lstat_off(pl.nseg_max)) : nullptr;
    w.lclaim = pl.lane ? (uint32_t *)(ws + pl.o_hand + lclaim_off(pl.nseg_max)) : nullptr;
    // lane extensions longer than this many cuts go to warps: 40 when the segments
    // fill (>= 3/4 of) the lane slots (config 5: 24 -> 4.94 ms, 40 -> 4.80, 64 -> 4.97;
    // 32 GiB ramp mix: 24 -> 3.49, 40 -> 3.38), else 24 (16 GiB, 46% of the slots:
    // 24 -> 2.51 ms, 40 -> 2.71)
    w.lw_ext_cap = (uint32_t)std::max(
        1, env_int("SEQCDC_LW_EXT_CAP", pl.lane && 4ull * pl.nseg1 >= 3ull * pl.lane_slots ? 40 : 24));
    {   // late lanes: after SEQCDC_LW_LATE_PCT percent of the lanes finished their speculative part
        const int pct = env_int("SEQCDC_LW_LATE_PCT", 0);   // off: measured slower (cfg5 6.0 vs 4.9 ms at 90)
        w.lw_late = pl.lane && pct > 0 && pct < 100 ? (uint32_t)std::max<uint64_t>(1, pl.nseg1 * (uint64_t)pct / 100) : 0;
        const int pe = env_int("SEQCDC_LW_LATE_EXT_PCT", 0);
        w.lw_late_ext = pl.lane && pe > 0 && pe < 100 ? (uint32_t)std::max<uint64_t>(1, pl.nseg1 * (uint64_t)pe / 100) : 0;
    }
    w.ext_segs = (uint32_t)std::min<int>(K_EXT, std::max(1, env_int("SEQCDC_EXT_SEGS", (int)K_EXT)));
    w.cuts = d_cuts;
    w.cut_index = d_cut_index;
    w.ncuts = d_ncuts;
    w.tail = tail.tail;
    w.tail_n = tail.tail_n;
    w.tail_max = tail.max;
    w.summary = tail.summary;
    w.push_blk = tail.push_blk;
    w.push_flag = tail.push_flag;
    w.push_value = tail.push_value;
    if (tail.max && cudaMemsetAsync(tail.tail_n, 0, 8, st) != cudaSuccess) return SEQCDC_ECUDA;

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
        const size_t zb = pl.lane ? pl.o_hand - pl.o_ctrl + lzero_end(pl.nseg_max)
                                  : pl.o_Lcnt - pl.o_ctrl + 8 * pl.nseg1;
        if (cudaMemsetAsync(ws + pl.o_ctrl, 0, zb, st) != cudaSuccess)
            return SEQCDC_ECUDA;
    } else {
        k_setup<<<1, 1024, 0, st>>>(w);
        g_launches++;
    }
    const int ms = w.p.M == 4 ? 4 : (w.p.M < 4 ? 0 : -1);
    // MODE: bit 0 = Decreasing, bit 1 = signed-byte reading (flag)
    switch (p->mode | ((p->flags & SEQCDC_FLAG_SIGNED) ? 2u : 0u)) {
    case 0: launch_ms<0>(ms, w, pl, sms, st, pr); break;
    case 1: launch_ms<1>(ms, w, pl, sms, st, pr); break;
    case 2: launch_ms<2>(ms, w, pl, sms, st, pr); break;
    default: launch_ms<3>(ms, w, pl, sms, st, pr); break;
    }
#ifdef SEQCDC_DEBUG
    if (w.single && w.cuts) k_debug_sorted<<<sms, 256, 0, st>>>(w.cuts, w.ncuts);
#endif
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
                   uint64_t *d_ncuts, void *d_ws, size_t ws_bytes, cudaStream_t st, bool single_api,
                   const TailReq &tail = TailReq())
{
    DevParams geo;
    ring_geometry(p, geo);
    int sms, occ, occ_lane;
    int rc = device_info(sms, occ, &occ_lane);
    if (rc) return rc;
    g_last_occ = occ;
    Plan pl;
    const bool lane = use_lane_walker(total, p, single_api);
    make_plan(total, ns, p, sms, occ, pl, single_api, stop, tail.max > 0, lane ? occ_lane : 0);
    g_last_lane = lane;
    g_last_nseg = (uint32_t)pl.nseg_max;
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
    if (single_api) {                      // [0, n] offsets are implicit; the cut index lives in the workspace
        uint64_t *offs = (uint64_t *)ws;
        d_offsets = offs;
        d_cut_index = offs + 2;
    }
    rc = run(d_in, d_offsets, ns, total, stop, out_add, p, geo, d_cuts, d_cut_index, d_ncuts, ws + extra, pl.bytes,
             pl, sms, st, single_api, tail);
    if (owned) cudaFreeAsync(ws, st);
    return rc;
}

}  // namespace seqcdc

using namespace seqcdc;

// kernel launches made by the other translation units
void seqcdc_note_launches(int k) { g_launches += (uint64_t)k; }

// the library's stream-ordered pool (no trimming at synchronisation), for the
// other translation units' small per-call allocations
int seqcdc_internal_pool(cudaMemPool_t *pool) { return get_pool(*pool); }

// internal, used by seqcdc_range.cu (hidden visibility: not part of the ABI)
void seqcdc_ring_geometry(const seqcdc_params_t *p, uint32_t *bs, uint32_t *nb, uint32_t *ah)
{
    DevParams d;
    ring_geometry(p, d);
    *bs = d.bs;
    *nb = d.nb;
    *ah = d.ah;
}

SEQCDC_API int seqcdc_validate_params(const seqcdc_params_t *p)
{
    if (!p) return SEQCDC_EINVAL;
    if (p->mode > 1) return SEQCDC_EINVAL;
    if (p->seq_length < 2 || p->seq_length > SEQCDC_MAX_SEQ_LENGTH) return SEQCDC_EINVAL;
    if (p->skip_trigger < 1) return SEQCDC_EINVAL;
    if (p->min_size < p->seq_length) return SEQCDC_EINVAL;
    if (p->max_size < p->min_size) return SEQCDC_EINVAL;
    if (p->max_size > (1ull << 28)) return SEQCDC_EINVAL;  // implementation limit: 256 MiB chunks
    if ((p->flags & ~(SEQCDC_FLAG_SIGNED | SEQCDC_FLAG_PAIRS)) || p->reserved) return SEQCDC_EINVAL;
    if ((p->flags & SEQCDC_FLAG_PAIRS) && p->seq_length > SEQCDC_MAX_SEQ_LENGTH - 1) return SEQCDC_EINVAL;
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
    DevParams geo;
    ring_geometry(p, geo);
    int sms, occ, occ_lane;
    if (device_info(sms, occ, &occ_lane)) {   // no device: an upper bound (32 CTAs/SM)
        sms = 148;
        occ = 32;
        occ_lane = 8;
    }
    Plan pl, pb, pt, ql, qt;
    make_plan(total, ns ? ns : 1, p, sms, occ, pl, ns <= 1, total);
    make_plan(total, ns ? ns : 1, p, sms, occ, pb, false, total);
    make_plan(total, 1, p, sms, occ, pt, true, total, true);
    make_plan(total, 1, p, sms, occ, ql, true, total, false, occ_lane);
    make_plan(total, 1, p, sms, occ, qt, true, total, true, occ_lane);
    return std::max({pl.bytes, pb.bytes, pt.bytes, ql.bytes, qt.bytes}) + SINGLE_EXTRA;
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
        g_launches++;
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

static int range_chunk_tail_impl(const uint8_t *d_buf, uint64_t buf_len, uint64_t range_len, uint64_t entry,
                                 uint64_t global_offset, const seqcdc_params_t *p, uint64_t *d_cuts,
                                 uint64_t *d_ncuts, uint32_t tail_max, uint64_t *d_tail, uint64_t *d_tail_n,
                                 uint64_t *d_summary, void *d_ws, size_t ws_bytes, void *stream, uint64_t *push_blk,
                                 uint64_t *push_flag, uint64_t push_value)
{
    if (seqcdc_validate_params(p)) return SEQCDC_EINVAL;
    if (!d_ncuts || range_len > buf_len || entry > range_len) return SEQCDC_EINVAL;
    if (tail_max && (!d_tail || !d_tail_n)) return SEQCDC_EINVAL;
    if (push_blk && (!push_flag || !d_summary)) return SEQCDC_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    if (entry >= range_len) {
        if (cudaMemsetAsync(d_ncuts, 0, 8, st) != cudaSuccess) return SEQCDC_ECUDA;
        if (tail_max && cudaMemsetAsync(d_tail_n, 0, 8, st) != cudaSuccess) return SEQCDC_ECUDA;
        if (d_summary) k_set2<<<1, 1, 0, st>>>(d_summary, global_offset + entry, 0);
        if (push_blk) k_push_empty<<<1, 1, 0, st>>>(push_blk, push_flag, global_offset + entry, push_value);
        g_launches += (d_summary ? 1 : 0) + (push_blk ? 1 : 0);
        return cudaGetLastError() == cudaSuccess ? SEQCDC_OK : SEQCDC_ECUDA;
    }
    if (!d_buf || !d_cuts) return SEQCDC_EINVAL;
    TailReq t;
    t.tail = d_tail;
    t.tail_n = d_tail_n;
    t.max = tail_max;
    t.summary = d_summary;
    t.push_blk = push_blk;
    t.push_flag = push_flag;
    t.push_value = push_value;
    return enqueue(d_buf + entry, nullptr, 1, buf_len - entry, range_len - entry, global_offset + entry, p, d_cuts,
                   nullptr, d_ncuts, d_ws, ws_bytes, st, true, t);
}

SEQCDC_API int seqcdc_range_chunk_tail(const uint8_t *d_buf, uint64_t buf_len, uint64_t range_len, uint64_t entry,
                                       uint64_t global_offset, const seqcdc_params_t *p, uint64_t *d_cuts,
                                       uint64_t *d_ncuts, uint32_t tail_max, uint64_t *d_tail, uint64_t *d_tail_n,
                                       uint64_t *d_summary, void *d_ws, size_t ws_bytes, void *stream)
{
    return range_chunk_tail_impl(d_buf, buf_len, range_len, entry, global_offset, p, d_cuts, d_ncuts, tail_max,
                                 d_tail, d_tail_n, d_summary, d_ws, ws_bytes, stream, nullptr, nullptr, 0);
}

SEQCDC_API int seqcdc_range_chunk_tail_push(const uint8_t *d_buf, uint64_t buf_len, uint64_t range_len,
                                            uint64_t entry, uint64_t global_offset, const seqcdc_params_t *p,
                                            uint64_t *d_cuts, uint64_t *d_ncuts, uint32_t tail_max, uint64_t *d_tail,
                                            uint64_t *d_tail_n, uint64_t *d_summary, void *d_ws, size_t ws_bytes,
                                            uint64_t *d_peer_blk, uint64_t *d_peer_flag, uint64_t flag_value,
                                            void *stream)
{
    if (!d_peer_blk || !d_peer_flag) return SEQCDC_EINVAL;
    return range_chunk_tail_impl(d_buf, buf_len, range_len, entry, global_offset, p, d_cuts, d_ncuts, tail_max,
                                 d_tail, d_tail_n, d_summary, d_ws, ws_bytes, stream, d_peer_blk, d_peer_flag,
                                 flag_value);
}

// ------------------------------------------------------------------ peer-memory mailboxes (CUDA IPC)
namespace seqcdc {
// a small row stored into every rank's table (tables[p] = rank p's table, mapped
// into this process); the row's last word is the step, released at system scope
// after the data, so a reader that sees the step sees the row
__global__ void k_put_rows(const uint64_t *src, uint32_t nwords, uint64_t *const *tables, uint32_t P, uint32_t r,
                           uint64_t step)
{
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    uint64_t *row = tables[p] + (uint64_t)r * (nwords + 1);
    for (uint32_t i = 0; i < nwords; i++) row[i] = src[i];
    __threadfence_system();
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(row + nwords), "l"(step) : "memory");
}

// wait until every row of this rank's table carries `step` (acquire), at most
// timeout_ns; *status = 0 when complete, 1 on timeout
__global__ void k_wait_rows(const uint64_t *table, uint32_t nwords, uint32_t P, uint64_t step, uint64_t timeout_ns,
                            uint64_t *status, uint64_t *out)
{
    uint64_t t0, t, v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (uint32_t p = 0; p < P; p++) {
        const uint64_t *f = table + (uint64_t)p * (nwords + 1) + nwords;
#pragma unroll 1
        for (;;) {
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
            if (v == step) break;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > timeout_ns) {
                *status = 1;
                return;
            }
            __nanosleep(500);
        }
    }
    if (out)                                  // the rows' data, packed, for the caller's one host read
        for (uint32_t p = 0; p < P; p++)
            for (uint32_t i = 0; i < nwords; i++) out[(uint64_t)p * nwords + i] = table[(uint64_t)p * (nwords + 1) + i];
    *status = 0;
}
}  // namespace seqcdc

SEQCDC_API int seqcdc_xchg_put_rows(const uint64_t *d_src, uint32_t nwords, uint64_t *const *d_tables,
                                    uint32_t nranks, uint32_t row, uint64_t step, void *stream)
{
    if (!d_src || !d_tables || !nranks || row >= nranks || !nwords) return SEQCDC_EINVAL;
    k_put_rows<<<(nranks + 31) / 32, 32, 0, (cudaStream_t)stream>>>(d_src, nwords, d_tables, nranks, row, step);
    g_launches++;
    return cudaGetLastError() == cudaSuccess ? SEQCDC_OK : SEQCDC_ECUDA;
}

SEQCDC_API int seqcdc_xchg_wait_rows(const uint64_t *d_table, uint32_t nwords, uint32_t nranks, uint64_t step,
                                     uint64_t timeout_ns, uint64_t *d_status, uint64_t *d_out, void *stream)
{
    if (!d_table || !d_status || !nranks || !nwords) return SEQCDC_EINVAL;
    k_wait_rows<<<1, 1, 0, (cudaStream_t)stream>>>(d_table, nwords, nranks, step, timeout_ns, d_status, d_out);
    g_launches++;
    return cudaGetLastError() == cudaSuccess ? SEQCDC_OK : SEQCDC_ECUDA;
}

SEQCDC_API int seqcdc_xchg_alloc(size_t bytes, void **d_buf, void *ipc_handle)
{
    if (!d_buf || !ipc_handle || !bytes) return SEQCDC_EINVAL;
    void *p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) return SEQCDC_ENOMEM;
    cudaIpcMemHandle_t h;
    if (cudaMemset(p, 0, bytes) != cudaSuccess || cudaIpcGetMemHandle(&h, p) != cudaSuccess) {
        cudaFree(p);
        return SEQCDC_ECUDA;
    }
    memcpy(ipc_handle, &h, sizeof(h));
    *d_buf = p;
    return SEQCDC_OK;
}

SEQCDC_API int seqcdc_xchg_open(const void *ipc_handle, void **d_peer)
{
    if (!ipc_handle || !d_peer) return SEQCDC_EINVAL;
    cudaIpcMemHandle_t h;
    memcpy(&h, ipc_handle, sizeof(h));
    void *p = nullptr;
    if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        return SEQCDC_ECUDA;
    }
    *d_peer = p;
    return SEQCDC_OK;
}

SEQCDC_API int seqcdc_xchg_close(void *d_peer)
{
    return (d_peer && cudaIpcCloseMemHandle(d_peer) == cudaSuccess) ? SEQCDC_OK : SEQCDC_ECUDA;
}

SEQCDC_API int seqcdc_xchg_free(void *d_buf)
{
    return (d_buf && cudaFree(d_buf) == cudaSuccess) ? SEQCDC_OK : SEQCDC_ECUDA;
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

SEQCDC_API uint64_t seqcdc_launch_count(void)
{
    return g_launches.load();
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
    static char buf[512];
    int sms = 0, occ = 0, ol = 0;
    device_info(sms, occ, &ol);
    snprintf(buf, sizeof(buf),
             "seqcdc sm_100a; last call: %s walker, %u segments; warp walker: cp.async ring blk=%u nblk=%u "
             "ahead=%u, %d/SM, win_pairs=%u; lane walker: %u-B %s lines x2 (mbarrier-polled%s%s), %u pairs/step "
             "(%s masks), %u-thread CTAs, %d/SM max, pf=%u; k_ext=%u",
             g_last_lane ? "lane" : "warp", g_last_nseg, BLK, NBLK, AHEAD, g_last_occ, WIN_PAIRS, lw::LINE,
             SEQCDC_LW_BULK ? "cp.async.bulk" : "cp.async", SEQCDC_LW_LAZY ? " when needed" : " every step", SEQCDC_LW_PAIR ? ", pair fills on misses" : "",
             lw::GRP, SEQCDC_LW_PACKED ? "packed" : "per-word", lw::THREADS, ol, (unsigned)SEQCDC_LW_PF, K_EXT);
    return buf;
}

#ifdef SEQCDC_TIMELINE
SEQCDC_API int seqcdc_debug_lw_stats(uint64_t *out4, int reset)
{
    if (reset) {
        uint64_t z[4] = {0, 0, 0, 0};
        return cudaMemcpyToSymbol(lw::g_lw_stats, z, sizeof(z)) == cudaSuccess ? SEQCDC_OK : SEQCDC_ECUDA;
    }
    return cudaMemcpyFromSymbol(out4, lw::g_lw_stats, sizeof(uint64_t) * 4) == cudaSuccess ? SEQCDC_OK : SEQCDC_ECUDA;
}

SEQCDC_API int seqcdc_debug_timeline(uint64_t *d_buf, uint64_t nseg_cap)
{
    if (cudaMemcpyToSymbol(g_tl, &d_buf, sizeof(d_buf)) != cudaSuccess) return SEQCDC_ECUDA;
    if (cudaMemcpyToSymbol(g_tl_cap, &nseg_cap, sizeof(nseg_cap)) != cudaSuccess) return SEQCDC_ECUDA;
    return SEQCDC_OK;
}
#endif
