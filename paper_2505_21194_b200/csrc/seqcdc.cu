// seqcdc.cu -- B200 (sm_100a) SeqCDC chunking behind the C ABI in include/seqcdc.h.
//
// Pipeline for one call (all on the caller's stream, no host synchronisation):
//   1. k_setup     segment table: each stream is cut into segments of G bytes
//                  (G a multiple of max_size); list capacities; state reset.
//   2. k_walk      persistent CTAs, one warp each.  Each CTA takes segments in
//                  order and walks a SPECULATIVE chain from the segment start as
//                  if a cut were there ("the next cut depends only on the
//                  previous cut"), recording cuts < segment end in its list L_s
//                  (published every 32 cuts with release semantics).  At the
//                  first cut >= segment end the chain continues (EXTENSION),
//                  each cut checked against the list of the chain that owns that
//                  region; the first common cut is a merge point: from there on
//                  both chains are identical.  Extension cuts go to X_s.
//   3. k_stitch    per stream: follow the merges from the stream start (the
//                  only chain that is right from its start) to mark live
//                  chains and where each becomes valid; count valid cuts.
//   4. k_fallback  streams whose extension overflowed its budget (pathological
//                  phase-locked data) are re-walked by one warp end to end.
//   5. k_scan      exclusive scan of per-segment counts -> output offsets.
//   6. k_copy      gather valid L/X cuts into d_cuts.
// The hot loop (k_walk) streams every byte HBM->SMEM once with 1-D TMA and
// classifies lazily; see seqcdc_device.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "../../include/seqcdc.h"
#include "seqcdc_device.cuh"

#define SEQCDC_API extern "C" __attribute__((visibility("default")))

namespace seqcdc {

constexpr uint64_t DONE_BIT = 1ull << 63;
constexpr uint64_t CNT_MASK = DONE_BIT - 1;
constexpr int32_t TGT_UNSET = -1;
constexpr int32_t TGT_END = -2;
constexpr int32_t TGT_OVERFLOW = -3;
constexpr int64_t ENTRY_DEAD = -2;
constexpr uint32_t K_EXT = 4;            // extension budget, in segments
constexpr uint64_t G_FLOOR_CHUNKS = 32;  // minimum segment length, in max_size units

enum { C_NSEG = 0, C_NEXT = 1, C_NEXT_FB = 2, C_NFLAG = 3, C_BAD = 4, C_NWORDS = 8 };

struct Work {
    // inputs
    const uint8_t *in;
    const uint64_t *offs;  // [ns+1]
    uint32_t ns;
    uint64_t G;
    uint64_t total;
    DevParams p;
    // per stream
    uint32_t *str_first;   // [ns+1]
    uint32_t *str_flag;    // [ns]
    uint32_t *flagged;     // [ns]
    // per segment
    uint64_t *seg_lo, *seg_hi;
    uint32_t *seg_stream;
    uint64_t *Loff, *Xoff;
    uint32_t *Lcap, *Xcap;
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

// ------------------------------------------------------------------ block scan helper
// Exclusive scan over n items with a 1024-thread block; get(i) -> u64, put(i, excl).
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
            uint64_t w = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0, wi = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint64_t t = __shfl_up_sync(FULL, wi, o);
                if (lane >= o) wi += t;
            }
            warp_tot[lane] = wi - w;
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

// ------------------------------------------------------------------ 1. setup
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
    // segments per stream -> first segment index
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
        w.ctrl[C_NEXT_FB] = 0;
        w.ctrl[C_NFLAG] = 0;
        w.ctrl[C_BAD] = 0;
    }
    __syncthreads();
    // per segment: bounds, capacities, state
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
        const uint64_t b = (a + G < E) ? a + G : E;
        const bool last = (s + 1 == w.str_first[j + 1]);
        w.seg_lo[s] = a;
        w.seg_hi[s] = last ? E : b;
        w.seg_stream[s] = j;
        w.Lcap[s] = (uint32_t)(((last ? E : b) - a) / mn + 2);
        uint64_t xr = last ? 0 : E - b;
        if (xr > K_EXT * G) xr = K_EXT * G;
        w.Xcap[s] = last ? 0 : (uint32_t)(xr / mn + 2);
        w.Lcnt[s] = 0;
        w.Xcnt[s] = 0;
        w.target[s] = TGT_UNSET;
        w.midx[s] = -1;
    }
    __syncthreads();
    block_scan(nseg, [&](uint64_t s) -> uint64_t { return w.Lcap[s]; },
               [&](uint64_t s, uint64_t ex) { w.Loff[s] = ex; });
    block_scan(nseg, [&](uint64_t s) -> uint64_t { return w.Xcap[s]; },
               [&](uint64_t s, uint64_t ex) { w.Xoff[s] = ex; });
}

// ------------------------------------------------------------------ 2. walk
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

// Publish the first b.n entries of a spec list (release), optionally final.
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
    uint64_t w;    // this lane's window entry
};

// Is relative offset `rel` a cut of chain t (implicit start or in L_t)?
__device__ int check_cut(const Work &w, Cursor &c, uint32_t t, uint64_t rel, int64_t &idx, int lane)
{
    if ((int64_t)t != c.t) {
        c.t = t;
        c.j = 0;
        c.nv = 0;
    }
    if (rel == w.seg_lo[t]) {
        idx = -1;
        return CK_MERGE;
    }
    const uint64_t *Lt = w.L + w.Loff[t];
#pragma unroll 1
    for (;;) {
        if (c.nv > 0) {
            const uint32_t hit = __ballot_sync(FULL, lane < (int)c.nv && c.w == rel);
            if (hit) {
                idx = (int64_t)(c.j + __ffs(hit) - 1);
                return CK_MERGE;
            }
            const uint64_t last = __shfl_sync(FULL, c.w, c.nv - 1);
            if (last > rel) return CK_NO;
            if (c.nv == 32) {
                c.j += 32;
                c.nv = 0;
            } else {
                const uint64_t word = ld_acquire_u64(w.Lcnt + t);
                const uint64_t cnt = word & CNT_MASK;
                if (cnt > c.j + c.nv) {
                    c.nv = (uint32_t)(cnt - c.j < 32 ? cnt - c.j : 32);
                    c.w = lane < (int)c.nv ? __ldcg(Lt + c.j + lane) : 0;
                    continue;
                }
                return (word & DONE_BIT) ? CK_NO : CK_UNDECIDED;
            }
        }
        const uint64_t word = ld_acquire_u64(w.Lcnt + t);
        const uint64_t cnt = word & CNT_MASK;
        if (cnt > c.j) {
            c.nv = (uint32_t)(cnt - c.j < 32 ? cnt - c.j : 32);
            c.w = lane < (int)c.nv ? __ldcg(Lt + c.j + lane) : 0;
            continue;
        }
        return (word & DONE_BIT) ? CK_NO : CK_UNDECIDED;
    }
}

template <int MODE, bool SMALL_M>
__device__ void walk_segment(const Work &w, Ring &rg, uint32_t s, int lane)
{
    const uint64_t abase = (uint64_t)(uintptr_t)w.in;
    const uint32_t j = w.seg_stream[s];
    const uint64_t S0 = w.offs[j], E = w.offs[j + 1];
    const uint32_t first = w.str_first[j];
    const bool last = (s + 1 == w.str_first[j + 1]);
    const uint64_t lo = w.seg_lo[s], hi = w.seg_hi[s];
    const uint64_t Eabs = abase + E;
    ring_start(rg, abase + lo, Eabs, abase + lo);

    uint64_t *Ls = w.L + w.Loff[s];
    ListBuf lb{0, 0};
    uint64_t base = abase + lo;
    uint64_t cut = 0;
    bool extend = false;
#pragma unroll 1
    while (base < Eabs) {
        cut = resolve_chunk<MODE, SMALL_M>(rg, w.p, base, Eabs, lane);
        if (!last && cut >= abase + hi) {
            extend = true;
            break;
        }
        lb_push(lb, cut - abase, Ls, lane);
        if ((lb.n & 31) == 0) publish(w.Lcnt + s, lb.n, false, lane);
        base = cut;
    }
    lb_flush(lb, Ls, lane);
    publish(w.Lcnt + s, lb.n, true, lane);
    if (!extend) return;

    // ---- extension: walk on until a cut coincides with the chain owning it
    uint64_t *Xs = w.X + w.Xoff[s];
    const uint32_t xcap = w.Xcap[s];
    ListBuf xb{0, 0};
    Cursor cur{-1, 0, 0, 0};
    int32_t tgt = TGT_OVERFLOW;
    int64_t mi = -1;
#pragma unroll 1
    for (;;) {
        if (xb.n == xcap) {
            tgt = TGT_OVERFLOW;
            break;
        }
        const uint64_t rel = cut - abase;
        lb_push(xb, rel, Xs, lane);
        if (rel == E) {
            tgt = TGT_END;
            break;
        }
        const uint32_t t = first + (uint32_t)((rel - S0) / w.G);
        int64_t idx;
        if (check_cut(w, cur, t, rel, idx, lane) == CK_MERGE) {
            tgt = (int32_t)t;
            mi = idx;
            break;
        }
        base = cut;
        cut = resolve_chunk<MODE, SMALL_M>(rg, w.p, base, Eabs, lane);
    }
    lb_flush(xb, Xs, lane);
    if (lane == 0) {
        w.Xcnt[s] = xb.n;
        w.target[s] = tgt;
        w.midx[s] = mi;
    }
}

template <int MODE, bool SMALL_M>
__global__ void __launch_bounds__(32) k_walk(Work w)
{
    extern __shared__ __align__(128) uint8_t smem[];
    const int lane = threadIdx.x;
    Ring rg;
    rg.buf = smem_u32(smem);
    rg.bar = smem_u32(smem + RING);
    rg.pending = 0;
    rg.nextpar = 0;
    rg.t_first = rg.t_next = rg.t_end = 0;
    rg.a_lo = rg.a_hi = 0;
    if (lane < STAGES) mbar_init(rg.bar + 8 * lane, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    if (w.ctrl[C_BAD]) return;
    const uint32_t nseg = w.ctrl[C_NSEG];
#pragma unroll 1
    for (;;) {
        uint32_t s = 0;
        if (lane == 0) s = atomicAdd(w.ctrl + C_NEXT, 1u);
        s = __shfl_sync(FULL, s, 0);
        if (s >= nseg) break;
        walk_segment<MODE, SMALL_M>(w, rg, s, lane);
    }
    ring_drain(rg);
}

// ------------------------------------------------------------------ 3. stitch
__global__ void __launch_bounds__(1024) k_stitch(Work w)
{
    extern __shared__ __align__(16) uint8_t sm[];
    if (w.ctrl[C_BAD]) return;
    __shared__ uint32_t flag;
    for (uint32_t j = blockIdx.x; j < w.ns; j += gridDim.x) {
        const uint32_t f = w.str_first[j], k = w.str_first[j + 1] - f;
        if (k == 1) {
            if (threadIdx.x == 0) {
                w.entry[f] = -1;
                w.seg_count[f] = w.Lcnt[f] & CNT_MASK;
                w.str_flag[j] = 0;
            }
            continue;
        }
        int32_t *tg = (int32_t *)sm;                              // [k]
        int64_t *en = (int64_t *)(sm + ((4ull * k + 15) & ~15ull));  // [k]
        for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) {
            int32_t t = w.target[f + i];
            tg[i] = t >= 0 ? t - (int32_t)f : t;
            en[i] = ENTRY_DEAD;
        }
        if (threadIdx.x == 0) flag = 0;
        __syncthreads();
        if (threadIdx.x < 32) {
            const int lane = threadIdx.x;
            uint32_t cur = 0;
            int64_t ent = -1;
#pragma unroll 1
            for (;;) {
                const uint32_t i = cur + lane;
                const int32_t t = i < k ? tg[i] : 0;
                const bool pass = (i + 1 < k) && t == (int32_t)(i + 1);
                const uint32_t nb = __ballot_sync(FULL, !pass);
                const int js = nb ? __ffs(nb) - 1 : 32;
                if (lane <= js && i < k)
                    en[i] = lane == 0 ? ent : w.midx[f + i - 1];
                if (js == 32) {
                    ent = w.midx[f + cur + 31];
                    cur += 32;
                    continue;
                }
                const uint32_t ic = cur + js;
                if (ic + 1 == k) break;               // stream's last segment ends at E
                const int32_t tj = tg[ic];
                if (tj == TGT_END) break;
                if (tj < 0) {                         // overflow (or never set)
                    if (lane == 0) flag = 1;
                    break;
                }
                ent = w.midx[f + ic];
                cur = (uint32_t)tj;
            }
        }
        __syncthreads();
        if (flag) {
            for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) {
                w.seg_count[f + i] = 0;
                w.entry[f + i] = ENTRY_DEAD;
            }
            if (threadIdx.x == 0) {
                w.str_flag[j] = 1;
                w.flagged[atomicAdd(w.ctrl + C_NFLAG, 1u)] = j;
            }
        } else {
            for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) {
                const int64_t e = en[i];
                uint64_t c = 0;
                if (e != ENTRY_DEAD) c = (w.Lcnt[f + i] & CNT_MASK) - (uint64_t)(e + 1) + w.Xcnt[f + i];
                w.seg_count[f + i] = c;
                w.entry[f + i] = e;
            }
            if (threadIdx.x == 0) w.str_flag[j] = 0;
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ 4. fallback (rare)
template <int MODE, bool SMALL_M>
__global__ void __launch_bounds__(32) k_fallback(Work w)
{
    extern __shared__ __align__(128) uint8_t smem[];
    const int lane = threadIdx.x;
    if (w.ctrl[C_BAD] || w.ctrl[C_NFLAG] == 0) return;
    Ring rg;
    rg.buf = smem_u32(smem);
    rg.bar = smem_u32(smem + RING);
    rg.pending = 0;
    rg.nextpar = 0;
    rg.t_first = rg.t_next = rg.t_end = 0;
    rg.a_lo = rg.a_hi = 0;
    if (lane < STAGES) mbar_init(rg.bar + 8 * lane, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const uint64_t abase = (uint64_t)(uintptr_t)w.in;
    const uint32_t nflag = w.ctrl[C_NFLAG];
#pragma unroll 1
    for (;;) {
        uint32_t q = 0;
        if (lane == 0) q = atomicAdd(w.ctrl + C_NEXT_FB, 1u);
        q = __shfl_sync(FULL, q, 0);
        if (q >= nflag) break;
        const uint32_t j = w.flagged[q];
        const uint64_t S0 = w.offs[j], E = w.offs[j + 1];
        uint64_t *dst = w.FB + (S0 - w.offs[0]) / w.p.mn + j;
        ring_start(rg, abase + S0, abase + E, abase + S0);
        ListBuf lb{0, 0};
        uint64_t base = abase + S0;
#pragma unroll 1
        while (base < abase + E) {
            const uint64_t cut = resolve_chunk<MODE, SMALL_M>(rg, w.p, base, abase + E, lane);
            lb_push(lb, cut - abase, dst, lane);
            base = cut;
        }
        lb_flush(lb, dst, lane);
        if (lane == 0) w.seg_count[w.str_first[j]] = lb.n;
    }
    ring_drain(rg);
}

// ------------------------------------------------------------------ 5. scan, 6. copy
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
    const uint32_t nseg = w.ctrl[C_NSEG];
    const int lane = threadIdx.x & 31;
    const uint32_t warps = gridDim.x * (blockDim.x >> 5);
    for (uint32_t s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); s < nseg; s += warps) {
        const uint32_t j = w.seg_stream[s];
        uint64_t *out = w.cuts + w.seg_out[s];
        if (w.str_flag[j]) {
            if (s != w.str_first[j]) continue;
            const uint64_t *src = w.FB + (w.offs[j] - w.offs[0]) / w.p.mn + j;
            const uint64_t n = w.seg_count[s];
            for (uint64_t i = lane; i < n; i += 32) out[i] = src[i];
            continue;
        }
        const int64_t e = w.entry[s];
        if (e == ENTRY_DEAD) continue;
        const uint64_t nl = (w.Lcnt[s] & CNT_MASK) - (uint64_t)(e + 1);
        const uint64_t *Ls = w.L + w.Loff[s] + (e + 1);
        for (uint64_t i = lane; i < nl; i += 32) out[i] = Ls[i];
        const uint64_t nx = w.Xcnt[s];
        const uint64_t *Xs = w.X + w.Xoff[s];
        for (uint64_t i = lane; i < nx; i += 32) out[nl + i] = Xs[i];
    }
}

__global__ void k_empty(uint64_t *cut_index, uint64_t *ncuts)
{
    cut_index[0] = 0;
    *ncuts = 0;
}

// ------------------------------------------------------------------ host side
struct Plan {
    uint64_t G, nseg_max, L_items, X_items, FB_items;
    size_t bytes;
    size_t o_ctrl, o_str_first, o_str_flag, o_flagged, o_seg_lo, o_seg_hi, o_seg_stream, o_Loff, o_Xoff,
        o_Lcap, o_Xcap, o_Lcnt, o_Xcnt, o_target, o_midx, o_entry, o_seg_count, o_seg_out, o_L, o_X, o_FB;
    uint32_t walk_grid;
};

static int g_sms = 0, g_occ = 0;
static uint64_t g_force_G = 0;
static std::mutex g_mu;
static cudaMemPool_t g_pool[64];
static bool g_pool_ok[64];

static int device_info(int &sms, int &occ)
{
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_sms) {
        int dev;
        if (cudaGetDevice(&dev) != cudaSuccess) return SEQCDC_ECUDA;
        if (cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
            return SEQCDC_ECUDA;
        const int smem = RING + STAGES * 8;
        auto set_attrs = [&](const void *fn) {
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        };
        set_attrs((const void *)k_walk<0, true>);
        set_attrs((const void *)k_walk<1, true>);
        set_attrs((const void *)k_walk<0, false>);
        set_attrs((const void *)k_walk<1, false>);
        set_attrs((const void *)k_fallback<0, true>);
        set_attrs((const void *)k_fallback<1, true>);
        set_attrs((const void *)k_fallback<0, false>);
        set_attrs((const void *)k_fallback<1, false>);
        cudaFuncSetAttribute((const void *)k_stitch, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        int occ_ = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_, k_walk<0, true>, 32, smem) != cudaSuccess)
            return SEQCDC_ECUDA;
        g_occ = occ_ > 0 ? occ_ : 1;
    }
    sms = g_sms;
    occ = g_occ;
    return SEQCDC_OK;
}

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

static void make_plan(uint64_t total, uint32_t ns, const seqcdc_params_t *p, int sms, int occ, Plan &pl)
{
    const uint64_t walkers = (uint64_t)sms * occ;
    uint64_t denom = walkers > 2ull * ns ? walkers - ns : std::max<uint64_t>(walkers / 2, 1);
    uint64_t G = (total + denom - 1) / denom;
    G = std::max<uint64_t>(G, G_FLOOR_CHUNKS * p->max_size);
    if (g_force_G) G = std::max<uint64_t>(g_force_G, p->max_size);
    G = (G + p->max_size - 1) / p->max_size * p->max_size;
    pl.G = G;
    pl.nseg_max = (uint64_t)ns + total / G + 1;
    pl.L_items = total / p->min_size + 2 * pl.nseg_max + 2;
    pl.X_items = K_EXT * (total / p->min_size) + 2 * pl.nseg_max + 2;
    pl.FB_items = total / p->min_size + ns + 2;
    pl.walk_grid = (uint32_t)std::min<uint64_t>(pl.nseg_max, walkers);
    size_t o = 0;
    auto take = [&](size_t bytes) {
        size_t r = o;
        o = align_up(o + bytes, 256);
        return r;
    };
    const uint64_t S = pl.nseg_max;
    pl.o_ctrl = take(C_NWORDS * 4);
    pl.o_str_first = take(4ull * (ns + 1));
    pl.o_str_flag = take(4ull * ns);
    pl.o_flagged = take(4ull * ns);
    pl.o_seg_lo = take(8 * S);
    pl.o_seg_hi = take(8 * S);
    pl.o_seg_stream = take(4 * S);
    pl.o_Loff = take(8 * S);
    pl.o_Xoff = take(8 * S);
    pl.o_Lcap = take(4 * S);
    pl.o_Xcap = take(4 * S);
    pl.o_Lcnt = take(8 * S);
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

template <int MODE, bool SMALL_M>
static void launch_walkers(const Work &w, const Plan &pl, int sms, cudaStream_t st)
{
    const int smem = RING + STAGES * 8;
    k_walk<MODE, SMALL_M><<<pl.walk_grid, 32, smem, st>>>(w);
    const uint64_t kmax = std::min<uint64_t>(pl.nseg_max, w.total / pl.G + 2);
    k_stitch<<<std::min<uint64_t>(w.ns, 4ull * sms), 1024, (size_t)(kmax * 12 + 32), st>>>(w);
    k_fallback<MODE, SMALL_M><<<sms, 32, smem, st>>>(w);
}

static int run(const uint8_t *d_in, const uint64_t *d_offsets, uint32_t ns, uint64_t total,
               const seqcdc_params_t *p, uint64_t *d_cuts, uint64_t *d_cut_index, uint64_t *d_ncuts,
               void *d_ws, size_t ws_bytes, cudaStream_t st)
{
    int sms, occ;
    int rc = device_info(sms, occ);
    if (rc) return rc;
    Plan pl;
    make_plan(total, ns, p, sms, occ, pl);
    if (total / pl.G + 2 > 15000) return SEQCDC_EINVAL;  // stitch keeps one stream's segments in smem
    uint8_t *ws = (uint8_t *)d_ws;
    bool owned = false;
    if (ws) {
        if (ws_bytes < pl.bytes) return SEQCDC_ENOMEM;
    } else {
        cudaMemPool_t pool;
        if ((rc = get_pool(pool))) return rc;
        if (cudaMallocFromPoolAsync((void **)&ws, pl.bytes, pool, st) != cudaSuccess) return SEQCDC_ENOMEM;
        owned = true;
    }
    Work w;
    memset(&w, 0, sizeof(w));
    w.in = d_in;
    w.offs = d_offsets;
    w.ns = ns;
    w.G = pl.G;
    w.total = total;
    w.p.L = p->seq_length;
    w.p.T = p->skip_trigger;
    w.p.S = p->skip_size;
    w.p.M = p->seq_length - 1;
    w.p.mn = p->min_size;
    w.p.mx = p->max_size;
    w.ctrl = (uint32_t *)(ws + pl.o_ctrl);
    w.str_first = (uint32_t *)(ws + pl.o_str_first);
    w.str_flag = (uint32_t *)(ws + pl.o_str_flag);
    w.flagged = (uint32_t *)(ws + pl.o_flagged);
    w.seg_lo = (uint64_t *)(ws + pl.o_seg_lo);
    w.seg_hi = (uint64_t *)(ws + pl.o_seg_hi);
    w.seg_stream = (uint32_t *)(ws + pl.o_seg_stream);
    w.Loff = (uint64_t *)(ws + pl.o_Loff);
    w.Xoff = (uint64_t *)(ws + pl.o_Xoff);
    w.Lcap = (uint32_t *)(ws + pl.o_Lcap);
    w.Xcap = (uint32_t *)(ws + pl.o_Xcap);
    w.Lcnt = (uint64_t *)(ws + pl.o_Lcnt);
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

    k_setup<<<1, 1024, 0, st>>>(w);
    const bool small = p->seq_length <= 5;
    if (p->mode == SEQCDC_INCREASING) {
        if (small) launch_walkers<0, true>(w, pl, sms, st); else launch_walkers<0, false>(w, pl, sms, st);
    } else {
        if (small) launch_walkers<1, true>(w, pl, sms, st); else launch_walkers<1, false>(w, pl, sms, st);
    }
    k_scan<<<1, 1024, 0, st>>>(w);
    k_copy<<<std::max(1, sms * 4), 256, 0, st>>>(w);
    rc = cudaGetLastError() == cudaSuccess ? SEQCDC_OK : SEQCDC_ECUDA;
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
    if (p->max_size > (1ull << 40)) return SEQCDC_EINVAL;
    if (p->flags || p->reserved) return SEQCDC_EINVAL;
    return SEQCDC_OK;
}

SEQCDC_API int seqcdc_default_params(uint32_t avg_kib, uint32_t mode, seqcdc_params_t *out)
{
    if (!out || mode > 1) return SEQCDC_EINVAL;
    uint32_t L = 5, T, S;
    if (avg_kib == 4) { T = 55; S = 256; }
    else if (avg_kib == 8) { T = 50; S = 256; }
    else if (avg_kib == 16) { T = 50; S = 512; }
    else return SEQCDC_EINVAL;
    memset(out, 0, sizeof(*out));
    out->mode = mode;
    out->seq_length = L;
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
        occ = 16;
    }
    Plan pl;
    make_plan(total, ns ? ns : 1, p, sms, occ, pl);
    return pl.bytes + 256;  // + the offsets slice seqcdc_chunk() keeps in front
}

SEQCDC_API int seqcdc_chunk_batch(const uint8_t *d_in, const uint64_t *d_offsets, uint32_t ns,
                                  uint64_t total, const seqcdc_params_t *p, uint64_t *d_cuts,
                                  uint64_t *d_cut_index, uint64_t *d_ncuts, void *d_ws, size_t ws_bytes,
                                  void *stream)
{
    if (seqcdc_validate_params(p)) return SEQCDC_EINVAL;
    if (!d_offsets || !d_cut_index || !d_ncuts) return SEQCDC_EINVAL;
    if (total && (!d_in || !d_cuts)) return SEQCDC_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    if (ns == 0) {
        k_empty<<<1, 1, 0, st>>>(d_cut_index, d_ncuts);
        return cudaGetLastError() == cudaSuccess ? SEQCDC_OK : SEQCDC_ECUDA;
    }
    return run(d_in, d_offsets, ns, total, p, d_cuts, d_cut_index, d_ncuts, d_ws, ws_bytes, st);
}

namespace seqcdc {
__global__ void k_single_offsets(uint64_t *offs, uint64_t n)
{
    offs[0] = 0;
    offs[1] = n;
}
}  // namespace seqcdc

SEQCDC_API int seqcdc_chunk(const uint8_t *d_in, uint64_t n, const seqcdc_params_t *p, uint64_t *d_cuts,
                            uint64_t *d_ncuts, void *d_ws, size_t ws_bytes, void *stream)
{
    if (seqcdc_validate_params(p)) return SEQCDC_EINVAL;
    if (!d_ncuts) return SEQCDC_EINVAL;
    if (n && (!d_in || !d_cuts)) return SEQCDC_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    // offsets[2] + cut_index[2] live in a small extra workspace slice
    int sms, occ;
    int rc = device_info(sms, occ);
    if (rc) return rc;
    Plan pl;
    make_plan(n, 1, p, sms, occ, pl);
    const size_t extra = 256;
    uint8_t *ws = (uint8_t *)d_ws;
    bool owned = false;
    if (ws) {
        if (ws_bytes < pl.bytes + extra) return SEQCDC_ENOMEM;
    } else {
        cudaMemPool_t pool;
        if ((rc = get_pool(pool))) return rc;
        if (cudaMallocFromPoolAsync((void **)&ws, pl.bytes + extra, pool, st) != cudaSuccess)
            return SEQCDC_ENOMEM;
        owned = true;
    }
    uint64_t *offs = (uint64_t *)ws;
    uint64_t *cidx = offs + 2;
    k_single_offsets<<<1, 1, 0, st>>>(offs, n);
    rc = run(d_in, offs, 1, n, p, d_cuts, cidx, d_ncuts, ws + extra, pl.bytes, st);
    if (owned) cudaFreeAsync(ws, st);
    return rc;
}

SEQCDC_API int seqcdc_set_segment_bytes(uint64_t g)
{
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
    static char buf[160];
    snprintf(buf, sizeof(buf), "seqcdc sm_100a tile=%u stages=%d ring=%u win_pairs=%u k_ext=%u", TILE, STAGES,
             RING, WIN_PAIRS, K_EXT);
    return buf;
}
