// seqcdc_device.cuh -- the warp-cooperative SeqCDC walker for sm_100a.
//
// One warp owns one speculative chain.  Its CTA streams the chain's bytes
// HBM -> shared memory through a ring of TILE-byte slots filled by 1-D TMA bulk
// copies (cp.async.bulk, completion on one mbarrier per slot).  The walk reads
// only the windows the method examines, classifying adjacent byte pairs
// lazily with SIMD-in-word compares (4 pairs per 32-bit word, one word per
// lane => 128 pairs per window):
//
//   F (favourable)  x<y (Increasing) / x>y (Decreasing)      P:215 "cmpgt"
//   O (opposing)    the reverse, strict                       P:217 "cmplt"
//   R               F at pairs i-L+2..i (a run of L bytes
//                   ending at byte i+1 -> cut at i+2)
//   d               the T-th O counted from the anchor
//
// Resolution of one chunk f(base) (the method):
//   a = base+min-L; limit = min(base+max, end); examined pairs are a..limit-2.
//   r = first R pair >= a+L-2; d = T-th O pair >= a.  r < d -> cut r+2.
//   d < r -> a = d+1+S (counters reset, reading c3) and repeat.  Neither ->
//   cut = limit.
// ballot/__ffs play the paper's builtin_ffs, the ballot bit-plane prefix +
// SWAR byte select its pdep+tzcnt, __popc/__reduce_add_sync its popcnt
// (P:229-231).
//
// Positions inside the walker are 32-bit offsets from a RING-aligned base
// address `rb` (so smem slot offsets are just `pos & RING_MASK` and 16-byte
// alignment of TMA sources is preserved); chains are rebased at chunk
// boundaries if they ever run 1 GiB past it.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace seqcdc {

#ifndef SEQCDC_TILE_SHIFT
#define SEQCDC_TILE_SHIFT 11
#endif
#ifndef SEQCDC_STAGES
#define SEQCDC_STAGES 4
#endif
constexpr int TILE_SHIFT = SEQCDC_TILE_SHIFT;        // 2 KiB ring slots
constexpr uint32_t TILE = 1u << TILE_SHIFT;
constexpr int STAGES = SEQCDC_STAGES;                // power of two
constexpr uint32_t RING = TILE * STAGES;             // 8 KiB per walker
constexpr uint32_t RING_MASK = RING - 1;
constexpr uint32_t WIN_PAIRS = 128;                  // pairs per window (32 lanes x 4)
constexpr uint32_t FULL = 0xffffffffu;
constexpr uint32_t H = 0x80808080u;
constexpr uint32_t REL_CLAMP = 0xC0000000u;          // relative positions stay below this
constexpr uint32_t REBASE_AT = 0x40000000u;          // rebase a chain past 1 GiB
constexpr uint32_t SMEM_WALK = RING + STAGES * 8;    // dynamic smem of one walker

struct DevParams {
    uint32_t L, T, S, M;   // M = L-1 favourable pairs per run
    uint64_t mn, mx;
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_tx(uint32_t bar, uint32_t tx)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tx) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_1d(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}

__device__ __forceinline__ uint32_t lds32(uint32_t addr)
{
    uint32_t v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

__device__ __forceinline__ void sts8(uint32_t addr, uint32_t v)
{
    asm volatile("st.shared.b8 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// shl/shr with PTX clamp semantics (shift >= 32 gives 0)
__device__ __forceinline__ uint32_t shl_c(uint32_t x, uint32_t s)
{
    uint32_t r;
    asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(s));
    return r;
}
__device__ __forceinline__ uint32_t shr_c(uint32_t x, uint32_t s)
{
    uint32_t r;
    asm("shr.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(s));
    return r;
}

__device__ __forceinline__ uint32_t lanemask_lt()
{
    uint32_t r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

__device__ __forceinline__ uint64_t ld_acquire_u64(const uint64_t *p)
{
    uint64_t v;
    asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_u64(uint64_t *p, uint64_t v)
{
    asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ------------------------------------------------------------------ byte-pair classification
// bit 7 of each byte of `lt` = [x_k < y_k], of `gt` = [x_k > y_k] (unsigned,
// strict); other bits are junk.  t = (~x & 7F) + (y & 7F) carries into bit 7
// iff low7(y) > low7(x); 0xFEFEFEFE - t is the same sum with x and y swapped.
__device__ __forceinline__ void lt_gt_flags(uint32_t x, uint32_t y, uint32_t &lt, uint32_t &gt)
{
    uint32_t t = (~x & 0x7f7f7f7fu) + (y & 0x7f7f7f7fu);
    uint32_t u = 0xfefefefeu - t;
    lt = (~x & y) | (~(x ^ y) & t);
    gt = (~y & x) | (~(x ^ y) & u);
}

// ------------------------------------------------------------------ one walker (warp-uniform state)
struct Walker {
    uint64_t rb;        // absolute address of relative position 0 (RING-aligned)
    uint32_t lo_rel;    // first loadable byte (relative)
    uint32_t end_rel;   // end of the stream (relative, clamped to REL_CLAMP)
    uint32_t buf, bar;  // shared addresses: ring, mbarriers
    uint32_t t_first;   // oldest tile still owned (relative tile index)
    uint32_t t_next;    // next tile to issue
    uint32_t t_end;     // one past the last tile with data
    uint32_t res_lo, res_hi;  // byte range known resident (all tiles waited)
    uint32_t pending;   // bit s: slot s holds an issued fill not yet waited for
    uint32_t nextpar;   // bit s: parity of the slot's next fill
};

__device__ __forceinline__ void ring_wait_slot(Walker &wk, uint32_t s)
{
    if (wk.pending & (1u << s)) {
        mbar_wait(wk.bar + 8 * s, ((wk.nextpar >> s) & 1u) ^ 1u);
        wk.pending &= ~(1u << s);
    }
}

__device__ __forceinline__ void ring_drain(Walker &wk)
{
#pragma unroll
    for (uint32_t s = 0; s < (uint32_t)STAGES; s++) ring_wait_slot(wk, s);
}

// Issue relative tile t (warp-uniform).  TMA moves the 16-byte-aligned
// interior; lanes copy the <16-byte ragged head/tail of the loadable range.
__device__ __forceinline__ void ring_issue(Walker &wk, uint32_t t, int lane)
{
    const uint32_t s = t & (STAGES - 1);
    ring_wait_slot(wk, s);  // never two fills in flight on one slot
    uint32_t lo = t << TILE_SHIFT, hi = lo + TILE;
    if (lo < wk.lo_rel) lo = wk.lo_rel;
    if (hi > wk.end_rel) hi = wk.end_rel;
    const uint32_t mlo = (lo + 15) & ~15u, mhi = hi & ~15u;
    uint32_t tx = 0;
    if (lo < hi && mlo < mhi) tx = mhi - mlo;
    const uint32_t bar = wk.bar + 8 * s;
    if (lane == 0) {
        mbar_arrive_tx(bar, tx);
        if (tx) tma_load_1d(wk.buf + (mlo & RING_MASK), (const void *)(wk.rb + mlo), tx, bar);
    }
    if (lo < hi && (lo != mlo || hi != mhi || !tx)) {
        uint32_t pos;
        bool ok;
        if (tx) {
            pos = lane < 16 ? lo + lane : mhi + (lane - 16);
            ok = lane < 16 ? pos < mlo : pos < hi;
        } else {
            pos = lo + lane;
            ok = pos < hi;
        }
        if (ok) sts8(wk.buf + (pos & RING_MASK), *(const volatile uint8_t *)(wk.rb + pos));
        __syncwarp();
    }
    wk.pending |= 1u << s;
    wk.nextpar ^= 1u << s;
}

// Slow path of ring_ensure: release tiles below need_lo, top up the ring,
// wait for the tiles covering [need_lo, need_hi).
__device__ __forceinline__ void ring_refill(Walker &wk, uint32_t need_lo, uint32_t need_hi, int lane)
{
    const uint32_t tlo = need_lo >> TILE_SHIFT, thi = (need_hi - 1) >> TILE_SHIFT;
    if (tlo > wk.t_first) {
        wk.t_first = tlo;
        if (wk.t_next < tlo) wk.t_next = tlo;
    }
#pragma unroll 1
    while (wk.t_next < wk.t_end && wk.t_next < wk.t_first + STAGES) {
        ring_issue(wk, wk.t_next, lane);
        wk.t_next++;
    }
    ring_wait_slot(wk, tlo & (STAGES - 1));
    if (thi != tlo) ring_wait_slot(wk, thi & (STAGES - 1));
    wk.res_lo = tlo << TILE_SHIFT;
    wk.res_hi = (thi + 1) << TILE_SHIFT;
}

__device__ __forceinline__ void ring_ensure(Walker &wk, uint32_t need_lo, uint32_t need_hi, int lane)
{
    if (need_lo < wk.res_lo || need_hi > wk.res_hi) ring_refill(wk, need_lo, need_hi, lane);
}

// Start a chain whose loadable data is absolute [a_lo, a_end); returns the
// relative position of a_lo.
__device__ __forceinline__ uint32_t walker_start(Walker &wk, uint64_t a_lo, uint64_t a_end)
{
    ring_drain(wk);
    wk.rb = a_lo & ~(uint64_t)RING_MASK;
    wk.lo_rel = (uint32_t)(a_lo - wk.rb);
    const uint64_t e = a_end - wk.rb;
    wk.end_rel = e > REL_CLAMP ? REL_CLAMP : (uint32_t)e;
    wk.t_end = wk.end_rel > 0 ? ((wk.end_rel - 1) >> TILE_SHIFT) + 1 : 0;
    wk.t_first = wk.t_next = wk.lo_rel >> TILE_SHIFT;
    wk.res_lo = wk.res_hi = 0;
    return wk.lo_rel;
}

// Move the relative origin forward so that `pos` stays small (only at chunk
// boundaries; keeps tile numbering consistent: shift is a RING multiple).
__device__ __forceinline__ uint32_t walker_rebase(Walker &wk, uint32_t pos, uint64_t a_end)
{
    if (pos < REBASE_AT) return pos;
    ring_drain(wk);
    const uint32_t sh = (pos - RING) & ~RING_MASK;
    wk.rb += sh;
    wk.lo_rel = 0;
    const uint64_t e = a_end - wk.rb;
    wk.end_rel = e > REL_CLAMP ? REL_CLAMP : (uint32_t)e;
    wk.t_end = wk.end_rel > 0 ? ((wk.end_rel - 1) >> TILE_SHIFT) + 1 : 0;
    const uint32_t np = pos - sh;
    wk.t_first = wk.t_next = np >> TILE_SHIFT;
    wk.res_lo = wk.res_hi = 0;
    return np;
}

// ------------------------------------------------------------------ one chunk
// f(base): the cut ending the chunk that starts at relative position `base`.
// Warp-uniform; every lane returns the same value.
template <int MODE>
__device__ __forceinline__ uint32_t resolve_chunk(Walker &wk, const DevParams &p, uint32_t base, int lane)
{
    const uint64_t lim64 = (uint64_t)base + p.mx;
    const uint32_t limit = lim64 < wk.end_rel ? (uint32_t)lim64 : wk.end_rel;
    if (limit - base < 2) return limit;
    const uint32_t lim2 = limit - 2;               // last pair that may be examined
    uint32_t a = base + (uint32_t)p.mn - p.L;      // P:179 (mn - L < max <= 2^40 checked on host)
    if ((uint64_t)base + p.mn - p.L > lim2) return limit;
    uint32_t oc = 0;                               // opposing pairs counted since the anchor a
    uint32_t carry = 0;                            // previous window's lane-31 masked F word
    uint32_t p0 = a & ~3u;
    uint32_t ra = a & 3u;                          // pairs of lane 0 below the anchor (first window)
    const uint32_t lt_mask = lanemask_lt();
#pragma unroll 1
    for (;;) {
        uint32_t need_hi = p0 + WIN_PAIRS + 4;
        if (need_hi > lim2 + 2) need_hi = lim2 + 2;
        ring_ensure(wk, p0, need_hi, lane);
        const uint32_t q = p0 + 4 * (uint32_t)lane;
        const uint32_t x = lds32(wk.buf + (q & RING_MASK));
        const uint32_t xn = lds32(wk.buf + ((q + 4) & RING_MASK));
        const uint32_t y = __funnelshift_r(x, xn, 8);     // y_k = byte q+k+1
        uint32_t lt, gt;
        lt_gt_flags(x, y, lt, gt);
        // valid pairs: a <= pair <= lim2
        const uint32_t rh = lim2 - p0 > 255u ? 255u : lim2 - p0;
        const int32_t sh = 32 * lane + 24 - 8 * (int32_t)rh;
        const uint32_t V = shl_c(FULL, lane ? 0u : 8u * ra) & shr_c(FULL, sh > 0 ? (uint32_t)sh : 0u) & H;
        const uint32_t Fm = (MODE == 0 ? lt : gt) & V;
        const uint32_t Om = (MODE == 0 ? gt : lt) & V;
        // runs of M favourable pairs ending at each pair (M <= 4 here; longer
        // runs are handled by resolve_chunk_long)
        const uint32_t up = __shfl_up_sync(FULL, Fm, 1);
        const uint32_t W1 = lane ? up : carry;
        uint32_t R = Fm;
        if (p.M > 1) R &= __funnelshift_l(W1, Fm, 8);
        if (p.M > 2) R &= __funnelshift_l(W1, Fm, 16);
        if (p.M > 3) R &= __funnelshift_l(W1, Fm, 24);
        const uint32_t rmask = __ballot_sync(FULL, R != 0);
        const uint32_t cnt = __popc(Om);
        const uint32_t total = __reduce_add_sync(FULL, cnt);
        const uint32_t need = p.T - oc;
        if (rmask == 0 && total < need) {          // nothing decided in this window
            oc += total;
            carry = __shfl_sync(FULL, Fm, 31);
            p0 += WIN_PAIRS;
            ra = 0;
            if (p0 > lim2) return limit;
            continue;
        }
        uint32_t r = FULL, d = FULL;
        if (rmask) {
            const int rl = __ffs(rmask) - 1;
            const uint32_t rbyte = (uint32_t)(__ffs(R) - 1) >> 3;
            r = p0 + 4 * (uint32_t)rl + __shfl_sync(FULL, rbyte, rl);
        }
        if (total >= need) {
            // exclusive prefix of per-lane counts (0..4) from ballot bit planes
            const uint32_t b0 = __ballot_sync(FULL, cnt & 1), b1 = __ballot_sync(FULL, cnt & 2),
                           b2 = __ballot_sync(FULL, cnt & 4);
            const uint32_t excl = __popc(b0 & lt_mask) + 2 * __popc(b1 & lt_mask) + 4 * __popc(b2 & lt_mask);
            const int dl = __ffs(__ballot_sync(FULL, excl + cnt >= need)) - 1;
            // in lane dl: the k-th flag (k = need - excl); byte j holds flags of bytes 0..j
            const uint32_t k = need - excl;
            const uint32_t pc = (Om >> 7) * 0x01010101u;
            const uint32_t ge = ((pc | H) - k * 0x01010101u) & 0x00808080u;
            const uint32_t dbyte = 3u - __popc(ge);
            d = p0 + 4 * (uint32_t)dl + __shfl_sync(FULL, dbyte, dl);
        }
        if (r < d) return r + 2;                   // boundary after the run
        if (p.S >= lim2 - d) return limit;         // skip lands past the last pair (c8)
        a = d + 1 + p.S;                           // content-defined skip (c3)
        oc = 0;
        carry = 0;
        p0 = a & ~3u;
        ra = a & 3u;
    }
}

// Same resolution for 5 < L <= 16: runs of up to 15 favourable pairs span up
// to four words back; the previous window's words come in by shuffles.
template <int MODE>
__device__ __forceinline__ uint32_t resolve_chunk_long(Walker &wk, const DevParams &p, uint32_t base, int lane)
{
    const uint64_t lim64 = (uint64_t)base + p.mx;
    const uint32_t limit = lim64 < wk.end_rel ? (uint32_t)lim64 : wk.end_rel;
    if (limit - base < 2) return limit;
    const uint32_t lim2 = limit - 2;
    uint32_t a = base + (uint32_t)p.mn - p.L;
    if ((uint64_t)base + p.mn - p.L > lim2) return limit;
    uint32_t oc = 0;
    uint32_t prevwin = 0;   // previous window's masked F word of this lane
    uint32_t p0 = a & ~3u;
    uint32_t ra = a & 3u;
    const uint32_t lt_mask = lanemask_lt();
#pragma unroll 1
    for (;;) {
        uint32_t need_hi = p0 + WIN_PAIRS + 4;
        if (need_hi > lim2 + 2) need_hi = lim2 + 2;
        ring_ensure(wk, p0, need_hi, lane);
        const uint32_t q = p0 + 4 * (uint32_t)lane;
        const uint32_t x = lds32(wk.buf + (q & RING_MASK));
        const uint32_t xn = lds32(wk.buf + ((q + 4) & RING_MASK));
        const uint32_t y = __funnelshift_r(x, xn, 8);
        uint32_t lt, gt;
        lt_gt_flags(x, y, lt, gt);
        const uint32_t rh = lim2 - p0 > 255u ? 255u : lim2 - p0;
        const int32_t sh = 32 * lane + 24 - 8 * (int32_t)rh;
        const uint32_t V = shl_c(FULL, lane ? 0u : 8u * ra) & shr_c(FULL, sh > 0 ? (uint32_t)sh : 0u) & H;
        const uint32_t Fm = (MODE == 0 ? lt : gt) & V;
        const uint32_t Om = (MODE == 0 ? gt : lt) & V;
        uint32_t Wd[5];
        Wd[0] = Fm;
#pragma unroll
        for (int k = 1; k <= 4; k++) {
            const uint32_t a1 = __shfl_sync(FULL, Fm, (lane - k) & 31);
            const uint32_t b1 = __shfl_sync(FULL, prevwin, (lane - k) & 31);
            Wd[k] = lane >= k ? a1 : b1;
        }
        uint32_t R = Fm;
#pragma unroll
        for (uint32_t j = 1; j < 16; j++)
            if (j < p.M) R &= __funnelshift_l(Wd[(j >> 2) + 1], Wd[j >> 2], 8 * (j & 3));
        const uint32_t rmask = __ballot_sync(FULL, R != 0);
        const uint32_t cnt = __popc(Om);
        const uint32_t total = __reduce_add_sync(FULL, cnt);
        const uint32_t need = p.T - oc;
        if (rmask == 0 && total < need) {
            oc += total;
            prevwin = Fm;
            p0 += WIN_PAIRS;
            ra = 0;
            if (p0 > lim2) return limit;
            continue;
        }
        uint32_t r = FULL, d = FULL;
        if (rmask) {
            const int rl = __ffs(rmask) - 1;
            const uint32_t rbyte = (uint32_t)(__ffs(R) - 1) >> 3;
            r = p0 + 4 * (uint32_t)rl + __shfl_sync(FULL, rbyte, rl);
        }
        if (total >= need) {
            const uint32_t b0 = __ballot_sync(FULL, cnt & 1), b1 = __ballot_sync(FULL, cnt & 2),
                           b2 = __ballot_sync(FULL, cnt & 4);
            const uint32_t excl = __popc(b0 & lt_mask) + 2 * __popc(b1 & lt_mask) + 4 * __popc(b2 & lt_mask);
            const int dl = __ffs(__ballot_sync(FULL, excl + cnt >= need)) - 1;
            const uint32_t k = need - excl;
            const uint32_t pc = (Om >> 7) * 0x01010101u;
            const uint32_t ge = ((pc | H) - k * 0x01010101u) & 0x00808080u;
            const uint32_t dbyte = 3u - __popc(ge);
            d = p0 + 4 * (uint32_t)dl + __shfl_sync(FULL, dbyte, dl);
        }
        if (r < d) return r + 2;
        if (p.S >= lim2 - d) return limit;
        a = d + 1 + p.S;
        oc = 0;
        prevwin = 0;
        p0 = a & ~3u;
        ra = a & 3u;
    }
}

template <int MODE, bool LONG>
__device__ __forceinline__ uint32_t resolve(Walker &wk, const DevParams &p, uint32_t base, int lane)
{
    return LONG ? resolve_chunk_long<MODE>(wk, p, base, lane) : resolve_chunk<MODE>(wk, p, base, lane);
}

}  // namespace seqcdc
