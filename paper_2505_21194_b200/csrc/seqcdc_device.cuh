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

// ------------------------------------------------------------------ walker / producer pair
// Each CTA runs one chain with two warps: warp 0 walks (consumer), warp 1 is
// the TMA producer.  The producer streams the job's tiles in order into a
// STAGES-slot ring: tile t goes to slot t % STAGES, completion on full[slot]
// (arrive.expect_tx + cp.async.bulk).  The walker waits on full[] in tile
// order and releases each tile (arrive on empty[slot]) only after it waited
// for it, so every wait targets the slot's next fill (no phase ambiguity);
// the producer reuses a slot once empty[] shows the previous tile released.
// Fill sequence numbers g run on across jobs; the relative origin rb of a job
// is chosen so that slot(tile) == g % STAGES.
struct RingCtl {                 // in shared memory, after the ring
    uint64_t full[STAGES];
    uint64_t empty[STAGES];
    uint64_t rb;                 // job: absolute address of relative 0
    uint32_t lo_rel, end_rel;    // job: loadable relative byte range
    uint32_t t0, t_end;          // job: first / one-past-last tile
    uint32_t g0;                 // job: fill sequence number of tile t0
    volatile uint32_t stop;      // walker -> producer: job finished
    uint32_t g_next;             // producer -> walker: sequence after the last issued fill
    uint32_t quit;               // walker -> producer: no more jobs
};
constexpr uint32_t LOG_STAGES = STAGES == 2 ? 1 : STAGES == 4 ? 2 : STAGES == 8 ? 3 : 4;
constexpr uint32_t SMEM_WALK = RING + ((sizeof(RingCtl) + 127) & ~127u);  // dynamic smem of one pair
constexpr int PAIR_THREADS = 64;
constexpr int PAIR_BARRIER = 1;                                           // named barrier id

__device__ __forceinline__ void pair_sync()
{
    asm volatile("bar.sync %0, %1;" ::"n"(PAIR_BARRIER), "n"(PAIR_THREADS) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// try_wait with a suspend-time hint: the waiting thread sleeps (no issue
// slots) until the phase completes or ~hint ns pass.
__device__ __forceinline__ bool mbar_try_sleep(uint32_t bar, uint32_t parity)
{
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity), "r"(1000u)
        : "memory");
    return ok != 0;
}

struct Walker {
    uint64_t rb;        // absolute address of relative position 0
    uint32_t lo_rel;    // first loadable byte (relative)
    uint32_t end_rel;   // end of the stream (relative, clamped to REL_CLAMP)
    uint32_t buf;       // shared address of the ring
    uint32_t full, empty;  // shared addresses of the barrier arrays
    RingCtl *ctl;
    uint32_t t0, g0;    // first tile of the job and its fill sequence number
    uint32_t t_rel;     // next tile to release
    uint32_t t_wait;    // next tile to wait for (all tiles below were waited)
    uint32_t res_lo, res_hi;  // byte range resident: tiles [res_lo, res_hi) waited, not released
    uint32_t g;         // fill sequence number after the last job
};

__device__ __forceinline__ uint32_t tile_parity(const Walker &wk, uint32_t t)
{
    return ((wk.g0 + (t - wk.t0)) >> LOG_STAGES) & 1u;
}

// Both warps: set up the ring and barriers of a pair whose smem starts at `smem`.
__device__ __forceinline__ RingCtl *pair_init(uint8_t *smem, int tid)
{
    RingCtl *ctl = (RingCtl *)(smem + RING);
    if (tid < STAGES) {
        mbar_init(smem_u32(&ctl->full[tid]), 1);
        mbar_init(smem_u32(&ctl->empty[tid]), 1);
    }
    if (tid == 0) {
        ctl->stop = 0;
        ctl->quit = 0;
        ctl->g_next = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    pair_sync();
    return ctl;
}

__device__ __forceinline__ void walker_init(Walker &wk, uint8_t *smem, RingCtl *ctl)
{
    wk.buf = smem_u32(smem);
    wk.ctl = ctl;
    wk.full = smem_u32(&ctl->full[0]);
    wk.empty = smem_u32(&ctl->empty[0]);
    wk.g = 0;
    wk.rb = 0;
    wk.lo_rel = wk.end_rel = 0;
    wk.t0 = wk.g0 = wk.t_rel = wk.t_wait = 0;
    wk.res_lo = wk.res_hi = 0;
}

// Walker: start a job whose loadable data is absolute [a_lo, a_end); returns
// the relative position of a_lo.  Pairs with the producer's job wait.
__device__ __forceinline__ uint32_t walker_begin(Walker &wk, uint64_t a_lo, uint64_t a_end, int lane)
{
    const uint32_t k = wk.g & (STAGES - 1);
    wk.rb = (a_lo & ~(uint64_t)(TILE - 1)) - (uint64_t)k * TILE;
    wk.lo_rel = (uint32_t)(a_lo - wk.rb);
    const uint64_t e = a_end > a_lo ? a_end - wk.rb : wk.lo_rel;
    wk.end_rel = e > REL_CLAMP ? REL_CLAMP : (uint32_t)e;
    wk.t0 = k;
    wk.g0 = wk.g;
    wk.t_rel = wk.t_wait = k;
    wk.res_lo = wk.res_hi = 0;
    if (lane == 0) {
        RingCtl *c = wk.ctl;
        c->rb = wk.rb;
        c->lo_rel = wk.lo_rel;
        c->end_rel = wk.end_rel;
        c->t0 = k;
        c->t_end = wk.end_rel > wk.lo_rel ? ((wk.end_rel - 1) >> TILE_SHIFT) + 1 : k;
        c->g0 = wk.g;
        c->stop = 0;
        c->quit = 0;
    }
    pair_sync();   // job visible to the producer
    return wk.lo_rel;
}

__device__ __forceinline__ void walker_wait_tile(Walker &wk, uint32_t t)
{
    mbar_wait(wk.full + 8 * (t & (STAGES - 1)), tile_parity(wk, t));
}

__device__ __forceinline__ void walker_release_tile(Walker &wk, uint32_t t, int lane)
{
    if (lane == 0) mbar_arrive(wk.empty + 8 * (t & (STAGES - 1)));
}

// Walker slow path: make bytes [need_lo, need_hi) resident (need_hi-need_lo <= TILE);
// tiles below need_lo are released (after being waited, in order).
__device__ __forceinline__ void walker_need(Walker &wk, uint32_t need_lo, uint32_t need_hi, int lane)
{
    const uint32_t tlo = need_lo >> TILE_SHIFT, thi = (need_hi - 1) >> TILE_SHIFT;
#pragma unroll 1
    for (uint32_t t = wk.t_wait; t <= thi; t++) {
#pragma unroll 1
        while (wk.t_rel < tlo && wk.t_rel + STAGES <= t) {
            walker_release_tile(wk, wk.t_rel, lane);
            wk.t_rel++;
        }
        walker_wait_tile(wk, t);
    }
    if (wk.t_wait <= thi) wk.t_wait = thi + 1;
#pragma unroll 1
    while (wk.t_rel < tlo) {
        walker_release_tile(wk, wk.t_rel, lane);
        wk.t_rel++;
    }
    wk.res_lo = tlo << TILE_SHIFT;
    wk.res_hi = wk.t_wait << TILE_SHIFT;
}

// Walker: finish the job (producer stops; every issued tile waited + released).
__device__ __forceinline__ void walker_end(Walker &wk, int lane)
{
    if (lane == 0) wk.ctl->stop = 1;
    pair_sync();   // producer has stopped and published g_next
    const uint32_t gn = wk.ctl->g_next;
    const uint32_t t_hi = wk.t0 + (gn - wk.g0);
#pragma unroll 1
    for (uint32_t t = wk.t_wait; t < t_hi; t++) walker_wait_tile(wk, t);
    if (wk.t_wait < t_hi) wk.t_wait = t_hi;
#pragma unroll 1
    for (uint32_t t = wk.t_rel; t < t_hi; t++) walker_release_tile(wk, t, lane);
    wk.t_rel = t_hi;
    wk.g = gn;
    __syncwarp();
}

// Walker: no more jobs.
__device__ __forceinline__ void walker_quit(Walker &wk, int lane)
{
    if (lane == 0) wk.ctl->quit = 1;
    pair_sync();
}

// Producer warp: serve jobs until the walker quits.
__device__ __noinline__ void producer_loop(uint8_t *smem, RingCtl *ctl, int lane)
{
    const uint32_t buf = smem_u32(smem);
    const uint32_t full = smem_u32(&ctl->full[0]), empty = smem_u32(&ctl->empty[0]);
#pragma unroll 1
    for (;;) {
        pair_sync();                       // job posted (or quit)
        if (ctl->quit) break;
        const uint64_t rb = ctl->rb;
        const uint32_t lo_rel = ctl->lo_rel, end_rel = ctl->end_rel, t_end = ctl->t_end;
        uint32_t t = ctl->t0, g = ctl->g0;
#pragma unroll 1
        for (; t < t_end; t++, g++) {
            const uint32_t s = t & (STAGES - 1);
            if (g >= (uint32_t)STAGES) {   // slot reuse: the walker released the slot's previous tile
                const uint32_t par = ((g >> LOG_STAGES) - 1) & 1u;
                bool stopped = false;
#pragma unroll 1
                while (!mbar_try_sleep(empty + 8 * s, par)) {
                    if (ctl->stop) {
                        stopped = true;
                        break;
                    }
                }
                if (stopped) break;
            }
            if (ctl->stop) break;
            const uint32_t bar = full + 8 * s;
            uint32_t lo = t << TILE_SHIFT, hi = lo + TILE;
            if (lo >= lo_rel && hi <= end_rel) {
                if (lane == 0) {
                    mbar_arrive_tx(bar, TILE);
                    tma_load_1d(buf + s * TILE, (const void *)(rb + lo), TILE, bar);
                }
            } else {
                if (lo < lo_rel) lo = lo_rel;
                if (hi > end_rel) hi = end_rel;
                const uint32_t mlo = (lo + 15) & ~15u, mhi = hi & ~15u;
                const uint32_t tx = (lo < hi && mlo < mhi) ? mhi - mlo : 0;
                if (lo < hi) {   // ragged head/tail bytes by lanes, before the arrive
                    uint32_t pos;
                    bool ok;
                    if (tx) {
                        pos = lane < 16 ? lo + lane : mhi + (lane - 16);
                        ok = lane < 16 ? pos < mlo : pos < hi;
                    } else {
                        pos = lo + lane;
                        ok = pos < hi;
                    }
                    if (ok) sts8(buf + (pos & RING_MASK), *(const volatile uint8_t *)(rb + pos));
                }
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive_tx(bar, tx);
                    if (tx) tma_load_1d(buf + (mlo & RING_MASK), (const void *)(rb + mlo), tx, bar);
                }
            }
        }
        if (lane == 0) ctl->g_next = g;
        pair_sync();                       // job finished (pairs with walker_end)
    }
}

// ------------------------------------------------------------------ one chunk
// Favourable-run mask R for M = L-1 pairs.  MSPEC = 4: exactly four (L = 5,
// Table I); MSPEC = 0: any M <= 4 (runtime); MSPEC = -1: 5 <= M <= 15, using up
// to four words back (the previous window's words arrive by shuffles).
template <int MSPEC>
__device__ __forceinline__ uint32_t run_mask(uint32_t Fm, uint32_t carry1, uint32_t prevwin, uint32_t M, int lane)
{
    if (MSPEC >= 0) {
        const uint32_t up = __shfl_up_sync(FULL, Fm, 1);
        const uint32_t W1 = lane ? up : carry1;
        if (MSPEC == 4)
            return Fm & __funnelshift_l(W1, Fm, 8) & __funnelshift_l(W1, Fm, 16) & __funnelshift_l(W1, Fm, 24);
        uint32_t R = Fm;
        if (M > 1) R &= __funnelshift_l(W1, Fm, 8);
        if (M > 2) R &= __funnelshift_l(W1, Fm, 16);
        if (M > 3) R &= __funnelshift_l(W1, Fm, 24);
        return R;
    } else {
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
            if (j < M) R &= __funnelshift_l(Wd[(j >> 2) + 1], Wd[j >> 2], 8 * (j & 3));
        return R;
    }
}

// f(base): the cut ending the chunk that starts at relative position `base`.
// Warp-uniform; every lane returns the same value.
template <int MODE, int MSPEC>
__device__ __forceinline__ uint32_t resolve_chunk(Walker &wk, const DevParams &p, uint32_t base, int lane)
{
    const uint64_t lim64 = (uint64_t)base + p.mx;
    const uint32_t limit = lim64 < wk.end_rel ? (uint32_t)lim64 : wk.end_rel;
    if (limit - base < 2) return limit;
    const uint32_t lim2 = limit - 2;               // last pair that may be examined
    if ((uint64_t)base + p.mn - p.L > lim2) return limit;
    uint32_t a = base + (uint32_t)p.mn - p.L;
    uint32_t need = p.T;                           // opposing pairs still needed for a skip
    uint32_t carry = 0;                            // previous window's masked F (lane 31 / per lane)
    uint32_t p0 = a & ~3u;
    uint32_t lomask = FULL << (8 * (a & 3u));      // lane 0: pairs below the anchor
    const uint32_t lt_mask = lanemask_lt();
    const uint32_t qoff = 4 * (uint32_t)lane;
#pragma unroll 1
    for (;;) {
        if (p0 < wk.res_lo || p0 + (WIN_PAIRS + 4) > wk.res_hi) {
            uint32_t need_hi = p0 + WIN_PAIRS + 4;
            if (need_hi > lim2 + 2) need_hi = lim2 + 2;
            if (p0 < wk.res_lo || need_hi > wk.res_hi) walker_need(wk, p0, need_hi, lane);
        }
        const uint32_t q = p0 + qoff;
        const uint32_t x = lds32(wk.buf + (q & RING_MASK));
        const uint32_t xn = lds32(wk.buf + ((q + 4) & RING_MASK));
        const uint32_t y = __funnelshift_r(x, xn, 8);     // y_k = byte q+k+1
        uint32_t lt, gt;
        lt_gt_flags(x, y, lt, gt);
        uint32_t V = (lane ? FULL : lomask) & H;
        if (p0 + (WIN_PAIRS - 1) > lim2) {                // window crosses the last pair
            const int32_t sh = (int32_t)qoff * 8 + 24 - 8 * (int32_t)(lim2 - p0);
            V &= shr_c(FULL, sh > 0 ? (uint32_t)sh : 0u);
        }
        const uint32_t Fm = (MODE == 0 ? lt : gt) & V;
        const uint32_t Om = (MODE == 0 ? gt : lt) & V;
        const uint32_t R = run_mask<MSPEC>(Fm, carry, carry, p.M, lane);
        const uint32_t rmask = __ballot_sync(FULL, R != 0);
        const uint32_t cnt = __popc(Om);
        const uint32_t total = __reduce_add_sync(FULL, cnt);
        if (rmask == 0 && total < need) {          // nothing decided in this window
            need -= total;
            carry = MSPEC >= 0 ? __shfl_sync(FULL, Fm, 31) : Fm;
            p0 += WIN_PAIRS;
            lomask = FULL;
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
            // in lane dl: the k-th flag (k = need - excl); byte j of pc = flags in bytes 0..j
            const uint32_t k = need - excl;
            const uint32_t pc = (Om >> 7) * 0x01010101u;
            const uint32_t ge = ((pc | H) - k * 0x01010101u) & 0x00808080u;
            const uint32_t dbyte = 3u - __popc(ge);
            d = p0 + 4 * (uint32_t)dl + __shfl_sync(FULL, dbyte, dl);
        }
        if (r < d) return r + 2;                   // boundary after the run
        if (p.S >= lim2 - d) return limit;         // skip lands past the last pair (c8)
        a = d + 1 + p.S;                           // content-defined skip (c3)
        need = p.T;
        carry = 0;
        p0 = a & ~3u;
        lomask = FULL << (8 * (a & 3u));
    }
}

template <int MODE, int MSPEC>
__device__ __forceinline__ uint32_t resolve(Walker &wk, const DevParams &p, uint32_t base, int lane)
{
    return resolve_chunk<MODE, MSPEC>(wk, p, base, lane);
}

}  // namespace seqcdc
