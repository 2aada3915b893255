// seqcdc_device.cuh -- the warp-cooperative SeqCDC walker for sm_100a.
//
// One warp owns one speculative chain.  Its CTA streams the chain's bytes
// HBM -> shared memory through a ring of TILE-byte slots filled by 1-D TMA bulk
// copies (cp.async.bulk, completion on an mbarrier per slot).  The walk reads
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
// The ballot / __ffs / __reduce_add_sync / warp-scan primitives here play the
// role the paper gives to builtin_ffs, pdep+tzcnt and popcnt.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace seqcdc {

constexpr int TILE_SHIFT = 11;                       // 2 KiB ring slots
constexpr uint32_t TILE = 1u << TILE_SHIFT;
constexpr int STAGES = 8;                            // power of two
constexpr uint32_t RING = TILE * STAGES;             // 16 KiB per walker
constexpr uint32_t RING_MASK = RING - 1;
constexpr uint32_t WIN_PAIRS = 128;                  // pairs per window (32 lanes x 4)
constexpr uint32_t FULL = 0xffffffffu;
constexpr uint32_t H = 0x80808080u;

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
// bit 7 of each byte of the result = [x_k < y_k] (unsigned); other bits are junk.
// t = (~x & 7F) + (y & 7F) carries into bit 7 iff low7(y) > low7(x).
__device__ __forceinline__ void lt_gt_flags(uint32_t x, uint32_t y, uint32_t &lt, uint32_t &gt)
{
    uint32_t t = (~x & 0x7f7f7f7fu) + (y & 0x7f7f7f7fu);
    uint32_t u = 0xfefefefeu - t;  // = (~y & 7F) + (x & 7F), no inter-byte carries
    lt = (~x & y) | (~(x ^ y) & t);
    gt = (~y & x) | (~(x ^ y) & u);
}

// ------------------------------------------------------------------ shared-memory ring
struct Ring {
    uint32_t buf;       // shared address of the ring
    uint32_t bar;       // shared address of STAGES mbarriers (8 B each)
    uint64_t t_first;   // oldest tile still owned
    uint64_t t_next;    // next tile to issue
    uint64_t t_end;     // one past the last tile with data
    uint64_t a_lo, a_hi;  // absolute address range that may be loaded
    uint32_t pending;   // bit s: slot s holds an issued fill not yet waited for
    uint32_t nextpar;   // bit s: parity of the slot's next fill
};

__device__ __forceinline__ void ring_wait_slot(Ring &rg, uint32_t s)
{
    if (rg.pending & (1u << s)) {
        mbar_wait(rg.bar + 8 * s, ((rg.nextpar >> s) & 1u) ^ 1u);
        rg.pending &= ~(1u << s);
    }
}

__device__ __forceinline__ void ring_drain(Ring &rg)
{
#pragma unroll 1
    for (uint32_t s = 0; s < (uint32_t)STAGES; s++) ring_wait_slot(rg, s);
}

// Issue tile t (warp-uniform call).  TMA moves the 16-byte-aligned interior,
// lanes copy the <16-byte ragged head/tail of the loadable range.
__device__ __forceinline__ void ring_issue(Ring &rg, uint64_t t, int lane)
{
    const uint32_t s = (uint32_t)t & (STAGES - 1);
    ring_wait_slot(rg, s);  // never two fills in flight on one slot
    uint64_t lo = t << TILE_SHIFT, hi = lo + TILE;
    if (lo < rg.a_lo) lo = rg.a_lo;
    if (hi > rg.a_hi) hi = rg.a_hi;
    uint64_t mlo = (lo + 15) & ~15ull, mhi = hi & ~15ull;
    uint32_t tx = 0;
    if (lo < hi && mlo < mhi) tx = (uint32_t)(mhi - mlo);
    const uint32_t bar = rg.bar + 8 * s;
    if (lane == 0) {
        mbar_arrive_tx(bar, tx);
        if (tx) tma_load_1d(rg.buf + ((uint32_t)mlo & RING_MASK), (const void *)mlo, tx, bar);
    }
    if (lo < hi) {
        uint64_t addr;
        bool ok;
        if (tx) {
            addr = lane < 16 ? lo + lane : mhi + (lane - 16);
            ok = lane < 16 ? addr < mlo : addr < hi;
        } else {
            addr = lo + lane;
            ok = addr < hi;
        }
        if (ok) sts8(rg.buf + ((uint32_t)addr & RING_MASK), *(const volatile uint8_t *)addr);
    }
    __syncwarp();
    rg.pending |= 1u << s;
    rg.nextpar ^= 1u << s;
}

// Make absolute bytes [need_lo, need_hi) resident (need_hi - need_lo <= TILE).
__device__ __forceinline__ void ring_ensure(Ring &rg, uint64_t need_lo, uint64_t need_hi, int lane)
{
    const uint64_t tlo = need_lo >> TILE_SHIFT, thi = (need_hi - 1) >> TILE_SHIFT;
    if (tlo > rg.t_first) {
        rg.t_first = tlo;
        if (rg.t_next < tlo) rg.t_next = tlo;
    }
#pragma unroll 1
    while (rg.t_next < rg.t_end && rg.t_next < rg.t_first + STAGES) {
        ring_issue(rg, rg.t_next, lane);
        rg.t_next++;
    }
    ring_wait_slot(rg, (uint32_t)tlo & (STAGES - 1));
    if (thi != tlo) ring_wait_slot(rg, (uint32_t)thi & (STAGES - 1));
}

__device__ __forceinline__ void ring_start(Ring &rg, uint64_t a_lo, uint64_t a_hi, uint64_t from)
{
    ring_drain(rg);
    rg.a_lo = a_lo;
    rg.a_hi = a_hi;
    rg.t_end = a_hi > a_lo ? ((a_hi - 1) >> TILE_SHIFT) + 1 : 0;
    rg.t_first = rg.t_next = from >> TILE_SHIFT;
}

// ------------------------------------------------------------------ one chunk
// "shfl_up by k with carry-in from the previous window": lanes < k take the
// previous window's word from lane 32-k+lane.
__device__ __forceinline__ uint32_t prev_word(uint32_t cur, uint32_t prevwin, int k, int lane)
{
    uint32_t a = __shfl_sync(FULL, cur, (lane - k) & 31);
    uint32_t b = __shfl_sync(FULL, prevwin, (lane - k) & 31);
    return lane >= k ? a : b;
}

// R for pairs of this lane's word: AND over j in [0, M) of F shifted by j pairs.
template <bool SMALL_M>
__device__ __forceinline__ uint32_t runs(uint32_t Fm, uint32_t Fprev, uint32_t M, int lane)
{
    uint32_t R = Fm;
    if (M <= 1) return R;
    uint32_t W1 = prev_word(Fm, Fprev, 1, lane);
    if (SMALL_M) {  // M <= 4: one word back suffices
#pragma unroll
        for (uint32_t j = 1; j < 4; j++)
            if (j < M) R &= __funnelshift_l(W1, Fm, 8 * j);
        return R;
    } else {        // M <= 16: up to four words back
        uint32_t W[5];
        W[0] = Fm;
        W[1] = W1;
        W[2] = prev_word(Fm, Fprev, 2, lane);
        W[3] = prev_word(Fm, Fprev, 3, lane);
        W[4] = prev_word(Fm, Fprev, 4, lane);
#pragma unroll
        for (uint32_t j = 1; j < 16; j++)
            if (j < M) R &= __funnelshift_l(W[(j >> 2) + 1], W[j >> 2], 8 * (j & 3));
        return R;
    }
}

// f(base): the cut ending the chunk that starts at absolute address `base` of a
// stream ending at `end`.  Warp-uniform; all lanes return the same value.
template <int MODE, bool SMALL_M>
__device__ __forceinline__ uint64_t resolve_chunk(Ring &rg, const DevParams &p, uint64_t base, uint64_t end,
                                               int lane)
{
    uint64_t limit = base + p.mx;
    if (limit > end) limit = end;
    if (limit - base < 2) return limit;
    const uint64_t lim2 = limit - 2;               // last pair that may be examined
    uint64_t a = base + p.mn - p.L;
    if (a > lim2) return limit;
    uint32_t oc = 0;                               // opposing pairs counted since a
    uint32_t Fprev = 0;                            // previous window's masked F word
    uint64_t p0 = a & ~3ull;
#pragma unroll 1
    for (;;) {
        uint64_t need_hi = p0 + WIN_PAIRS + 4;
        if (need_hi > lim2 + 2) need_hi = lim2 + 2;
        ring_ensure(rg, p0, need_hi, lane);
        const uint64_t q = p0 + 4 * (uint32_t)lane;
        const uint32_t x = lds32(rg.buf + ((uint32_t)q & RING_MASK));
        const uint32_t xn = lds32(rg.buf + ((uint32_t)(q + 4) & RING_MASK));
        const uint32_t y = __funnelshift_r(x, xn, 8);     // y_k = byte (q+k+1)
        uint32_t lt, gt;
        lt_gt_flags(x, y, lt, gt);
        uint32_t F = MODE == 0 ? lt : gt;
        uint32_t O = MODE == 0 ? gt : lt;
        // valid pairs: a <= pair <= lim2
        const int32_t ra = a > p0 ? (int32_t)(a - p0) : 0;                 // 0..3
        const uint64_t dh = lim2 - p0;
        const int32_t rh = dh > 256 ? 256 : (int32_t)dh;
        const int32_t lo_l = ra - 4 * lane, hi_l = rh - 4 * lane;
        const uint32_t slo = lo_l <= 0 ? 0u : (uint32_t)lo_l * 8u;
        const uint32_t shi = hi_l >= 3 ? 0u : (hi_l < 0 ? 32u : (uint32_t)(3 - hi_l) * 8u);
        const uint32_t V = shl_c(FULL, slo) & shr_c(FULL, shi) & H;
        const uint32_t Fm = F & V, Om = O & V;
        const uint32_t R = runs<SMALL_M>(Fm, Fprev, p.M, lane);
        const uint32_t rmask = __ballot_sync(FULL, R != 0);
        const uint32_t cnt = __popc(Om);
        const uint32_t total = __reduce_add_sync(FULL, cnt);
        const uint32_t need = p.T - oc;
        if (rmask == 0 && total < need) {          // nothing decided in this window
            oc += total;
            Fprev = Fm;
            p0 += WIN_PAIRS;
            if (p0 > lim2) return limit;
            continue;
        }
        uint64_t r = ~0ull, d = ~0ull;
        if (rmask) {
            const int rl = __ffs(rmask) - 1;
            const uint32_t rb = (uint32_t)(__ffs(R) - 1) >> 3;
            r = p0 + 4 * (uint32_t)rl + __shfl_sync(FULL, rb, rl);
        }
        if (total >= need) {
            uint32_t incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t v = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += v;
            }
            const int dl = __ffs(__ballot_sync(FULL, incl >= need)) - 1;
            uint32_t k = need - (incl - cnt);       // rank inside lane dl (valid there)
            uint32_t m = Om;
            for (uint32_t j = 1; j < k && j < 4; j++) m &= m - 1;
            const uint32_t db = (uint32_t)(__ffs(m) - 1) >> 3;
            d = p0 + 4 * (uint32_t)dl + __shfl_sync(FULL, db, dl);
        }
        if (r < d) return r + 2;                   // boundary after the run
        a = d + 1 + p.S;                           // content-defined skip (c3)
        if (a > lim2) return limit;
        oc = 0;
        Fprev = 0;
        p0 = a & ~3ull;
    }
}

}  // namespace seqcdc
