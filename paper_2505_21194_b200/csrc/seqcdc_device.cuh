// seqcdc_device.cuh -- the warp-cooperative SeqCDC walker for sm_100a.
//
// One warp owns one speculative chain.  It streams the chain's bytes
// HBM -> shared memory through a ring of NBLK blocks of BLK bytes, each block
// one cp.async group of 16-byte per-lane copies (LDGSTS, L1-bypassing .cg),
// kept AHEAD blocks in front of the walk.  The walk reads only the
// windows the method examines and classifies adjacent byte pairs lazily with
// SIMD-in-word compares (4 pairs per 32-bit word, one word per lane => 128
// pairs per window):
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
// address `rb` (so a byte's ring slot offset is just `pos & RING_MASK` and
// 16-byte alignment of the copies is preserved).  A job (segment + its
// extension, or one <=1 GiB piece of a fallback walk) stays far below 2^32.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace seqcdc {

// Device-side invariant checks (a -DSEQCDC_DEBUG build; compute-sanitizer is
// not available on the GPU pool): a violated invariant stops the kernel with
// __trap(), which the next synchronisation reports as a launch failure.
#ifdef SEQCDC_DEBUG
#define SEQCDC_ASSERT(cond)      \
    do {                         \
        if (!(cond)) __trap();   \
    } while (0)
#else
#define SEQCDC_ASSERT(cond) \
    do {                    \
    } while (0)
#endif

// A chunk [base, cut) of a stream whose data ends at `end` (relative
// positions): it is not empty, at most max_size long, and at least
// min_size long unless it is the stream's last chunk (c9).
#define SEQCDC_ASSERT_CUT(base, cut, p, end) \
    SEQCDC_ASSERT((cut) > (base) && (cut) - (base) <= (p).mx && ((cut) - (base) >= (p).mn || (cut) == (end)))

// Ring geometry (profiles/r01/sweeps.md): 2 KiB blocks (4 x 16-byte cp.async per
// lane each), 4 slots, 2 blocks (4 KiB) in flight ahead of the window.
#ifndef SEQCDC_BLK_SHIFT
#define SEQCDC_BLK_SHIFT 11
#endif
#ifndef SEQCDC_NBLK
#define SEQCDC_NBLK 4
#endif
#ifndef SEQCDC_AHEAD
#define SEQCDC_AHEAD 2
#endif
#ifndef SEQCDC_L2PF
#define SEQCDC_L2PF 0
#endif
constexpr int BLK_SHIFT = SEQCDC_BLK_SHIFT;          // ring block size (log2)
constexpr uint32_t BLK = 1u << BLK_SHIFT;
constexpr uint32_t NBLK = SEQCDC_NBLK;               // blocks in the ring (power of two)
constexpr uint32_t AHEAD = SEQCDC_AHEAD;             // blocks kept in flight past the window
#ifndef SEQCDC_SPARSE
#define SEQCDC_SPARSE 0
#endif
#ifndef SEQCDC_HINT_BLOCKS
#define SEQCDC_HINT_BLOCKS 3
#endif
constexpr uint32_t SBLK_SHIFT = 9;                   // sparse cache: 512-byte blocks (one 16-B copy per lane)
constexpr uint32_t SBLK = 1u << SBLK_SHIFT;
constexpr uint32_t NS = 32;                          // sparse cache slots (16 KiB)
constexpr uint32_t DRING = BLK * NBLK;               // dense ring: 8 KiB per walker (default geometry)
constexpr uint32_t SRING = SBLK * NS;                // sparse block cache: 16 KiB per walker
#if SEQCDC_SPARSE
constexpr uint32_t RING = SRING;                     // the walker k_walk & co. use (build option)
#else
constexpr uint32_t RING = DRING;
#endif
static_assert(AHEAD + 2 <= NBLK, "ring must hold the window's two blocks plus the lookahead");
static_assert(BLK >= 512 && BLK % 512 == 0, "a block is whole rounds of 32 x 16-byte copies");
constexpr uint32_t WIN_PAIRS = 128;                  // pairs per window (32 lanes x 4)
constexpr uint32_t FULL = 0xffffffffu;
constexpr uint32_t H = 0x80808080u;
constexpr uint32_t REL_CLAMP = 0xC0000000u;          // relative positions stay below this
constexpr uint32_t JOB_SPAN = 0x40000000u;           // fallback walks restart a job every 1 GiB
constexpr uint32_t SMEM_WALK = RING;                 // dynamic smem of one walker

struct DevParams {
    uint32_t L, T, S, M;   // M = L-1 favourable pairs per run
    uint32_t mn, mx;       // min/max chunk sizes (<= 2^28, validated on the host)
    uint32_t mnL;          // mn - L: offset of the scan anchor from the chunk start
    uint32_t bs, nb, ah;   // ring geometry (reported; compile-time in this build)
};

// the walker's ring is a static __shared__ array: no dynamic shared memory
__host__ __device__ __forceinline__ uint32_t walker_smem(const DevParams &) { return 0; }

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void cp_async16(uint32_t dst, uint64_t src)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}

__device__ __forceinline__ void cp_async_commit()
{
    asm volatile("cp.async.commit_group;" ::: "memory");
}

template <int N>
__device__ __forceinline__ void cp_async_wait()
{
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// wait until at most n (0..7) of this thread's most recent groups are pending
__device__ __forceinline__ void cp_async_wait_n(uint32_t n)
{
    switch (n) {
    case 0: cp_async_wait<0>(); break;
    case 1: cp_async_wait<1>(); break;
    case 2: cp_async_wait<2>(); break;
    case 3: cp_async_wait<3>(); break;
    case 4: cp_async_wait<4>(); break;
    case 5: cp_async_wait<5>(); break;
    case 6: cp_async_wait<6>(); break;
    default: cp_async_wait<7>(); break;
    }
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

// shr with PTX clamp semantics (shift >= 32 gives 0)
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

// ------------------------------------------------------------------ the shared-memory ring
// Software-pipelined cp.async ring: BLK-byte blocks are issued strictly in order,
// one cp.async group each; the walk keeps exactly AHEAD groups in flight past
// the block holding the end of its current window, so `cp.async.wait_group
// AHEAD` (a constant) proves that window resident.  Block b lives in slot
// b % NBLK; a slot is only refilled once its previous block is known to have
// landed (else the ring drains first -- only after jumps of > NBLK-AHEAD blocks).
struct DWalker {
    static constexpr uint32_t BYTES = DRING, MASK = DRING - 1;
    uint64_t rb;        // absolute address of relative position 0 (RING-aligned)
    uint32_t lo_rel;    // first loadable byte (relative)
    uint32_t end_rel;   // end of the stream (relative, clamped to REL_CLAMP)
    uint32_t buf;       // shared address of the ring
    uint32_t b_next;    // next block to issue
    uint32_t b_ok;      // blocks below b_ok have landed (or were never issued)
};

// Issue block b (warp-uniform): one cp.async group (empty past the data).
__device__ __forceinline__ void ring_issue(DWalker &wk, uint32_t b, int lane)
{
    const uint32_t b0 = b << BLK_SHIFT;
#if SEQCDC_L2PF > 0
    {   // pull the block SEQCDC_L2PF blocks further ahead into L2 (one bulk prefetch, no smem)
        const uint32_t pf = b0 + SEQCDC_L2PF * BLK;
        if (lane == 0 && pf + BLK <= wk.end_rel)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(wk.rb + pf), "r"(BLK) : "memory");
    }
#endif
    if (b0 >= wk.lo_rel && b0 + BLK <= wk.end_rel) {
        SEQCDC_ASSERT(b0 + BLK <= REL_CLAMP);
        // a whole block: one base address per side, the k*512 steps become
        // immediate offsets of the copies (a block never wraps the ring)
        const uint32_t dst = wk.buf + (b0 & DWalker::MASK) + 16 * (uint32_t)lane;
        const uint64_t src = wk.rb + b0 + 16 * (uint32_t)lane;
#pragma unroll
        for (uint32_t k = 0; k < BLK / 512; k++) cp_async16(dst + k * 512, src + k * 512);
    } else if (b0 < wk.end_rel) {
#pragma unroll 1
        for (uint32_t k = 0; k < BLK / 512; k++) {
            const uint32_t c = b0 + k * 512 + 16 * (uint32_t)lane;
            if (c >= wk.lo_rel && c + 16 <= wk.end_rel) {
                cp_async16(wk.buf + (c & DWalker::MASK), wk.rb + c);
            } else {
#pragma unroll 1
                for (uint32_t x = c; x < c + 16; x++)
                    if (x >= wk.lo_rel && x < wk.end_rel)
                        sts8(wk.buf + (x & DWalker::MASK), *(const volatile uint8_t *)(wk.rb + x));
            }
        }
    }
    cp_async_commit();
}

// Make bytes [need_lo, need_hi) resident (need_hi - need_lo <= BLK + 4).
__device__ __forceinline__ void ring_need(DWalker &wk, uint32_t need_lo, uint32_t need_hi, int lane)
{
    const uint32_t bw = (need_hi - 1) >> BLK_SHIFT;
    if (bw + AHEAD >= wk.b_next) {
        if (bw + AHEAD >= wk.b_ok + NBLK) {      // a big jump: let everything in flight land
            cp_async_wait<0>();
            wk.b_ok = wk.b_next;
            const uint32_t blo = need_lo >> BLK_SHIFT;
            if (wk.b_next < blo) wk.b_next = wk.b_ok = blo;   // blocks jumped over are never loaded
        }
#pragma unroll 1
        do {
            ring_issue(wk, wk.b_next, lane);
            wk.b_next++;
        } while (wk.b_next <= bw + AHEAD);
    }
    cp_async_wait<AHEAD>();                      // every block <= b_next-1-AHEAD (>= bw) has landed
    __syncwarp();                                // other lanes' copies visible
    wk.b_ok = wk.b_next - AHEAD;
}

// `ring` is a static __shared__ array of RING bytes in the calling kernel (its
// shared address is then a link-time constant).
__device__ __forceinline__ void walker_init(DWalker &wk, uint8_t *smem, const DevParams &, int)
{
    // opaque to the compiler: kept in a register instead of being re-derived from
    // the CTA's shared window id (S2UR, long latency) at every use
    uint32_t sb = smem_u32(smem);
    asm volatile("mov.b32 %0, %0;" : "+r"(sb));
    wk.buf = sb;
    wk.rb = 0;
    wk.lo_rel = wk.end_rel = 0;
    wk.b_next = wk.b_ok = 0;
}

// Start a job whose loadable data is absolute [a_lo, a_end); returns the
// relative position of a_lo.  Outstanding copies of the previous job land first.
__device__ __forceinline__ uint32_t walker_begin(DWalker &wk, uint64_t a_lo, uint64_t a_end)
{
    cp_async_wait<0>();
    __syncwarp();
    wk.rb = a_lo & ~(uint64_t)DWalker::MASK;
    wk.lo_rel = (uint32_t)(a_lo - wk.rb);
    const uint64_t e = a_end > a_lo ? a_end - wk.rb : wk.lo_rel;
    wk.end_rel = e > REL_CLAMP ? REL_CLAMP : (uint32_t)e;
    wk.b_next = wk.b_ok = wk.lo_rel >> BLK_SHIFT;
    return wk.lo_rel;
}

__device__ __forceinline__ void walker_finish(DWalker &wk)
{
    cp_async_wait<0>();
    __syncwarp();
}

// (dense ring: no hint needed, the ring streams every byte)
__device__ __forceinline__ void ring_hint_next(DWalker &, uint32_t, uint32_t, int) {}
// ------------------------------------------------------------------ sparse (skip-aware) block cache, NEXT-2
// Instead of streaming every byte, the walker fetches only the 512-byte blocks
// it examines, into a direct-mapped cache of NS slots (slot = block % NS), plus
// prefetches: the next two blocks past each window, and at each chunk start the
// region where the NEXT chunk's scan will most likely start (anchor + min - L,
// P:179).  The sub-minimum region of every chunk and most of each content-
// defined skip are never read from HBM: this is the paper's skipping
// turned into saved memory traffic.  Tags live one per lane (lane s = slot s).
struct SWalker {
    static constexpr uint32_t BYTES = SRING, MASK = SRING - 1;
    uint64_t rb;        // absolute address of relative position 0 (cache-aligned)
    uint32_t lo_rel;    // first loadable byte (relative)
    uint32_t end_rel;   // end of the stream (relative, clamped to REL_CLAMP)
    uint32_t buf;       // shared address of the cache
    uint32_t tag;       // this lane's slot: block held (FULL = none)
    uint32_t seq;       // this lane's slot: cp.async group that fills it
    uint32_t gseq;      // groups committed so far (warp-uniform)
    uint32_t ready;     // slots known to have landed (warp-uniform bit mask)
};

__device__ __forceinline__ void cache_fill(SWalker &wk, uint32_t b, int lane)
{
    const uint32_t s = b & (NS - 1);
    const uint32_t x0 = b << SBLK_SHIFT;
    const uint32_t dst = wk.buf + (s << SBLK_SHIFT);
    if (x0 >= wk.lo_rel && x0 + SBLK <= wk.end_rel) {
        cp_async16(dst + 16 * (uint32_t)lane, wk.rb + x0 + 16 * (uint32_t)lane);
    } else if (x0 < wk.end_rel) {
#pragma unroll 1
        for (uint32_t x = x0 + (uint32_t)lane; x < x0 + SBLK; x += 32)
            if (x >= wk.lo_rel && x < wk.end_rel)
                sts8(dst + (x - x0), *(const volatile uint8_t *)(wk.rb + x));
    }
    cp_async_commit();
    if (lane == (int)s) {
        wk.tag = b;
        wk.seq = wk.gseq;
    }
    wk.gseq++;
    wk.ready &= ~(1u << s);
}

// wait until slot s has landed (every lane committed the same groups)
__device__ __forceinline__ void cache_wait(SWalker &wk, uint32_t s)
{
    const uint32_t after = wk.gseq - 1 - __shfl_sync(FULL, wk.seq, s);   // groups committed after it
    const uint32_t n = after < 7 ? after : 7;
    cp_async_wait_n(n);
    __syncwarp();
    const uint32_t done = wk.gseq - 1 - n;                               // groups <= done have landed
    wk.ready |= __ballot_sync(FULL, wk.tag != FULL && wk.seq <= done);
}

// make block b resident (warp-uniform)
__device__ __forceinline__ void cache_need(SWalker &wk, uint32_t b, int lane)
{
    const uint32_t s = b & (NS - 1);
    if (__shfl_sync(FULL, wk.tag, s) != b) cache_fill(wk, b, lane);
    if (!((wk.ready >> s) & 1u)) cache_wait(wk, s);
}

// start fetching block b unless present or its slot holds a block of the window [wl, wh]
__device__ __forceinline__ void cache_prefetch(SWalker &wk, uint32_t b, uint32_t wl, uint32_t wh, int lane)
{
    const uint32_t s = b & (NS - 1);
    if (b > (wk.end_rel >> SBLK_SHIFT) || ((b - wl) & (NS - 1)) <= wh - wl) return;
    if (__shfl_sync(FULL, wk.tag, s) != b) cache_fill(wk, b, lane);
}

// Make bytes [need_lo, need_hi) resident (need_hi - need_lo <= SBLK + 4).
__device__ __forceinline__ void ring_need(SWalker &wk, uint32_t need_lo, uint32_t need_hi, int lane)
{
    const uint32_t bl = need_lo >> SBLK_SHIFT, bh = (need_hi - 1) >> SBLK_SHIFT;
    cache_need(wk, bl, lane);
    if (bh != bl) cache_need(wk, bh, lane);
    cache_prefetch(wk, bh + 1, bl, bh, lane);
    cache_prefetch(wk, bh + 2, bl, bh, lane);
}

// at a chunk's first window (anchor a): prefetch where the next chunk's scan starts
__device__ __forceinline__ void ring_hint_next(SWalker &wk, uint32_t next_lo, uint32_t a, int lane)
{
    const uint32_t wl = a >> SBLK_SHIFT;
    const uint32_t b0 = next_lo >> SBLK_SHIFT;
#pragma unroll
    for (uint32_t k = 0; k < SEQCDC_HINT_BLOCKS; k++) cache_prefetch(wk, b0 + k, wl, wl + 1, lane);
}

__device__ __forceinline__ void walker_init(SWalker &wk, uint8_t *smem, const DevParams &, int)
{
    uint32_t sb = smem_u32(smem);
    asm volatile("mov.b32 %0, %0;" : "+r"(sb));
    wk.buf = sb;
    wk.rb = 0;
    wk.lo_rel = wk.end_rel = 0;
    wk.tag = FULL;
    wk.seq = 0;
    wk.gseq = 0;
    wk.ready = 0;
}

__device__ __forceinline__ uint32_t walker_begin(SWalker &wk, uint64_t a_lo, uint64_t a_end)
{
    cp_async_wait<0>();
    __syncwarp();
    wk.rb = a_lo & ~(uint64_t)SWalker::MASK;
    wk.lo_rel = (uint32_t)(a_lo - wk.rb);
    const uint64_t e = a_end > a_lo ? a_end - wk.rb : wk.lo_rel;
    wk.end_rel = e > REL_CLAMP ? REL_CLAMP : (uint32_t)e;
    wk.tag = FULL;
    wk.ready = 0;
    return wk.lo_rel;
}

__device__ __forceinline__ void walker_finish(SWalker &)
{
    cp_async_wait<0>();
    __syncwarp();
}

#if SEQCDC_SPARSE
using Walker = SWalker;
#else
using Walker = DWalker;
#endif
constexpr uint32_t RING_MASK = RING - 1;

// ------------------------------------------------------------------ one chunk
// Favourable-run mask R for M = L-1 pairs.  MSPEC = 4: exactly four (L = 5,
// Table I); MSPEC = 0: any M <= 4 (runtime); MSPEC = -1: 5 <= M <= 15, using up
// to four words back (the previous window's words arrive by shuffles).
template <int MSPEC>
__device__ __forceinline__ uint32_t run_mask(uint32_t Fm, uint32_t carry, uint32_t M, int lane)
{
    if (MSPEC >= 0) {
        const uint32_t up = __shfl_up_sync(FULL, Fm, 1);
        const uint32_t W1 = lane ? up : carry;
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
            const uint32_t b1 = __shfl_sync(FULL, carry, (lane - k) & 31);
            Wd[k] = lane >= k ? a1 : b1;
        }
        uint32_t R = Fm;
#pragma unroll
        for (uint32_t j = 1; j < 16; j++)
            if (j < M) R &= __funnelshift_l(Wd[(j >> 2) + 1], Wd[j >> 2], 8 * (j & 3));
        return R;
    }
}

// f(base): the cut ending the chunk that starts at relative position `base`
// (base < end_rel).  Warp-uniform; every lane returns the same value.
//
// One round per examined window of 128 pairs (4 per lane).  Each lane finds
// its own candidates, a warp min-reduction (REDUX) picks the first of each:
//   r = first pair ending a favourable run (per-lane __ffs, "builtin_ffs")
//   d = the need-th opposing pair: per-lane exclusive prefix of the opposing
//       counts from three count-bit ballots, the crossing lane's byte by a
//       SWAR prefix ("pdep + tzcnt").
// r < d -> cut r+2; d < r -> skip to d+1+S with fresh counters;
// neither -> next window.  Pairs and bytes come from the warp's ring.
// (The min-reduction replaced ballot + ffs + shuffle: lone-walker latency
// 0.80 -> 0.745 us per chunk, profiles/r01/sweeps.md.)
// RED selects how the decision finds the first run end / the T-th opposing
// pair: true = per-lane candidates + two warp min-reductions (REDUX: shortest
// dependent chain, used where a walker runs alone, i.e. extensions and
// re-walks), false = two ballots + __ffs + two shuffles (cheaper in issue
// slots, used for the speculative bulk, which shares the SM with 21 others).
#ifndef SEQCDC_DEC_FORCE
#define SEQCDC_DEC_FORCE -1   // tuning: 0 = ballots everywhere, 1 = REDUX everywhere
#endif
template <int MODE, int MSPEC, bool RED_ = true, class W = Walker>
__device__ __forceinline__ uint32_t resolve(W &wk, const DevParams &p, uint32_t base, int lane)
{
    constexpr bool RED = SEQCDC_DEC_FORCE < 0 ? RED_ : SEQCDC_DEC_FORCE == 1;
    uint32_t limit = base + p.mx;                  // P:266 (no overflow: base < 3 GiB, mx <= 2^28)
    if (limit > wk.end_rel) limit = wk.end_rel;
    const uint32_t lim2 = limit - 2;               // last pair that may be examined
    uint32_t a = base + p.mnL;
    if (limit - base < 2 || a > lim2) return limit;
    uint32_t need = p.T;                           // opposing pairs still needed for a skip
    uint32_t carry = 0;                            // previous window's masked F (lane 31 / per lane)
    uint32_t p0 = a & ~3u;
    uint32_t lomask = FULL << (8 * (a & 3u));      // lane 0: pairs below the anchor
    const uint32_t qoff = 4 * (uint32_t)lane;
    const uint32_t lt_mask = lanemask_lt();
    bool first = true;
#pragma unroll 1
    for (;;) {
        {
            uint32_t need_hi = p0 + WIN_PAIRS + 4;
            if (need_hi > lim2 + 2) need_hi = lim2 + 2;
            ring_need(wk, p0, need_hi, lane);
            if (first) {                           // the next chunk's scan starts near a + min - L
                ring_hint_next(wk, a + p.mnL, p0, lane);
                first = false;
            }
        }
        SEQCDC_ASSERT(p0 + 4 > wk.lo_rel && p0 <= lim2);
        const uint32_t q = p0 + qoff;
        // MODE bit 0: Decreasing; bit 1: signed reading (flipping bit 7 of every
        // byte maps int8 order onto uint8 order)
        constexpr uint32_t XM = (MODE & 2) ? H : 0u;
        const uint32_t x = lds32(wk.buf + (q & W::MASK)) ^ XM;
        const uint32_t xn = lds32(wk.buf + ((q + 4) & W::MASK)) ^ XM;
        const uint32_t y = __funnelshift_r(x, xn, 8);     // y_k = byte q+k+1
        uint32_t lt, gt;
        lt_gt_flags(x, y, lt, gt);
        // Pairs past lim2 (the window's tail at the chunk limit) are NOT masked: the
        // ring bytes there may be stale, so any event found past lim2 is discarded
        // below (events are taken in pair order, so a stale one can only come after
        // every valid one).
        const uint32_t V = (lane ? FULL : lomask) & H;
        const uint32_t Fm = ((MODE & 1) == 0 ? lt : gt) & V;
        const uint32_t Om = ((MODE & 1) == 0 ? gt : lt) & V;
        const uint32_t R = run_mask<MSPEC>(Fm, carry, p.M, lane);
        const uint32_t cnt = __popc(Om);
        const uint32_t b0 = __ballot_sync(FULL, cnt & 1), b1 = __ballot_sync(FULL, cnt & 2),
                       b2 = __ballot_sync(FULL, cnt & 4);
        const uint32_t excl = __popc(b0 & lt_mask) + 2 * __popc(b1 & lt_mask) + 4 * __popc(b2 & lt_mask);
        constexpr uint32_t NONE = 0xffffffffu;
        uint32_t r = NONE, d = NONE, rmask = 0, dmask = 0;
        if (RED) {
            // per-lane candidates, the first of each by a warp min-reduction
            const uint32_t rc = R ? 4 * (uint32_t)lane + ((uint32_t)(__ffs(R) - 1) >> 3) : NONE;
            const uint32_t pcr = (Om >> 7) * 0x01010101u;
            const uint32_t ger = ((pcr | H) - (need - excl) * 0x01010101u) & 0x00808080u;
            const uint32_t dc = (excl < need && excl + cnt >= need) ? 4 * (uint32_t)lane + 3u - __popc(ger) : NONE;
            r = __reduce_min_sync(FULL, rc);
            d = __reduce_min_sync(FULL, dc);
        } else {
            rmask = __ballot_sync(FULL, R != 0);
            dmask = __ballot_sync(FULL, excl + cnt >= need);
        }
        if (RED ? (r & d) == NONE : (rmask | dmask) == 0) {   // nothing decided in this window
            need -= __popc(b0) + 2 * __popc(b1) + 4 * __popc(b2);
            carry = MSPEC >= 0 ? __shfl_sync(FULL, Fm, 31) : Fm;
            const bool flat = !__any_sync(FULL, (Fm | Om) != 0);
            p0 += WIN_PAIRS;
            lomask = FULL;
            if (p0 > lim2) return limit;
            if (flat) {
                // A window of equal bytes only (zero runs, constant data): neither
                // favourable nor opposing pairs, so the counters do not
                // move.  Gallop 512 pairs per step (16 per lane) while the bytes stay
                // equal; resume window by window at the first step with a change.
#pragma unroll 1
                for (;;) {
                    uint32_t nh = p0 + 4 * WIN_PAIRS + 4;
                    if (nh > lim2 + 2) nh = lim2 + 2;
                    ring_need(wk, p0, nh, lane);
                    const uint32_t q16 = p0 + 16 * (uint32_t)lane;
                    uint32_t wv[5];
#pragma unroll
                    for (int k = 0; k < 5; k++) wv[k] = lds32(wk.buf + ((q16 + 4 * k) & W::MASK));
                    uint32_t diff = 0;
#pragma unroll
                    for (int k = 0; k < 4; k++) diff |= wv[k] ^ __funnelshift_r(wv[k], wv[k + 1], 8);
                    if (__any_sync(FULL, diff != 0)) break;   // (stale bytes past lim2 only cost a window)
                    p0 += 4 * WIN_PAIRS;
                    if (p0 > lim2) return limit;
                }
            }
            continue;
        }
        if (!RED) {
            // per lane: byte of its first run end, byte of its k-th opposing pair
            // (k = need - excl; byte j of pc = opposing flags in bytes 0..j)
            const uint32_t rbyte = (uint32_t)(__ffs(R) - 1) >> 3;
            const uint32_t pc = (Om >> 7) * 0x01010101u;
            const uint32_t ge = ((pc | H) - (need - excl) * 0x01010101u) & 0x00808080u;
            const uint32_t dbyte = 3u - __popc(ge);
            const uint32_t rl = rmask ? (uint32_t)__ffs(rmask) - 1 : 32u;
            const uint32_t dl = dmask ? (uint32_t)__ffs(dmask) - 1 : 32u;
            r = 4 * rl + __shfl_sync(FULL, rbyte, rl & 31);
            d = 4 * dl + __shfl_sync(FULL, dbyte, dl & 31);
        }
        if (r < d) {                               // the run completes first: boundary after it
            const uint32_t ra = p0 + r;
            return ra <= lim2 ? ra + 2 : limit;
        }
        const uint32_t da = p0 + d;                // the need-th opposing pair triggers a skip
        if (da > lim2 || p.S >= lim2 - da) return limit;   // no skip before the limit / lands past it (c8)
        a = da + 1 + p.S;                          // content-defined skip (c3)
        need = p.T;
        carry = 0;
        p0 = a & ~3u;
        lomask = FULL << (8 * (a & 3u));
    }
}

}  // namespace seqcdc
