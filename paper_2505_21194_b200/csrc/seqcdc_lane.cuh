// seqcdc_lane.cuh -- the per-lane, skip-aware SeqCDC walker (SURVEY.md 8(f)
// NEXT-2 made the hot path for long streams).  Included by seqcdc.cu after the
// segment helpers (Work, Seg, get_seg, seg_start, fix_overflows).
//
// Why: the method itself never reads the sub-minimum region of a chunk
// nor the bytes a content-defined skip jumps over; on config 5
// it compares bytes in only 3.8% of the stream's 32-B sectors.  The warp
// walker streams every byte through shared memory and is therefore bound by
// HBM at ~n / 6.6 TB/s.  Here every LANE owns one speculative chain (one
// segment) and fetches only the 128-B lines its scan touches, as 16-B
// cp.async copies into two private line slots whose completion arrives on the
// slot's own mbarrier (cp.async.mbarrier.arrive.noinc).  A lane whose line has
// not landed simply skips that loop iteration (mbarrier.test_wait, no
// blocking), so the warp keeps scanning for the lanes whose data is there;
// thousands of chains per SM hide the HBM latency of the dependent
// chunk-to-chunk jumps.  (Measured alternatives, profiles/r02/lane_walker.md:
// one cp.async.bulk per line is slower -- 5.23 vs 4.37 ms on config 5 --, and
// testing every pending slot each step costs more than testing only the slot
// the scan needs, because every barrier test is a per-thread operation.)
//
// One loop iteration of a lane examines one group of GRP = 32 byte pairs
// (bytes q..q+32), classified with SIMD-in-word compares (4 pairs per 32-bit
// word) and packed into 32-bit pair masks in pair order; the
// favourable-run mask is an AND of shifted copies of the favourable mask with
// the previous group's pairs shifted in, the opposing count a
// popc, the SkipTrigger-th opposing pair a popc bisection.
// Decision in pair order: run end first -> cut; T-th opposing pair
// first -> skip to d+1+S with fresh counters (reading c3); neither ->
// next group; past the limit -> forced cut.
//
// Segment protocol (same lists as the warp walker, so the post kernels are
// shared): the lane records its speculative cuts < segment end in L_s and
// publishes the count with release semantics ONCE, when the speculative part
// is complete (DONE).  Its extension then walks on, checking each cut against
// the DONE list of the chain owning that region (a cut not yet decidable is
// simply walked past: after a merge both chains are identical, so any later
// common cut is a merge too).
#pragma once

namespace seqcdc {
namespace lw {

#ifndef SEQCDC_LW_LINE_SHIFT
#define SEQCDC_LW_LINE_SHIFT 7
#endif
#ifndef SEQCDC_LW_WARPS
#define SEQCDC_LW_WARPS 4
#endif
#ifndef SEQCDC_LW_PF
#define SEQCDC_LW_PF 96        // prefetch the next line once the scan is this far into a line
#endif
#ifndef SEQCDC_LW_PACKED
#define SEQCDC_LW_PACKED 1     // packed pair masks (scan_group_p); 0: the per-word form (scan_group)
#endif
#ifndef SEQCDC_LW_LAZY
#define SEQCDC_LW_LAZY 1       // test a slot's barrier only when its line is needed (barrier ops are costly)
#endif
#ifndef SEQCDC_LW_GROUP
#define SEQCDC_LW_GROUP 32     // byte pairs examined per lane per step (16 or 32; 32 needs SEQCDC_LW_PACKED)
#endif
#ifndef SEQCDC_LW_BATCH
#define SEQCDC_LW_BATCH 0      // fills of one warp step complete on one of 8 per-warp barriers (no per-lane arrive loop)
#endif
#ifndef SEQCDC_LW_PAIR
#define SEQCDC_LW_PAIR 1       // a dependent miss fills the line and its successor with one barrier arrival (4.81 -> 4.63 ms on config 5)
#endif
#ifndef SEQCDC_LW_BULK
#define SEQCDC_LW_BULK 0       // line fills by cp.async.bulk (TMA) instead of 8 x 16-B cp.async
#endif
#ifndef SEQCDC_LW_ONEFILL
#define SEQCDC_LW_ONEFILL 0    // one fill site (measured slower: 4.85 vs 4.61 ms on config 5)
#endif
#ifndef SEQCDC_LW_L2PF
#define SEQCDC_LW_L2PF 0       // lines of the likely next anchor region warmed in L2 per chunk
#endif
#ifndef SEQCDC_LW_L2PF_OFF
#define SEQCDC_LW_L2PF_OFF 0   // ... starting this many bytes past anchor + min - L
#endif

constexpr uint32_t LSH = SEQCDC_LW_LINE_SHIFT;
constexpr uint32_t LINE = 1u << LSH;                 // bytes per bulk copy / slot
constexpr uint32_t LMASK = LINE - 1;
constexpr uint32_t STRIDE = 2 * LINE + 16;           // per lane: 2 slots + 16 B of padding; 16 B mod 128 B keeps
                                                     // the 8 lanes of each LDS.128 phase on distinct banks
constexpr uint32_t WARPS = SEQCDC_LW_WARPS;
constexpr uint32_t THREADS = 32 * WARPS;
constexpr uint32_t NBATCH = 8;                       // per-warp batch barriers (SEQCDC_LW_BATCH)
constexpr uint32_t SMEM_LANES = THREADS * STRIDE;
constexpr uint32_t SMEM = SMEM_LANES + (SEQCDC_LW_BATCH ? WARPS * NBATCH * 8 : 0);

static_assert(SMEM <= 48 * 1024, "static shared memory");
constexpr uint32_t GRP = SEQCDC_LW_GROUP;             // pairs per step
constexpr uint32_t GMASK = GRP - 1;
static_assert(!SEQCDC_LW_PAIR || (SEQCDC_LW_LAZY && !SEQCDC_LW_BATCH && !SEQCDC_LW_BULK && !SEQCDC_LW_ONEFILL), "pair fills need the lazy per-lane form");
static_assert(GRP == 16 || (GRP == 32 && SEQCDC_LW_PACKED), "group of 16 or (packed) 32 pairs");
static_assert(SEQCDC_LW_PF % GRP == 0 && SEQCDC_LW_PF < (int)LINE, "prefetch point inside a line");

enum { PH_SPEC = 0, PH_EXT = 1, PH_TAIL = 2, PH_DONE = 3 };
#ifdef SEQCDC_TIMELINE
__device__ unsigned long long g_lw_stats[4];   // warp steps, groups scanned, fills issued
#endif

#ifdef SEQCDC_TIMELINE
// per segment: globaltimer at start / end of the speculative part / end, and
// (speculative cuts << 32 | extension cuts)  (tools/lane_timeline.py)
__device__ __forceinline__ void tl_lane(uint32_t s, int k, uint64_t v = 0)
{
    if (g_tl && s < g_tl_cap) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_tl[4 * s + k] = k == 3 ? v : t;
    }
}
#define TL_LANE(s, k, v) tl_lane((s), (k), (v))
#else
#define TL_LANE(s, k, v)
#endif
constexpr uint32_t NONE = 0xffffffffu;

// ------------------------------------------------------------------ PTX
__device__ __forceinline__ uint4 lds128(uint32_t addr)
{
    uint4 v;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}

// ------------------------------------------------------------------ the lane's byte source
// Two slots of one LINE each; line l lives in slot l & 1, so the slots hold
// consecutive lines and a byte's shared address is base + (x mod 2 LINE).  A
// fill is 16-byte cp.async copies whose completion arrives on the slot's own
// mbarrier (cp.async.mbarrier.arrive); a lane polls it with a non-blocking
// test_wait (a per-thread instruction), so a warp step never waits for memory:
// lanes whose line has not landed simply do not scan in that step.
struct Src {
    uint64_t rb;         // absolute address of relative position 0 (LINE-aligned)
    uint32_t lo_rel;     // first byte of the job (relative)
    uint32_t end_rel;    // end of the loadable data (relative, clamped)
    uint32_t sb;         // shared address of this lane's region
    uint32_t tag0, tag1; // line held (or being filled) by each slot (NONE: none)
    uint32_t pend;       // bit k: slot k's fill not yet seen complete
    uint32_t par;        // bit k: parity slot k's barrier completes next
    uint32_t bsel;       // (SEQCDC_LW_BATCH) bits 4k..4k+3: slot k's batch barrier (3 bits) and phase parity
    uint32_t wb;         // (SEQCDC_LW_BATCH) shared address of this warp's batch barriers
};

__device__ __forceinline__ uint32_t mb_of(const Src &s, uint32_t k) { return s.sb + 2 * LINE + 8 * k; }

__device__ __forceinline__ void mb_init(uint32_t mb)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
}

__device__ __forceinline__ void mb_inval(uint32_t mb)
{
    asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(mb) : "memory");
}

__device__ __forceinline__ bool mb_test(uint32_t mb, uint32_t parity)
{
    uint32_t ok;
    asm volatile("{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(ok) : "r"(mb), "r"(parity) : "memory");
    return ok != 0;
}

// Start filling line `ln` into its slot (whose earlier fill is complete).
__device__ __forceinline__ void fill(Src &s, uint32_t ln)
{
    const uint32_t k = ln & 1u;
    const uint32_t dst = s.sb + k * LINE, mb = mb_of(s, k);
    const uint32_t x0 = ln << LSH;
#ifdef SEQCDC_TIMELINE
    atomicAdd(&g_lw_stats[2], 1ull);
#endif
    if (x0 >= s.lo_rel && x0 + LINE <= s.end_rel) {
        const uint64_t src = s.rb + x0;
#if SEQCDC_LW_BULK
        // one bulk copy (TMA) per line: one 128-B L2 request instead of eight 16-B ones
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(LINE) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(dst), "l"(src), "r"(LINE), "r"(mb) : "memory");
#else
#pragma unroll
        for (uint32_t i = 0; i < LINE; i += 16) cp_async16(dst + i, src + i);
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(mb) : "memory");
#endif
    } else {
        // a line at the edge of the data: copy the bytes that exist, one by one
#pragma unroll 1
        for (uint32_t i = 0; i < LINE; i++) {
            const uint32_t x = x0 + i;
            if (x >= s.lo_rel && x < s.end_rel) sts8(dst + i, *(const volatile uint8_t *)(s.rb + x));
        }
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(mb) : "memory");
    }
    if (k) s.tag1 = ln; else s.tag0 = ln;
    s.pend |= 1u << k;
}

// Poll the slots with a fill in flight (one non-blocking barrier test each).
__device__ __forceinline__ void poll(Src &s)
{
#pragma unroll
    for (uint32_t k = 0; k < 2; k++)
        if (((s.pend >> k) & 1u) && mb_test(mb_of(s, k), (s.par >> k) & 1u)) {
            s.pend &= ~(1u << k);
            s.par ^= 1u << k;
        }
}

__device__ __forceinline__ bool check(Src &s, uint32_t k);

__device__ __forceinline__ void drain(Src &s)
{
#if SEQCDC_LW_PAIR
#pragma unroll 1
    while (s.pend & 3u) {
        check(s, 0);
        check(s, 1);
    }
#else
#pragma unroll 1
    while (s.pend) poll(s);
#endif
}

__device__ __forceinline__ bool has(const Src &s, uint32_t ln) { return ((ln & 1u) ? s.tag1 : s.tag0) == ln; }

// Is line ln resident and complete?
__device__ __forceinline__ bool ready(const Src &s, uint32_t ln)
{
    return has(s, ln) && !((s.pend >> (ln & 1u)) & 1u);
}

// Start filling line ln unless its slot's earlier fill is still in flight.
__device__ __forceinline__ void request(Src &s, uint32_t ln)
{
    if (!((s.pend >> (ln & 1u)) & 1u)) fill(s, ln);
}

// Lazy form: a slot's barrier is tested only when its line is needed (every
// mbarrier test is a per-thread operation of the SM's sync unit, which the
// cp.async completions also use; testing each pending slot every step costs
// more than the scan).  A pending slot is never refilled before it is seen
// complete.
__device__ __forceinline__ bool check(Src &s, uint32_t k)
{
    if (!((s.pend >> k) & 1u)) return true;
#if SEQCDC_LW_PAIR
    // pend bit 2+k: slot k was filled together with the other slot and its
    // completion arrives on the other slot's barrier (fill2)
    const uint32_t j = ((s.pend >> (2 + k)) & 1u) ? k ^ 1u : k;
    if (!mb_test(mb_of(s, j), (s.par >> j) & 1u)) return false;
    const uint32_t o = j ^ 1u;
    uint32_t clr = 1u << j;
    if ((s.pend >> (2 + o)) & 1u) clr |= (1u << o) | (4u << o);   // the pair's other line landed too
    s.pend &= ~clr;
    s.par ^= 1u << j;
#else
    if (!mb_test(mb_of(s, k), (s.par >> k) & 1u)) return false;
    s.pend &= ~(1u << k);
    s.par ^= 1u << k;
#endif
    return true;
}

#if SEQCDC_LW_PAIR
// Fill lines ln and ln + 1 (both slots, both complete, both wholly inside the
// data) with ONE barrier arrival: the arrive of a per-lane barrier is a
// uniform-register instruction the compiler loops over the filling lanes, so
// a dependent miss (chunk start, skip landing) fetches the line after it in
// the same fill instead of a second fill one prefetch later.
__device__ __forceinline__ void fill2(Src &s, uint32_t ln)
{
    const uint32_t k = ln & 1u;
    const uint32_t d0 = s.sb + k * LINE, d1 = s.sb + (k ^ 1u) * LINE, mb = mb_of(s, k);
    const uint64_t src = s.rb + ((uint64_t)ln << LSH);
#ifdef SEQCDC_TIMELINE
    atomicAdd(&g_lw_stats[2], 1ull);
#endif
#pragma unroll
    for (uint32_t i = 0; i < LINE; i += 16) cp_async16(d0 + i, src + i);
#pragma unroll
    for (uint32_t i = 0; i < LINE; i += 16) cp_async16(d1 + i, src + LINE + i);
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(mb) : "memory");
    if (k) { s.tag1 = ln; s.tag0 = ln + 1; } else { s.tag0 = ln; s.tag1 = ln + 1; }
    s.pend |= 3u | (4u << (k ^ 1u));
}

// A missing line: with its successor when that one is absent too and both
// slots are free, else alone (the line at the edge of the data: fill()).
__device__ __forceinline__ void request_pair(Src &s, uint32_t ln)
{
    const uint32_t k = ln & 1u;
    if (!check(s, k)) return;
    const uint32_t x0 = ln << LSH;
    if (!has(s, ln + 1) && x0 >= s.lo_rel && x0 + 2 * LINE <= s.end_rel && check(s, k ^ 1u))
        fill2(s, ln);
    else
        fill(s, ln);
}
#endif

__device__ __forceinline__ bool ready_lazy(Src &s, uint32_t ln) { return has(s, ln) && check(s, ln & 1u); }

__device__ __forceinline__ void request_lazy(Src &s, uint32_t ln)
{
    if (check(s, ln & 1u)) fill(s, ln);
}

// Batch form (SEQCDC_LW_BATCH): the lanes that fill in one warp step all arrive
// on the same per-warp barrier (a warp-uniform address: one arrive instruction
// instead of a loop over the filling lanes' own barriers); a slot remembers
// its batch barrier and phase.  A batch barrier is re-armed only once its
// previous phase completed, so a recorded phase can never be confused.
__device__ __forceinline__ bool check_b(Src &s, uint32_t k)
{
    if (!((s.pend >> k) & 1u)) return true;
    const uint32_t bs = (s.bsel >> (4 * k)) & 0xfu;
    if (!mb_test(s.wb + 8 * (bs & 7u), bs >> 3)) return false;
    s.pend &= ~(1u << k);
    return true;
}

__device__ __forceinline__ void fill_b(Src &s, uint32_t ln, uint32_t mb, uint32_t kb, uint32_t par)
{
    const uint32_t k = ln & 1u;
    const uint32_t dst = s.sb + k * LINE;
    const uint32_t x0 = ln << LSH;
    if (x0 >= s.lo_rel && x0 + LINE <= s.end_rel) {
        const uint64_t src = s.rb + x0;
#pragma unroll
        for (uint32_t i = 0; i < LINE; i += 16) cp_async16(dst + i, src + i);
        asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];" ::"r"(mb) : "memory");   // pending +1
        s.pend |= 1u << k;
        s.bsel = (s.bsel & ~(0xfu << (4 * k))) | ((kb | (par << 3)) << (4 * k));
    } else {
        // a line at the edge of the data: copied here, complete at once (only this lane reads it)
#pragma unroll 1
        for (uint32_t i = 0; i < LINE; i++) {
            const uint32_t x = x0 + i;
            if (x >= s.lo_rel && x < s.end_rel) sts8(dst + i, *(const volatile uint8_t *)(s.rb + x));
        }
    }
    if (k) s.tag1 = ln; else s.tag0 = ln;
}

__device__ __forceinline__ uint32_t slot_addr(const Src &s, uint32_t x) { return s.sb + (x & (2 * LINE - 1)); }

// ------------------------------------------------------------------ one lane's chain state
struct Chain {
    uint32_t base, q, lim2, limit, need, carry, la;   // chunk start, group, limits, counters
    uint32_t ph;
    uint32_t hi_rel, stop_rel, ext_end;
    uint64_t off;                                     // relative position -> offset into `in`
    uint64_t *list;                                   // L_s, X_s or the tail list (by phase)
    uint32_t n, cap;                                  // entries in `list`, its capacity
    uint32_t nL;                                      // final count of L_s
    // extension: segment owning the current cut, its list and a cursor into it
    uint32_t t, j;
    bool fresh;                                       // cursor not yet set up for segment t
    uint64_t t_next, t_lo, t_Loff, t_word, cand;
};

// Set up the scan of the chunk starting at `base` (relative); false when the
// chunk is decided without examining any pair (cut = limit).
__device__ __forceinline__ bool chunk_begin(Chain &c, const Src &s, const DevParams &p, uint32_t base)
{
    c.base = base;
    c.limit = base + p.mx < s.end_rel ? base + p.mx : s.end_rel;     // P:266 / stream end (c9)
    c.lim2 = c.limit - 2;
    const uint32_t a = base + p.mnL;
    if (c.limit - base < 2 || a > c.lim2) return false;
    c.need = p.T;
    c.carry = 0;
    c.q = a & ~GMASK;
    c.la = a & GMASK;
#if SEQCDC_LW_L2PF
    {   // the next chunk's scan most likely starts a little past a + min - L (its
        // cut comes soon after this anchor): warm those lines in L2 now, so the
        // dependent fill at the next anchor is an L2 hit (a guess; costs no slot)
#pragma unroll
        for (int k = 0; k < SEQCDC_LW_L2PF; k++) {
            const uint32_t x = a + p.mnL + SEQCDC_LW_L2PF_OFF + k * LINE;
            if (x + LINE <= s.end_rel)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(s.rb + x));
        }
    }
#endif
    return true;
}

// Scan the 16-pair group at c.q (resident).  Returns the cut, or NONE when the
// chunk continues (skip or next group; c updated).
template <int MODE, bool M4>
__device__ __forceinline__ uint32_t scan_group(Chain &c, const Src &s, const DevParams &p)
{
    constexpr uint32_t XM = (MODE & 2) ? H : 0u;                      // signed reading: flip bit 7
    const uint32_t q = c.q;
    const uint4 v = lds128(slot_addr(s, q));
    const uint32_t x4 = (q + 16 <= c.lim2 + 1) ? lds32(slot_addr(s, q + 16)) : 0u;
    uint32_t xw[5] = {v.x ^ XM, v.y ^ XM, v.z ^ XM, v.w ^ XM, x4 ^ XM};
    uint32_t F[4], O[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const uint32_t y = __funnelshift_r(xw[k], xw[k + 1], 8);        // y_b = byte q+4k+b+1
        uint32_t lt, gt;
        lt_gt_flags(xw[k], y, lt, gt);
        // pairs below the anchor (first group of a chunk / after a skip) are not examined
        const uint32_t sh = (uint32_t)max((int)(8u * c.la) - 32 * k, 0);
        uint32_t m;
        asm("shl.b32 %0, %1, %2;" : "=r"(m) : "r"(H), "r"(sh));        // shift >= 32 -> 0
        F[k] = ((MODE & 1) == 0 ? lt : gt) & m;
        O[k] = ((MODE & 1) == 0 ? gt : lt) & m;
    }
    uint32_t R[4];
    uint32_t prev = c.carry;
#pragma unroll
    for (int k = 0; k < 4; k++) {
        if (M4) {
            R[k] = F[k] & __funnelshift_l(prev, F[k], 8) & __funnelshift_l(prev, F[k], 16) &
                   __funnelshift_l(prev, F[k], 24);
        } else {
            uint32_t r = F[k];
            if (p.M > 1) r &= __funnelshift_l(prev, F[k], 8);
            if (p.M > 2) r &= __funnelshift_l(prev, F[k], 16);
            if (p.M > 3) r &= __funnelshift_l(prev, F[k], 24);
            R[k] = r;
        }
        prev = F[k];
    }
    const uint32_t c0 = __popc(O[0]), c1 = __popc(O[1]), c2 = __popc(O[2]), c3 = __popc(O[3]);
    const uint32_t ctot = c0 + c1 + c2 + c3;
    if (((R[0] | R[1]) | (R[2] | R[3])) == 0 && ctot < c.need) {     // nothing decided in this group
        c.need -= ctot;
        c.carry = F[3];
        c.la = 0;
        c.q = q + 16;
        return q + 16 > c.lim2 ? c.limit : NONE;                      // every pair up to the limit examined
    }
    // first run end (pair index in the group)
    uint32_t r = NONE;
#pragma unroll
    for (int k = 3; k >= 0; k--)
        if (R[k]) r = 4u * k + ((uint32_t)(__ffs(R[k]) - 1) >> 3);
    // the need-th opposing pair
    uint32_t d = NONE;
    if (ctot >= c.need) {
        const uint32_t e1 = c0, e2 = c0 + c1, e3 = c0 + c1 + c2;
        const uint32_t k = c.need <= e1 ? 0u : (c.need <= e2 ? 1u : (c.need <= e3 ? 2u : 3u));
        const uint32_t ex = k == 0 ? 0u : (k == 1 ? e1 : (k == 2 ? e2 : e3));
        const uint32_t Ok = k == 0 ? O[0] : (k == 1 ? O[1] : (k == 2 ? O[2] : O[3]));
        const uint32_t pc = (Ok >> 7) * 0x01010101u;
        const uint32_t ge = ((pc | H) - (c.need - ex) * 0x01010101u) & 0x00808080u;
        d = 4u * k + 3u - __popc(ge);
    }
    if (r < d) {                                                      // the run completes first
        const uint32_t pr = q + r;
        return pr <= c.lim2 ? pr + 2 : c.limit;
    }
    const uint32_t pd = q + d;                                        // the need-th opposing pair: skip
    if (pd > c.lim2 || p.S >= c.lim2 - pd) return c.limit;           // lands past the limit (c8)
    const uint32_t a = pd + 1 + p.S;                                  // reading c3
    c.need = p.T;
    c.carry = 0;
    c.q = a & ~15u;
    c.la = a & 15u;
    return NONE;
}

// ------------------------------------------------------------------ packed-mask form of the group scan
// The same decision as scan_group, on 16-bit masks in pair order (bit i = pair
// q+i): fewer instructions per step, and every lane of a warp runs the same
// straight-line code.
//
// nib: the flag bits (bit 7 of each byte) of one word -> bits 0..3 of
// the result in byte order; bits 4..7 are zero, bits >= 8 garbage.  With
// w & H = sum b_k 2^(8k+7) and c = sum_j 2^(25-7j), the product's terms sit at
// 2^(32 + 8k - 7j): k = j lands on high-word bit k, k > j at high bits >= 8, k < j
// on six distinct low-word bits (no carries).
__device__ __forceinline__ uint32_t nib(uint32_t w) { return __umulhi(w & H, 0x02040810u); }

__device__ __forceinline__ uint32_t pack16(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3)
{
    const uint32_t a = __byte_perm(nib(w0), nib(w1), 0x0040);     // byte0 = n0, byte1 = n1
    const uint32_t b = __byte_perm(nib(w2), nib(w3), 0x4000);     // byte2 = n2, byte3 = n3
    uint32_t w = __byte_perm(a, b, 0x7610);
    w |= w >> 4;                                                   // byte0 = n0|n1<<4, byte2 = n2|n3<<4
    return __byte_perm(w, 0u, 0x4420);
}

// Position of the n-th (1-based) set bit of a 16-bit mask holding >= n bits.
__device__ __forceinline__ uint32_t select16(uint32_t o, uint32_t n)
{
    uint32_t pos = 0, c;
    c = __popc(o & 0xffu);
    if (n > c) { n -= c; o >>= 8; pos += 8; }
    c = __popc(o & 0xfu);
    if (n > c) { n -= c; o >>= 4; pos += 4; }
    c = __popc(o & 0x3u);
    if (n > c) { n -= c; o >>= 2; pos += 2; }
    if (n > (o & 1u)) pos += 1;
    return pos;
}

__device__ __forceinline__ uint32_t select32(uint32_t o, uint32_t n)
{
    const uint32_t c = __popc(o & 0xffffu);
    return n > c ? 16u + select16(o >> 16, n - c) : select16(o & 0xffffu, n);
}

template <int MODE, bool M4>
__device__ __forceinline__ uint32_t scan_group_p(Chain &c, const Src &s, const DevParams &p)
{
    constexpr uint32_t XM = (MODE & 2) ? H : 0u;                      // signed reading: flip bit 7
    constexpr int NW = GRP / 4;                                       // words of 4 pairs
    const uint32_t q = c.q;
    uint32_t xw[NW + 1];
#pragma unroll
    for (int k = 0; k < NW; k += 4) {
        const uint4 v = lds128(slot_addr(s, q + 4 * k));
        xw[k] = v.x ^ XM; xw[k + 1] = v.y ^ XM; xw[k + 2] = v.z ^ XM; xw[k + 3] = v.w ^ XM;
    }
    xw[NW] = ((q + GRP <= c.lim2 + 1) ? lds32(slot_addr(s, q + GRP)) : 0u) ^ XM;
    uint32_t lt[NW], gt[NW];
#pragma unroll
    for (int k = 0; k < NW; k++) lt_gt_flags(xw[k], __funnelshift_r(xw[k], xw[k + 1], 8), lt[k], gt[k]);
    uint32_t LT = pack16(lt[0], lt[1], lt[2], lt[3]), GT = pack16(gt[0], gt[1], gt[2], gt[3]);
    if (GRP == 32) {
        LT |= pack16(lt[NW - 4], lt[NW - 3], lt[NW - 2], lt[NW - 1]) << 16;
        GT |= pack16(gt[NW - 4], gt[NW - 3], gt[NW - 2], gt[NW - 1]) << 16;
    }
    const uint32_t m = (GRP == 32 ? FULL : 0xffffu) << c.la;          // pairs below the anchor: not examined
    const uint32_t F = ((MODE & 1) == 0 ? LT : GT) & m;               // favourable pairs
    const uint32_t O = ((MODE & 1) == 0 ? GT : LT) & m;               // opposing pairs
    // bit i of R: pairs i, i-1, ..., i-M+1 all favourable -- a run ends at pair q+i;
    // the pairs below bit 0 are the previous group's (c.carry, zero at an anchor)
    uint32_t R = F;
    if (M4 || p.M > 1) R &= __funnelshift_l(c.carry, F, 1);
    if (M4 || p.M > 2) R &= __funnelshift_l(c.carry, F, 2);
    if (M4 || p.M > 3) R &= __funnelshift_l(c.carry, F, 3);
    const uint32_t ctot = __popc(O);
    if (R == 0 && ctot < c.need) {                                    // nothing decided in this group
        c.need -= ctot;
        c.carry = GRP == 32 ? F : F << 16;
        c.la = 0;
        c.q = q + GRP;
        return q + GRP > c.lim2 ? c.limit : NONE;                     // every pair up to the limit examined
    }
    const uint32_t r = R ? (uint32_t)__ffs(R) - 1u : GRP;
    if (r < GRP && (uint32_t)__popc(O & ((1u << r) - 1u)) < c.need) {   // the run completes first
        const uint32_t pr = q + r;
        return pr <= c.lim2 ? pr + 2 : c.limit;
    }
    const uint32_t pd = q + (GRP == 32 ? select32(O, c.need) : select16(O, c.need));   // skip
    if (pd > c.lim2 || p.S >= c.lim2 - pd) return c.limit;           // lands past the limit (c8)
    const uint32_t a = pd + 1 + p.S;                                  // reading c3
    c.need = p.T;
    c.carry = 0;
    c.q = a & ~GMASK;
    c.la = a & GMASK;
    return NONE;
}

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t *p)
{
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Publish a task for the warps: segment s's extension, with `tail` the range
// call's tail, with `spec` the rest of its speculative part (then its
// extension / tail); its list writes are ordered before the release store.
constexpr uint32_t TASK_TAIL = 0x80000000u, TASK_SPEC = 0x40000000u, TASK_SEG = 0x3fffffffu;
__device__ __forceinline__ void hand_off(const Work &w, uint32_t s, uint32_t kind)
{
    const uint32_t idx = atomicAdd(w.ctrl + C_HAND, 1u);
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(w.hand + idx), "r"((s + 1) | kind) : "memory");
}

// A cut of lane s's chain at relative position `cut`: record it where the
// phase says (speculative list, extension list with the merge check, or the
// range tail) and decide whether the chain goes on.  Returns false when the
// lane's work is done (its results are written).
__device__ __forceinline__ bool on_cut(const Work &w, Chain &c, const Src &src, const Seg &g, uint32_t s,
                                       uint64_t stop_abs, uint32_t cut, bool late_ext)
{
    const uint64_t cabs = c.off + cut;
    if (c.ph == PH_SPEC && cut >= c.hi_rel) {          // first cut past the segment: the extension starts
        TL_LANE(s, 1, 0);
        st_release_u64(w.Lcnt + s, (uint64_t)c.n | DONE_BIT);
        if (w.lw_late || w.lw_late_ext) atomicAdd(w.ctrl + C_SPECDONE, 1u);
        c.nL = c.n;
        c.ph = PH_EXT;
        c.list = w.X + g.Xoff;
        c.cap = g.Xcap;
        c.n = 0;
        c.t = s;
        c.t_next = seg_start(w, g, s + 1);
        c.fresh = true;
    }
    if (c.ph == PH_SPEC) {
        c.list[c.n++] = cabs;
        if (cut < c.stop_rel) return true;
        // the stream's (range's) last chunk
        st_release_u64(w.Lcnt + s, (uint64_t)c.n | DONE_BIT);
        if (w.lw_late || w.lw_late_ext) atomicAdd(w.ctrl + C_SPECDONE, 1u);
        w.Xcnt[s] = 0;
        w.target[s] = TGT_END;
        w.midx[s] = -1;
        w.cont_cnt[s] = 0;
        if (!(w.single && w.tail_max)) {
            c.ph = PH_DONE;
            return false;
        }
        // range call: the chain continues past the overhang (the next rank's
        // merge) -- handed to a warp, which walks the ~100 chunks much faster
        hand_off(w, s, TASK_TAIL);
        c.ph = PH_DONE;
        return false;
    }
    // PH_EXT
    int32_t tgt = TGT_OVERFLOW;
    int64_t mi = -1;
    if (c.n < c.cap && cut <= c.ext_end) {             // else: extension budget exhausted (phase-locked data)
        c.list[c.n++] = cabs;
        if (cabs >= stop_abs) {
            tgt = TGT_END;
        } else {
            bool moved = c.fresh;
#pragma unroll 1
            while (cabs >= c.t_next) {                 // segments are uniform within a stream
                c.t++;
                c.t_next += w.G;
                moved = true;
            }
            if (moved) {
                c.fresh = false;
                c.t_lo = seg_start(w, g, c.t);
                c.t_Loff = w.single ? (uint64_t)c.t * w.capL1 : w.Loff[c.t];
                c.t_word = 0;
                c.j = 0;
                c.cand = ~0ull;
            }
            if (cabs == c.t_lo) {                      // the owning chain's implicit first cut
                tgt = (int32_t)c.t;
            } else {
                if (!(c.t_word & DONE_BIT)) {
                    c.t_word = ld_acquire_u64(w.Lcnt + c.t);
                    if ((c.t_word & DONE_BIT) && (c.t_word & CNT_MASK)) c.cand = __ldcg(w.L + c.t_Loff + c.j);
                }
                if (!(c.t_word & DONE_BIT) && !late_ext) return true;   // not decidable yet: walk on
                const uint32_t cnt = (uint32_t)(c.t_word & CNT_MASK);
#pragma unroll 1
                while ((c.t_word & DONE_BIT) && c.cand < cabs && c.j + 1 < cnt) {
                    c.j++;
                    c.cand = __ldcg(w.L + c.t_Loff + c.j);
                }
                if (!(c.t_word & DONE_BIT) || c.cand != cabs) {   // not a cut of the owning chain: walk on
                    // (late in the walk, a warp continues the extension at once: ~30x faster per chunk)
                    if (c.n < w.lw_ext_cap && !late_ext) return true;
                    w.Xcnt[s] = c.n;                    // a long extension: a warp continues it
                    hand_off(w, s, 0u);
                    c.ph = PH_DONE;
                    return false;
                }
                tgt = (int32_t)c.t;
                mi = (int64_t)c.j;
            }
        }
    }
    w.Xcnt[s] = c.n;
    w.target[s] = tgt;
    w.midx[s] = mi;
    w.cont_cnt[s] = 0;
    if (tgt == TGT_OVERFLOW) atomicOr(w.ctrl + C_OVF, 1u);
    c.ph = PH_DONE;
    TL_LANE(s, 2, 0);
    TL_LANE(s, 3, ((uint64_t)c.nL << 32) | c.n);
    return false;
}


}  // namespace lw

// A task handed off by a lane, served by a whole warp with the warp walker
// (dense cp.async ring, seqcdc_device.cuh): continue segment s's extension
// from its last cut until a cut coincides with the chain owning its region (as
// walk_segment's extension does), walk a range call's tail (up to tail_max
// cuts past the overhang, only chunks wholly inside the buffer), or finish the
// speculative part of a late lane's segment and then its extension / tail.

#ifndef SEQCDC_LH_SPARSE
#define SEQCDC_LH_SPARSE 0     // k_lhand's warps read sparsely (512-B block cache + next-anchor prefetch)
#endif
#if SEQCDC_LH_SPARSE
using LWalker = SWalker;
#else
using LWalker = DWalker;
#endif
constexpr uint32_t LH_SMEM = LWalker::BYTES > RING ? LWalker::BYTES : RING;

#ifndef SEQCDC_LH_PF
#define SEQCDC_LH_PF 0         // lines of the next chunk's likely anchor region warmed in L2 per chunk (warps)
#endif
// A lone chain walked by a warp waits on memory once per chunk: the next
// chunk's scan starts at its cut + min - L, and the cut most often
// comes soon after this chunk's own anchor.  Warm that region in L2 while this
// chunk is resolved (a guess; one prefetch per lane, no ring slot).
__device__ __forceinline__ void lh_prefetch(const Work &w, uint64_t base_abs, uint64_t end_abs, int lane)
{
#if SEQCDC_LH_PF
    const uint64_t x = base_abs + w.p.mn + w.p.mnL + 128u * (uint32_t)lane;
    if (lane < SEQCDC_LH_PF && x < end_abs) asm volatile("prefetch.global.L2 [%0];" ::"l"(w.in + x));
#endif
}

// The range call's tail from segment s's last speculative cut (the overhang).
template <int MODE, int MSPEC>
__device__ void serve_tail(const Work &w, LWalker &wk, uint32_t s, const Seg &g, int lane)
{
    const uint64_t abase = (uint64_t)(uintptr_t)w.in;
    const uint64_t nl = __ldcg(w.Lcnt + s) & CNT_MASK;
    const uint64_t from = __ldcg(w.L + g.Loff + nl - 1);              // the overhang
    uint32_t base = walker_begin(wk, abase + from, abase + g.E);
    const uint64_t off = wk.rb - abase;
    ListBuf tb{0, 0};
    if (base < wk.end_rel) {
        lb_push(tb, from + w.out_add, w.tail, lane);
#pragma unroll 1
        while (tb.n < w.tail_max && base + w.p.mx <= wk.end_rel) {
            lh_prefetch(w, off + base, g.E, lane);
            const uint32_t c = resolve<MODE, MSPEC>(wk, w.p, base, lane);
            SEQCDC_ASSERT_CUT(base, c, w.p, wk.end_rel);
            lb_push(tb, off + c + w.out_add, w.tail, lane);
            base = c;
        }
    }
    lb_flush(tb, w.tail, lane);
    if (lane == 0) *w.tail_n = tb.n;
}

// The rest of a late lane's speculative part (its list holds >= 1 cut, count
// published with HANDED_BIT): walk from the last cut, append the cuts inside
// the segment, publish the list complete.  Returns true when the chain reached
// the stream's (range's) end inside the segment -- then its bookkeeping is done
// here, except a range call's tail.  Never waits on anything.
template <int MODE, int MSPEC>
__device__ bool serve_spec(const Work &w, LWalker &wk, uint32_t s, const Seg &g, int lane)
{
    const uint64_t abase = (uint64_t)(uintptr_t)w.in;
    uint64_t *Ls = w.L + g.Loff;
    const uint32_t n0 = (uint32_t)(__ldcg(w.Lcnt + s) & (HANDED_BIT - 1));
    const uint64_t from = __ldcg(Ls + n0 - 1);
    ListBuf lb;
    lb.n = n0;
    lb.v = lane < (int)(n0 & 31) ? __ldcg(Ls + (n0 & ~31u) + lane) : 0;   // the open batch
    uint32_t base = walker_begin(wk, abase + from, abase + g.E);
    const uint64_t off = wk.rb - abase;
    const uint64_t hi_abs = g.last ? ~0ull : g.hi;                    // (as the lane's hi_rel / stop_rel)
    const uint64_t stop_abs = w.single ? w.stop : g.E;
    bool end = false;
#pragma unroll 1
    for (;;) {
        lh_prefetch(w, off + base, g.E, lane);
        const uint32_t c = resolve<MODE, MSPEC>(wk, w.p, base, lane);
        SEQCDC_ASSERT_CUT(base, c, w.p, wk.end_rel);
        const uint64_t cut = off + c;
        if (cut >= hi_abs) break;                                     // the extension's first cut
        SEQCDC_ASSERT(lb.n < g.Lcap);
        lb_push(lb, cut, Ls, lane);
        if (cut >= stop_abs) {                                        // the stream's (range's) last chunk
            end = true;
            break;
        }
        base = c;
    }
    lb_flush(lb, Ls, lane);
    publish(w.Lcnt + s, lb.n, true, lane);
    if (end && lane == 0) {
        w.Xcnt[s] = 0;
        w.target[s] = TGT_END;
        w.midx[s] = -1;
        w.cont_cnt[s] = 0;
    }
    __syncwarp();
    return end;
}

template <int MODE, int MSPEC>
__device__ void lw_serve(const Work &w, LWalker &wk, uint32_t task, int lane)
{
    const uint32_t s = (task & lw::TASK_SEG) - 1;
    const uint64_t abase = (uint64_t)(uintptr_t)w.in;
    const Seg g = get_seg(w, s);
    if (task & lw::TASK_TAIL) {
        serve_tail<MODE, MSPEC>(w, wk, s, g, lane);
        return;
    }
    if (task & lw::TASK_SPEC) {
        uint32_t won = 0;
        if (lane == 0) won = atomicCAS(w.lclaim + s, 0u, 1u) == 0u;
        if (!__shfl_sync(FULL, won, 0)) return;                       // a waiting warp took it (below)
        if (serve_spec<MODE, MSPEC>(w, wk, s, g, lane)) {
            if (w.single && w.tail_max) serve_tail<MODE, MSPEC>(w, wk, s, g, lane);
            return;
        }
        if (lane == 0) w.Xcnt[s] = 0;                                 // the extension, from the last spec cut
        __syncwarp();
    }
    uint64_t *Xs = w.X + g.Xoff;
    const uint32_t n0 = __ldcg(w.Xcnt + s);
    // an extension handed off by a lane continues from its last cut; one after a
    // speculative part finished here (n0 = 0) starts at that part's last cut, so
    // its first cut -- the first past the segment -- is walked and checked again
    const uint64_t from = n0 ? __ldcg(Xs + n0 - 1) : __ldcg(w.L + g.Loff + ((__ldcg(w.Lcnt + s) & CNT_MASK) - 1));
    ListBuf xb;
    xb.n = n0;
    xb.v = lane < (int)(n0 & 31) ? __ldcg(Xs + (n0 & ~31u) + lane) : 0;   // the open batch
    uint32_t base = walker_begin(wk, abase + from, abase + g.E);
    uint64_t off = wk.rb - abase;
    const uint64_t stop_abs = w.single ? w.stop : g.E;
    const uint64_t ext_end = g.hi + (uint64_t)w.ext_segs * w.G;
    uint32_t t = g.first + (uint32_t)((from - g.S0) / w.G);
    uint64_t t_next = seg_start(w, g, t + 1);
    Cursor cur{-1, 0, 0, 0};
    uint64_t t_lo = 0, t_Loff = 0;
    int32_t tgt = TGT_OVERFLOW;
    int64_t mi = -1;
#pragma unroll 1
    for (;;) {
        lh_prefetch(w, off + base, g.E, lane);
        uint32_t c = resolve<MODE, MSPEC>(wk, w.p, base, lane);
        SEQCDC_ASSERT_CUT(base, c, w.p, wk.end_rel);
        const uint64_t cut = off + c;
        if (xb.n == g.Xcap || cut > ext_end) break;                     // budget exhausted: overflow
        lb_push(xb, cut, Xs, lane);
        if (cut >= stop_abs) {
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
            // served while lanes still walk: wait until the owning chain's list is
            // complete, so every cut is decided at once instead of being walked
            // past.  A lane never waits on a warp; a late lane's handed-off
            // speculative part is walked here if no warp has claimed it yet (a
            // speculative part never waits), so no warp waits on an unserved task.
#pragma unroll 1
            for (;;) {
                uint32_t act = 0;                                       // 0: complete, 1: wait, 2: walk it
                if (lane == 0) {
                    const uint64_t v = ld_acquire_u64(w.Lcnt + t);
                    act = (v & DONE_BIT) ? 0u : ((v & HANDED_BIT) && atomicCAS(w.lclaim + t, 0u, 1u) == 0u) ? 2u : 1u;
                }
                act = __shfl_sync(FULL, act, 0);
                if (act == 0) break;
                if (act == 1) {
                    __nanosleep(200);
                    continue;
                }
                const Seg gt = get_seg(w, t);
                if (serve_spec<MODE, MSPEC>(w, wk, t, gt, lane)) {
                    if (lane == 0 && w.single && w.tail_max) lw::hand_off(w, t, lw::TASK_TAIL);
                } else if (lane == 0) {
                    w.Xcnt[t] = 0;
                    lw::hand_off(w, t, 0u);                             // its extension: a new task
                }
                __syncwarp();
                c = walker_begin(wk, abase + cut, abase + g.E);         // back to this chain
                off = wk.rb - abase;
            }
            __syncwarp();
        }
        int64_t idx;
        if (check_cut(w, cur, t, t_lo, t_Loff, cut, idx, lane) == CK_MERGE) {
            tgt = (int32_t)t;
            mi = idx;
            break;
        }
        base = c;
    }
    lb_flush(xb, Xs, lane);
    if (lane == 0) {
        w.Xcnt[s] = xb.n;
        w.target[s] = tgt;
        w.midx[s] = mi;
        w.cont_cnt[s] = 0;
        if (tgt == TGT_OVERFLOW) atomicOr(w.ctrl + C_OVF, 1u);
    }
    __syncwarp();
}

// The per-lane walker kernel.  One segment per lane (grid = segments / THREADS).
template <int MODE, bool M4>
__global__ void __launch_bounds__(lw::THREADS) k_lwalk(Work w)
{
    using namespace lw;
    __shared__ __align__(128) uint8_t sm[SMEM];
    asm volatile("griddepcontrol.launch_dependents;");
    const int lane = threadIdx.x & 31;
    const uint32_t nseg = w.ctrl[C_BAD] ? 0u : nseg_total(w);
    const uint32_t s = blockIdx.x * THREADS + threadIdx.x;
    const uint64_t abase = (uint64_t)(uintptr_t)w.in;
    const DevParams p = w.p;

    Src src;
    {
        uint32_t sb = smem_u32(sm) + threadIdx.x * STRIDE;
        asm volatile("mov.b32 %0, %0;" : "+r"(sb));
        src.sb = sb;
    }
#if SEQCDC_LW_BATCH
    src.wb = smem_u32(sm) + SMEM_LANES + (threadIdx.x >> 5) * NBATCH * 8;
    if (lane < (int)NBATCH) mb_init(src.wb + 8 * lane);
    __syncwarp();
    src.bsel = 0;
    uint32_t wnext = 0, wpar = 0, wused = 0;          // warp-uniform: next batch barrier, phase parities, armed
#else
    mb_init(mb_of(src, 0));
    mb_init(mb_of(src, 1));
#endif
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    src.tag0 = src.tag1 = NONE;
    src.pend = src.par = 0;

    Chain c;
    c.ph = PH_DONE;
    Seg g;
    uint64_t stop_abs = 0;
    uint32_t pend = NONE;                             // a cut decided without examining any pair
    if (s < nseg) {
        g = get_seg(w, s);
        src.rb = (abase + g.lo) & ~(uint64_t)LMASK;
        src.lo_rel = (uint32_t)(abase + g.lo - src.rb);
        const uint64_t e = g.E > g.lo ? abase + g.E - src.rb : src.lo_rel;
        src.end_rel = e > REL_CLAMP ? REL_CLAMP : (uint32_t)e;
        c.off = src.rb - abase;
        c.hi_rel = g.last ? FULL : src.lo_rel + (uint32_t)(g.hi - g.lo);
        stop_abs = w.single ? w.stop : g.E;
        c.stop_rel = stop_abs - c.off < (uint64_t)FULL ? (uint32_t)(stop_abs - c.off) : FULL;
        c.ext_end = c.hi_rel + (uint32_t)(w.ext_segs * w.G);
        c.list = w.L + g.Loff;
        c.cap = g.Lcap;
        c.n = 0;
        TL_LANE(s, 0, 0);
        if (src.lo_rel < src.end_rel) {
            c.ph = PH_SPEC;
            if (!chunk_begin(c, src, p, src.lo_rel)) pend = c.limit;
        } else {                                      // an empty segment (empty stream)
            st_release_u64(w.Lcnt + s, DONE_BIT);
            w.Xcnt[s] = 0;
            w.target[s] = TGT_END;
            w.midx[s] = -1;
            w.cont_cnt[s] = 0;
            if (w.single && w.tail_max && g.last) *w.tail_n = 0;
        }
    }

#if SEQCDC_LW_LAZY
#define REQUEST(S, L) request_lazy((S), (L))
#else
#define REQUEST(S, L) request((S), (L))
#endif
    // One step of every lane per iteration, in lockstep: examine one group if
    // its lines are complete, handle a cut, keep the next lines on their way.
    uint32_t step = 0;
    bool late = false;                                // most lanes are past their speculative part:
    bool late_ext = false;                            // hand the rest of the segment / the extension to a warp
#pragma unroll 1
    while (__any_sync(FULL, c.ph != PH_DONE)) {
        step++;
        if ((w.lw_late || w.lw_late_ext) && !(late && late_ext) && (step & 31) == 0) {
            uint32_t v = 0;
            if (lane == 0) v = *(volatile const uint32_t *)(w.ctrl + C_SPECDONE);
            v = __shfl_sync(FULL, v, 0);
            late = w.lw_late && v >= w.lw_late;
            late_ext = w.lw_late_ext && v >= w.lw_late_ext;
        }
        uint32_t want = NONE;                           // (batch form) the line this lane asks for
        if (c.ph != PH_DONE) {
#if !SEQCDC_LW_LAZY && !SEQCDC_LW_BATCH
            if (src.pend) poll(src);
#endif
            uint32_t cut = pend;
            pend = NONE;
            if (cut == NONE) {
                const uint32_t l0 = c.q >> LSH;
                // byte q+GRP lies in the next line only for the line's last group
                const bool two = (c.q & LMASK) == LINE - GRP && c.q + GRP <= c.lim2 + 1;
#if SEQCDC_LW_BATCH
                const bool ok = has(src, l0) && check_b(src, l0 & 1u) &&
                                (!two || (has(src, l0 + 1) && check_b(src, (l0 + 1) & 1u)));
#elif SEQCDC_LW_LAZY
                const bool ok = ready_lazy(src, l0) && (!two || ready_lazy(src, l0 + 1));
#else
                const bool ok = ready(src, l0) && (!two || ready(src, l0 + 1));
#endif
                if (ok) {
#if SEQCDC_LW_PACKED
                    cut = scan_group_p<MODE, M4>(c, src, p);
#else
                    cut = scan_group<MODE, M4>(c, src, p);
#endif
#ifdef SEQCDC_TIMELINE
                    atomicAdd(&g_lw_stats[1], 1ull);
#endif
                }
            }
            if (cut != NONE) {
                SEQCDC_ASSERT_CUT(c.base, cut, p, src.end_rel);
                if (c.ph == PH_SPEC && cut < c.hi_rel && cut < c.stop_rel) {   // the common case
                    SEQCDC_ASSERT(c.n < c.cap);
                    c.list[c.n++] = c.off + cut;
                    if (late) {
                        // a late lane: a warp walks the rest of the segment ~30x faster
                        // (lw_serve); the count is published without DONE_BIT
                        st_release_u64(w.Lcnt + s, (uint64_t)c.n | HANDED_BIT);
                        hand_off(w, s, TASK_SPEC);
                        c.ph = PH_DONE;
                    } else if (!chunk_begin(c, src, p, cut)) pend = c.limit;
                } else if (on_cut(w, c, src, g, s, stop_abs, cut, late_ext)) {
                    if (!chunk_begin(c, src, p, cut)) pend = c.limit;
                }
            }
            if (c.ph != PH_DONE && pend == NONE) {          // the lines the next groups need, on their way
                const uint32_t l0 = c.q >> LSH;
#if SEQCDC_LW_BATCH
                if (!has(src, l0)) want = l0;
                else if ((c.q & LMASK) >= SEQCDC_LW_PF && !has(src, l0 + 1) && ((l0 + 1) << LSH) < src.end_rel)
                    want = l0 + 1;
                if (want != NONE && !check_b(src, want & 1u)) want = NONE;   // its slot's fill still in flight
#elif SEQCDC_LW_ONEFILL
                // one fill site: the current line if missing, else the next once the scan is past PF
                want = !has(src, l0) ? l0
                       : ((c.q & LMASK) >= SEQCDC_LW_PF && !has(src, l0 + 1) &&
                          ((l0 + 1) << LSH) < src.end_rel) ? l0 + 1 : NONE;
                if (want != NONE) REQUEST(src, want);
#else
                if (!has(src, l0)) {
#if SEQCDC_LW_PAIR
                    request_pair(src, l0);
#else
                    REQUEST(src, l0);
#endif
                } else if ((c.q & LMASK) >= SEQCDC_LW_PF && !has(src, l0 + 1) && ((l0 + 1) << LSH) < src.end_rel) {
                    REQUEST(src, l0 + 1);
                }
#endif
            }
        }
#if SEQCDC_LW_BATCH
        // this step's fills: one batch barrier for the whole warp (re-armed only
        // once its previous phase completed; if not, the lanes ask again next step)
        if (__ballot_sync(FULL, want != NONE)) {
            const uint32_t kb = wnext, mb = src.wb + 8 * kb, P = (wpar >> kb) & 1u;
            uint32_t free = 1;
            if ((wused >> kb) & 1u) {
                if (lane == 0) free = mb_test(mb, P ^ 1u) ? 1u : 0u;
                free = __shfl_sync(FULL, free, 0);
            }
            if (free) {
                if (want != NONE) fill_b(src, want, mb, kb, P);
                __syncwarp();                           // every async arrive counted before the phase can end
                if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(mb) : "memory");
                wused |= 1u << kb;
                wpar ^= 1u << kb;
                wnext = (kb + 1) & (NBATCH - 1);
            }
        }
#endif
    }
#undef REQUEST
#if SEQCDC_LW_BATCH
    // every armed batch complete before the shared memory is released
    if (lane < (int)NBATCH && ((wused >> lane) & 1u)) {
        const uint32_t mb = src.wb + 8 * lane, P = ((wpar >> lane) & 1u) ^ 1u;
#pragma unroll 1
        while (!mb_test(mb, P)) {
        }
    }
    __syncwarp();
    if (lane < (int)NBATCH) mb_inval(src.wb + 8 * lane);
#else
    drain(src);
    mb_inval(mb_of(src, 0));
    mb_inval(mb_of(src, 1));
#endif
    {   // this warp's lanes are done and their tasks published: count them (k_lhand waits for all)
        const uint32_t mine = __popc(__ballot_sync(FULL, s < nseg));
        if (lane == 0 && mine) {
            __threadfence();
            atomicAdd(w.ctrl + C_FIN, mine);
        }
    }
#ifdef SEQCDC_TIMELINE
    if (lane == 0) atomicAdd(&g_lw_stats[0], (unsigned long long)step);
#endif
}

// The handed-off tasks: persistent one-warp CTAs, launched behind k_lwalk with
// programmatic dependent launch, so they become resident only after every lane
// CTA is, and start serving tasks as soon as lanes publish them (the lane
// walk's tail and the hand-off work overlap).  A task index is claimed first,
// then waited for; a warp leaves when every lane is done (k_lwalk's C_FIN) and
// its claimed index holds no task.  The last warp to leave continues any
// extension on the valid path that ran out of budget (single stream; as k_walk
// does).
template <int MODE, int MSPEC>
__global__ void __launch_bounds__(32, SEQCDC_MIN_BLOCKS) k_lhand(Work w)
{
    __shared__ __align__(128) uint8_t ring[LH_SMEM];
    const int lane = threadIdx.x;
    const uint32_t nseg = w.ctrl[C_BAD] ? 0u : nseg_total(w);
    LWalker wk;
    walker_init(wk, ring, w.p, lane);
#pragma unroll 1
    for (;;) {
        uint32_t j = 0;
        if (lane == 0) j = atomicAdd(w.ctrl + C_HNEXT, 1u);
        j = __shfl_sync(FULL, j, 0);
        if (j >= 2 * nseg + 8) break;                           // at most two tasks per segment
        uint32_t task = 0;
        if (lane == 0) {
#pragma unroll 1
            for (;;) {
                task = lw::ld_acquire_u32(w.hand + j);
                if (task) break;
                // every lane done and every published task served: nobody can publish
                // another (only a lane, or a warp serving a task, hands one off)
                bool quiet = lw::ld_acquire_u32(w.ctrl + C_FIN) == nseg;
                if (quiet) {                        // served first: equal counts then mean none in service
                    const uint32_t served = lw::ld_acquire_u32(w.ctrl + C_SERVED);
                    quiet = served == lw::ld_acquire_u32(w.ctrl + C_HAND);
                }
                if (quiet) {
                    task = lw::ld_acquire_u32(w.hand + j);
                    if (!task) task = FULL;
                    break;
                }
                __nanosleep(400);
            }
        }
        task = __shfl_sync(FULL, task, 0);
        __syncwarp();
        if (task == FULL) break;
        lw_serve<MODE, MSPEC>(w, wk, task, lane);
        __syncwarp();
        if (lane == 0) {
            __threadfence();
            atomicAdd(w.ctrl + C_SERVED, 1u);
        }
    }
    asm volatile("griddepcontrol.launch_dependents;");
    if (w.single) {
        __syncwarp();
        uint32_t last = 0;
        if (lane == 0) {
#pragma unroll 1
            while (lw::ld_acquire_u32(w.ctrl + C_FIN) != nseg) __nanosleep(400);   // every lane done
            __threadfence();
            last = atomicAdd(w.ctrl + C_DONE, 1u) == gridDim.x - 1;
        }
        if (__shfl_sync(FULL, last, 0)) {
            __threadfence();
            if (*(volatile uint32_t *)(w.ctrl + C_OVF)) {
                walker_finish(wk);
                Walker fw;                              // the library's walker, on the same shared memory
                walker_init(fw, ring, w.p, lane);
                fix_overflows<MODE, MSPEC>(w, fw, lane);
                walker_finish(fw);
            }
        }
    }
    walker_finish(wk);
}

// Range calls on the lane walker, after k_lpost: if the last segment's chain
// turned out not to be the valid one (k_lpost then zeroed tail_n), walk the
// tail again from the true overhang (k_lpost's summary) with one warp; then
// push the exchange block into the next range's mailbox when asked (the fused
// exchange, as k_post does on the warp-walker path).
template <int MODE, int MSPEC>
__global__ void __launch_bounds__(32) k_ltail(Work w)
{
    __shared__ __align__(128) uint8_t ring[RING];
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int lane = threadIdx.x;
    if (w.tail_max && w.summary && *(volatile uint64_t *)w.tail_n == 0) {
        const uint64_t abase = (uint64_t)(uintptr_t)w.in;
        const uint64_t from = w.summary[0] - w.out_add;              // the overhang, offset into `in`
        Walker wk;
        walker_init(wk, ring, w.p, lane);
        uint32_t base = walker_begin(wk, abase + from, abase + w.total);
        const uint64_t off = wk.rb - abase;
        ListBuf tb{0, 0};
        if (from < w.total) {
            lb_push(tb, from + w.out_add, w.tail, lane);
#pragma unroll 1
            while (tb.n < w.tail_max && base + w.p.mx <= wk.end_rel) {
                const uint32_t c = resolve<MODE, MSPEC>(wk, w.p, base, lane);
                SEQCDC_ASSERT_CUT(base, c, w.p, wk.end_rel);
                lb_push(tb, off + c + w.out_add, w.tail, lane);
                base = c;
            }
        }
        lb_flush(tb, w.tail, lane);
        walker_finish(wk);
        if (lane == 0) *w.tail_n = tb.n;
    }
    if (w.push_blk) {
        __syncwarp();
        __threadfence();
        const uint64_t tn = w.tail_n ? min(*(volatile uint64_t *)w.tail_n, (uint64_t)w.tail_max) : 0;
        for (uint32_t i = lane; i < 3 + tn; i += 32)
            w.push_blk[i] = i == 0 ? w.summary[0] : i == 1 ? w.summary[1] : i == 2 ? tn : __ldcg(w.tail + (i - 3));
        __syncwarp();
        if (lane == 0) {
            __threadfence_system();
            asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(w.push_flag), "l"(w.push_value) : "memory");
        }
    }
}

}  // namespace seqcdc
