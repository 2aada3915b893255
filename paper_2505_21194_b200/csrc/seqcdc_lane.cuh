// seqcdc_lane.cuh -- the per-lane, skip-aware SeqCDC walker (SURVEY.md 8(f)
// NEXT-2 made the hot path for long streams).  Included by seqcdc.cu after the
// segment helpers (Work, Seg, get_seg, seg_start, fix_overflows).
//
// Why: the method itself never reads the sub-minimum region of a chunk
// nor the bytes a content-defined skip jumps over; on config 5
// it compares bytes in only 3.8% of the stream's 32-B sectors.  The warp
// walker streams every byte through shared memory and is therefore bound by
// HBM at ~n / 6.6 TB/s.  Here every LANE owns one speculative chain (one
// segment) and fetches only the 128-B lines its scan touches, with 1-D bulk
// copies (TMA, cp.async.bulk) into two private line slots, each completing on
// its own mbarrier.  A lane whose line has not landed simply skips that loop
// iteration (mbarrier.test_wait, no blocking), so the warp keeps scanning for
// the lanes whose data is there; thousands of chains per SM hide the HBM
// latency of the dependent chunk-to-chunk jumps.
//
// One loop iteration of a lane examines one 16-byte group: 16 byte pairs
// (bytes q..q+16), classified with SIMD-in-word compares (4 pairs per 32-bit
// word), the favourable-run mask by funnel-shift AND with the
// previous group's flags, the opposing count by popc and the
// SkipTrigger-th opposing pair by a SWAR byte select.  Decision in
// pair order: run end first -> cut; T-th opposing pair first -> skip
// to d+1+S with fresh counters (reading c3); neither -> next group; past
// the limit -> forced cut.
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
constexpr uint32_t SMEM = THREADS * STRIDE;

static_assert(SMEM <= 48 * 1024, "static shared memory");
static_assert(SEQCDC_LW_PF % 16 == 0 && SEQCDC_LW_PF < (int)LINE, "prefetch point inside a line");

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
#pragma unroll
        for (uint32_t i = 0; i < LINE; i += 16) cp_async16(dst + i, src + i);
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(mb) : "memory");
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

__device__ __forceinline__ void drain(Src &s)
{
#pragma unroll 1
    while (s.pend) poll(s);
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
    c.q = a & ~15u;
    c.la = a & 15u;
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

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t *p)
{
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Publish a task for the warps (segment s's extension, or with `tail` the
// range call's tail): its list writes are ordered before the release store.
__device__ __forceinline__ void hand_off(const Work &w, uint32_t s, bool tail)
{
    const uint32_t idx = atomicAdd(w.ctrl + C_HAND, 1u);
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(w.hand + idx), "r"((s + 1) | (tail ? 0x80000000u : 0u))
                 : "memory");
}

// A cut of lane s's chain at relative position `cut`: record it where the
// phase says (speculative list, extension list with the merge check, or the
// range tail) and decide whether the chain goes on.  Returns false when the
// lane's work is done (its results are written).
__device__ __forceinline__ bool on_cut(const Work &w, Chain &c, const Src &src, const Seg &g, uint32_t s,
                                       uint64_t stop_abs, uint32_t cut)
{
    const uint64_t cabs = c.off + cut;
    if (c.ph == PH_SPEC && cut >= c.hi_rel) {          // first cut past the segment: the extension starts
        TL_LANE(s, 1, 0);
        st_release_u64(w.Lcnt + s, (uint64_t)c.n | DONE_BIT);
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
        hand_off(w, s, true);
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
                if (!(c.t_word & DONE_BIT)) return true;   // not decidable yet: walk on
                const uint32_t cnt = (uint32_t)(c.t_word & CNT_MASK);
#pragma unroll 1
                while (c.cand < cabs && c.j + 1 < cnt) {
                    c.j++;
                    c.cand = __ldcg(w.L + c.t_Loff + c.j);
                }
                if (c.cand != cabs) {                   // not a cut of the owning chain: walk on
                    if (c.n < w.lw_ext_cap) return true;
                    w.Xcnt[s] = c.n;                    // a long extension: a warp continues it
                    hand_off(w, s, false);
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
// (dense cp.async ring in the warp's idle lane slots, seqcdc_device.cuh):
// continue segment s's extension from its last cut until a cut coincides with
// the chain owning its region (as walk_segment's extension does), or walk a
// range call's tail (up to tail_max cuts past the overhang, only chunks wholly
// inside the buffer).
template <int MODE, int MSPEC>
__device__ void lw_serve(const Work &w, Walker &wk, uint32_t task, int lane)
{
    const uint32_t s = (task & 0x7fffffffu) - 1;
    const bool tail = task >> 31;
    const uint64_t abase = (uint64_t)(uintptr_t)w.in;
    const Seg g = get_seg(w, s);
    if (tail) {
        const uint64_t nl = __ldcg(w.Lcnt + s) & CNT_MASK;
        const uint64_t from = __ldcg(w.L + g.Loff + nl - 1);          // the overhang
        uint32_t base = walker_begin(wk, abase + from, abase + g.E);
        const uint64_t off = wk.rb - abase;
        ListBuf tb{0, 0};
        if (base < wk.end_rel) {
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
        if (lane == 0) *w.tail_n = tb.n;
        return;
    }
    uint64_t *Xs = w.X + g.Xoff;
    const uint32_t n0 = __ldcg(w.Xcnt + s);
    const uint64_t from = __ldcg(Xs + n0 - 1);
    ListBuf xb;
    xb.n = n0;
    xb.v = lane < (int)(n0 & 31) ? __ldcg(Xs + (n0 & ~31u) + lane) : 0;   // the open batch
    uint32_t base = walker_begin(wk, abase + from, abase + g.E);
    const uint64_t off = wk.rb - abase;
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
        const uint32_t c = resolve<MODE, MSPEC>(wk, w.p, base, lane);
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
            // complete (its lane never waits on a warp), so every cut is decided
            // at once instead of being walked past
            if (lane == 0)
#pragma unroll 1
                while (!(ld_acquire_u64(w.Lcnt + t) & DONE_BIT)) __nanosleep(200);
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
    mb_init(mb_of(src, 0));
    mb_init(mb_of(src, 1));
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

    // One step of every lane per iteration, in lockstep: examine one group if
    // its lines are complete, handle a cut, keep the next lines on their way.
    uint32_t step = 0;
#pragma unroll 1
    while (__any_sync(FULL, c.ph != PH_DONE)) {
        step++;
        if (c.ph == PH_DONE) continue;
        if (src.pend) poll(src);
        uint32_t cut = pend;
        pend = NONE;
        if (cut == NONE) {
            const uint32_t l0 = c.q >> LSH;
            // byte q+16 lies in the next line only for the line's last group
            const bool two = (c.q & LMASK) == LINE - 16 && c.q + 16 <= c.lim2 + 1;
            if (ready(src, l0) && (!two || ready(src, l0 + 1))) {
                cut = scan_group<MODE, M4>(c, src, p);
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
                if (!chunk_begin(c, src, p, cut)) pend = c.limit;
            } else if (on_cut(w, c, src, g, s, stop_abs, cut)) {
                if (!chunk_begin(c, src, p, cut)) pend = c.limit;
            }
        }
        if (c.ph != PH_DONE && pend == NONE) {          // the lines the next groups need, on their way
            const uint32_t l0 = c.q >> LSH;
            if (!has(src, l0)) {
                request(src, l0);
            } else if ((c.q & LMASK) >= SEQCDC_LW_PF && !has(src, l0 + 1) && ((l0 + 1) << LSH) < src.end_rel) {
                request(src, l0 + 1);
            }
        }
    }
    drain(src);
    mb_inval(mb_of(src, 0));
    mb_inval(mb_of(src, 1));
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
    __shared__ __align__(128) uint8_t ring[RING];
    const int lane = threadIdx.x;
    const uint32_t nseg = w.ctrl[C_BAD] ? 0u : nseg_total(w);
    Walker wk;
    walker_init(wk, ring, w.p, lane);
#pragma unroll 1
    for (;;) {
        uint32_t j = 0;
        if (lane == 0) j = atomicAdd(w.ctrl + C_HNEXT, 1u);
        j = __shfl_sync(FULL, j, 0);
        if (j >= nseg) break;                                   // at most one task per lane
        uint32_t task = 0;
        if (lane == 0) {
#pragma unroll 1
            for (;;) {
                task = lw::ld_acquire_u32(w.hand + j);
                if (task) break;
                if (lw::ld_acquire_u32(w.ctrl + C_FIN) == nseg) {   // every task is published
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
            if (*(volatile uint32_t *)(w.ctrl + C_OVF)) fix_overflows<MODE, MSPEC>(w, wk, lane);
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
