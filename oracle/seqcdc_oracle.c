/*
 * seqcdc_oracle.c -- plain, slow, obviously-correct CPU SeqCDC (TEST INFRASTRUCTURE).
 *
 * This file is test infrastructure, not product code.  Only tests/, the
 * __graft_entry__.smoke() self-check and bench.py's cpu_baseline /
 * --impl reference legs may load it.  It shares no code, header, table or
 * constant with the CUDA path under paper_2505_21194_b200/ (and includes
 * nothing from it); neither side imports the other.
 *
 * It is a literal, byte-at-a-time transcription of the method in the order
 * the paper states it (PAPER.md = /root/reference/PAPER.md, "P:n" = line n):
 *
 *   P:153  "The sequence must have a length of SeqLength to be considered a
 *           boundary candidate. Once such a sequence is found, a boundary is
 *           inserted at its end."  -> a run of SeqLength bytes, each strictly
 *           greater (Increasing) / smaller (Decreasing) than the one before;
 *           the cut is the offset one past the run's last byte.
 *   P:163  Increasing and Decreasing modes are exclusive.
 *   P:179  "skips scanning data of size (minimum_chunk_size - SeqLength) at the
 *           beginning of each chunk" -> scanning starts at base + min - L.
 *   P:189  "When SkipTrigger pairs of bytes in opposing order are detected ...
 *           skips scanning the next few bytes ... resets its counters and
 *           resumes scanning."
 *   P:227  "The exact position to jump from is determined using the first set
 *           bit that causes the total to exceed SkipTrigger."
 *   P:215,217  the vector compares are strict (cmpgt / cmplt): equal bytes are
 *           neither favourable nor opposing.
 *   P:266  "a boundary is inserted at the maximum chunk size".
 *
 * Readings where the paper is silent or ambiguous (DESIGN.md "Readings",
 * SURVEY.md 8(c) c1-c9): SeqLength counts bytes (c1); the skip fires when the
 * opposing count REACHES SkipTrigger (c2); the scan resumes SkipSize bytes past
 * the second byte of the triggering pair, i.e. at d+1+S (c3); both counters
 * reset at chunk start and after a skip, the run also resets on any
 * non-favourable pair (c4); equal bytes set neither flag (c5); bytes compare
 * as UNSIGNED (c6; `flags` bit 0 selects the signed reading, P:215's
 * mm512_cmpgt without a type suffix could be the signed epi8 compare; `flags`
 * bit 1 selects c1's alternative: SeqLength counts favourable comparisons, so
 * a run of L+1 bytes ends a chunk, the scan anchor staying at base + min - L);
 * skipped bytes count toward max and a skip landing past the
 * limit gives the limit (c8); the last chunk may be shorter than min and the
 * last cut is n; n == 0 gives no cuts (c9).
 *
 * Pins: tests/test_oracle_pins.py (hand vectors from P:211-227 and SPEC
 * S:112-114, closed forms for ramps / constant data, brute force against an
 * independently written query formulation, invariants).
 */
#include <stdint.h>
#include <stddef.h>

#define ORACLE_OK 0
#define ORACLE_EINVAL 1
#define ORACLE_ECAP 2

/* Returns 0 when the parameters are acceptable (same rules as S:94-99). */
int oracle_check_params(uint32_t mode, uint32_t seq_length, uint32_t skip_trigger,
                        uint64_t min_size, uint64_t max_size)
{
    if (mode > 1) return ORACLE_EINVAL;
    if (seq_length < 2) return ORACLE_EINVAL;
    if (skip_trigger < 1) return ORACLE_EINVAL;
    if (min_size < seq_length) return ORACLE_EINVAL;
    if (max_size < min_size) return ORACLE_EINVAL;
    return ORACLE_OK;
}

/*
 * Measurement only (SURVEY.md 8(d) "algorithmic bytes"): the distinct aligned
 * units of 2^shift bytes (absolute stream offsets: origin + position) that hold
 * a byte of some compared pair (i, i+1) -- the bytes the method itself reads.
 * Pairs are visited in increasing i, so "distinct" is a running maximum.
 * Does not influence any cut.
 */
#define ORACLE_TOUCH_MAX 4
typedef struct {
    uint32_t nunits;
    uint32_t shift[ORACLE_TOUCH_MAX];
    uint64_t origin;                       /* absolute offset of b[0] */
    uint64_t first[ORACLE_TOUCH_MAX];      /* first unit touched (UINT64_MAX: none yet) */
    uint64_t last[ORACLE_TOUCH_MAX];       /* last unit touched  (UINT64_MAX: none yet) */
    uint64_t count[ORACLE_TOUCH_MAX];      /* distinct units touched */
} oracle_touch_t;

static void touch_byte(oracle_touch_t *t, uint64_t pos)
{
    for (uint32_t g = 0; g < t->nunits; g++) {
        uint64_t u = (t->origin + pos) >> t->shift[g];
        if (t->last[g] == UINT64_MAX || u > t->last[g]) {
            if (t->first[g] == UINT64_MAX) t->first[g] = u;
            t->last[g] = u;
            t->count[g]++;
        }
    }
}

/*
 * One chunk: the cut that ends the chunk starting at `base` of the stream
 * b[0..n).  Requires base < n.  *examined (if non-null) is incremented by the
 * number of byte pairs compared (the oracle's "algorithmic work" counter);
 * `touch` (if non-null) records the units those pairs' bytes lie in.
 */
static uint64_t next_cut_impl(const uint8_t *b, uint64_t n, uint64_t base,
                              uint32_t mode, uint32_t seq_length, uint32_t skip_trigger,
                              uint32_t skip_size, uint64_t min_size, uint64_t max_size,
                              uint32_t flags, uint64_t *examined, oracle_touch_t *touch)
{
    const uint32_t sgn = flags & 1u;               /* signed bytes (c6 alternative) */
    const uint32_t run_end = (flags & 2u) ? seq_length + 1 : seq_length;   /* bytes in a qualifying run (c1) */
    uint64_t limit = base + max_size;              /* P:266 max forced cut */
    if (limit > n) limit = n;                      /* end of stream (c9) */
    uint64_t i = base + min_size - seq_length;     /* P:179 sub-minimum skip */
    uint32_t run = 1;                              /* bytes in the current run */
    uint32_t opp = 0;                              /* opposing pairs since reset */
    for (;;) {
        if (i + 1 >= limit) return limit;          /* no pair (i, i+1) left */
        int x = sgn ? (int)(int8_t)b[i] : (int)b[i];          /* unsigned bytes (c6) */
        int y = sgn ? (int)(int8_t)b[i + 1] : (int)b[i + 1];  /* or signed (flag)    */
        if (examined) (*examined)++;
        if (touch) { touch_byte(touch, i); touch_byte(touch, i + 1); }
        int favourable, opposing;
        if (mode == 0) { favourable = x < y; opposing = x > y; }   /* Increasing */
        else           { favourable = x > y; opposing = x < y; }   /* Decreasing */
        if (favourable) {
            run += 1;
            if (run == run_end) return i + 2;      /* run ends at byte i+1 -> cut after it */
            i += 1;
        } else if (opposing) {
            run = 1;
            opp += 1;
            if (opp == skip_trigger) {             /* P:189 skip; reaches (c2) */
                i = i + 1 + skip_size;             /* land S past the pair's 2nd byte (c3) */
                run = 1;
                opp = 0;                           /* "resets its counters" */
                continue;
            }
            i += 1;
        } else {                                   /* equal bytes: neither (c5) */
            run = 1;
            i += 1;
        }
    }
}

uint64_t oracle_next_cut(const uint8_t *b, uint64_t n, uint64_t base,
                         uint32_t mode, uint32_t seq_length, uint32_t skip_trigger,
                         uint32_t skip_size, uint64_t min_size, uint64_t max_size,
                         uint32_t flags, uint64_t *examined)
{
    return next_cut_impl(b, n, base, mode, seq_length, skip_trigger, skip_size,
                         min_size, max_size, flags, examined, 0);
}

/*
 * Whole stream: cuts[0..k) = exclusive chunk ends, strictly increasing, the
 * last one equal to n.  Returns k >= 0, or -(error) on bad parameters or when
 * `cap` is too small.  *examined (optional) accumulates compared pairs.
 */
int64_t oracle_chunk(const uint8_t *b, uint64_t n,
                     uint32_t mode, uint32_t seq_length, uint32_t skip_trigger,
                     uint32_t skip_size, uint64_t min_size, uint64_t max_size,
                     uint32_t flags, uint64_t *cuts, uint64_t cap, uint64_t *examined)
{
    if (oracle_check_params(mode, seq_length, skip_trigger, min_size, max_size))
        return -ORACLE_EINVAL;
    uint64_t k = 0, base = 0;
    while (base < n) {
        uint64_t c = oracle_next_cut(b, n, base, mode, seq_length, skip_trigger,
                                     skip_size, min_size, max_size, flags, examined);
        if (k >= cap) return -ORACLE_ECAP;
        cuts[k++] = c;
        base = c;
    }
    return (int64_t)k;
}

/*
 * Many independent streams (files are chunked independently):
 * stream j is b[offsets[j] .. offsets[j+1]).  Cuts are written as ABSOLUTE
 * offsets into b, stream after stream; cut_index[j] = index of stream j's
 * first cut, cut_index[ns] = total.  Returns total or -(error).
 */
int64_t oracle_chunk_batch(const uint8_t *b, const uint64_t *offsets, uint32_t ns,
                           uint32_t mode, uint32_t seq_length, uint32_t skip_trigger,
                           uint32_t skip_size, uint64_t min_size, uint64_t max_size,
                           uint32_t flags, uint64_t *cuts, uint64_t cap, uint64_t *cut_index)
{
    uint64_t total = 0;
    for (uint32_t j = 0; j < ns; j++) {
        cut_index[j] = total;
        uint64_t lo = offsets[j], hi = offsets[j + 1];
        int64_t k = oracle_chunk(b + lo, hi - lo, mode, seq_length, skip_trigger, skip_size,
                                 min_size, max_size, flags, cuts + total, cap - total, NULL);
        if (k < 0) return k;
        for (int64_t q = 0; q < k; q++) cuts[total + q] += lo;
        total += (uint64_t)k;
    }
    cut_index[ns] = total;
    return (int64_t)total;
}

/*
 * Window form for checking a long cut list in independent pieces (measurement
 * and parity infrastructure; same loop as oracle_chunk): chunk b[0..n) from
 * offset 0 as a chunk start, stopping after the chunk that starts beyond
 * `last_start` (a chunk starting at base is fixed by b[base .. base+max), P:179,
 * P:189, so the caller passes n >= last_start + max_size unless b ends at
 * the stream end).  `touch` (optional) accumulates the units the compared pairs
 * touch.  Returns the number of cuts or -(error).
 */
int64_t oracle_chunk_window(const uint8_t *b, uint64_t n, uint64_t last_start,
                            uint32_t mode, uint32_t seq_length, uint32_t skip_trigger,
                            uint32_t skip_size, uint64_t min_size, uint64_t max_size,
                            uint32_t flags, uint64_t *cuts, uint64_t cap,
                            uint64_t *examined, oracle_touch_t *touch)
{
    if (oracle_check_params(mode, seq_length, skip_trigger, min_size, max_size))
        return -ORACLE_EINVAL;
    uint64_t k = 0, base = 0;
    while (base < n && base <= last_start) {
        uint64_t c = next_cut_impl(b, n, base, mode, seq_length, skip_trigger,
                                   skip_size, min_size, max_size, flags, examined, touch);
        if (k >= cap) return -ORACLE_ECAP;
        cuts[k++] = c;
        base = c;
    }
    return (int64_t)k;
}
