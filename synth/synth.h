/*
 * synth.h -- seeded, block-addressable synthetic byte streams.
 *
 * This module is the ONE piece shared by the product path and the CPU oracle
 * (DESIGN.md "Inputs"): it makes the bytes, and holds none of SeqCDC's
 * arithmetic.  The same inline functions compile for the host (gcc or nvcc's
 * host pass) and the device, so host and device produce identical bytes.
 *
 * Every stream is an infinite sequence indexed by absolute byte position.  It
 * is cut into SYNTH_BLOCK-byte blocks; block k is a pure function of
 * (kind, seed, k), so any range can be generated independently (shards,
 * streaming oracles, device-side generation for 64 GiB inputs).
 *
 * Kinds (stand-ins for the paper's datasets, which are not available here;
 * PAPER.md Table II):
 *   SYNTH_UNIFORM    i.i.d. uniform bytes ("randomized data")
 *   SYNTH_MARKOV     order-1 Markov text over 60 printable symbols with
 *                    Dirichlet-like skewed rows and ~5% repeated-token spans
 *                    (LNX/DEV-like source text)
 *   SYNTH_ZEROHEAVY  zero runs U[64,4096] alternating with random blocks
 *                    U[64,2710] (~60% zeros; DEB/TPCC VM-image-like)
 *   SYNTH_RAMPMIX    pieces of length U[2,600]: half uniform random, half
 *                    +-1 byte ramps (start U[0,255], direction 50/50)
 *                    (BASELINE config 5 adversarial mix)
 */
#ifndef SYNTH_H_
#define SYNTH_H_

#include <stdint.h>

#if defined(__CUDACC__)
#define SYNTH_HD __host__ __device__ __forceinline__
#else
#define SYNTH_HD static inline
#endif

#define SYNTH_UNIFORM 0
#define SYNTH_MARKOV 1
#define SYNTH_ZEROHEAVY 2
#define SYNTH_RAMPMIX 3
#define SYNTH_NKINDS 4

#define SYNTH_BLOCK_SHIFT 16
#define SYNTH_BLOCK ((uint64_t)1 << SYNTH_BLOCK_SHIFT) /* 64 KiB */

#define SYNTH_NSYM 60

/* SplitMix64 finaliser: counter-based generator, x = key + ctr * golden. */
SYNTH_HD uint64_t synth_mix64(uint64_t z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

SYNTH_HD uint64_t synth_rng(uint64_t key, uint64_t ctr)
{
    return synth_mix64(key + (ctr + 1) * 0x9E3779B97F4A7C15ull);
}

SYNTH_HD uint64_t synth_key(uint64_t seed, uint64_t kind, uint64_t block)
{
    return synth_mix64(synth_mix64(seed * 0xD1B54A32D192ED03ull + kind) ^ (block * 0xA24BAED4963EE407ull));
}

/* Uniform: byte i = byte (i & 7) of rng(seed, i >> 3).  Not block-sequential. */
SYNTH_HD uint8_t synth_uniform_byte(uint64_t seed, uint64_t i)
{
    uint64_t w = synth_rng(synth_key(seed, SYNTH_UNIFORM, 0), i >> 3);
    return (uint8_t)(w >> (8 * (i & 7)));
}

/* ---------------------------------------------------------------- Markov model */
typedef struct {
    uint8_t sym[SYNTH_NSYM];                  /* printable symbols */
    uint32_t cdf[SYNTH_NSYM][SYNTH_NSYM];     /* row r: P(next = j | prev = r), cumulative, 2^32 scale */
} synth_markov_t;

/* Integer-only model build (identical on host and device): 60 symbols drawn
 * from ASCII 32..126 by a seeded partial shuffle; row weights w = u^3 with u
 * a 16-bit uniform (a heavy-tailed, Dirichlet(~0.3)-like row). */
SYNTH_HD void synth_markov_build(uint64_t seed, synth_markov_t *m)
{
    uint8_t pool[95];
    for (int i = 0; i < 95; i++) pool[i] = (uint8_t)(32 + i);
    uint64_t key = synth_key(seed, SYNTH_MARKOV, 0xFFFFFFFFull);
    for (int i = 0; i < SYNTH_NSYM; i++) {
        int j = i + (int)(synth_rng(key, (uint64_t)i) % (uint64_t)(95 - i));
        uint8_t t = pool[i]; pool[i] = pool[j]; pool[j] = t;
        m->sym[i] = pool[i];
    }
    for (int r = 0; r < SYNTH_NSYM; r++) {
        uint64_t w[SYNTH_NSYM];
        uint64_t tot = 0;
        for (int j = 0; j < SYNTH_NSYM; j++) {
            uint64_t u = (synth_rng(key, 1000 + (uint64_t)r * SYNTH_NSYM + (uint64_t)j) >> 48) + 1;
            w[j] = u * u * u;                 /* <= 2^48 */
            tot += w[j];                      /* <= 60 * 2^48 < 2^54 */
        }
        uint64_t acc = 0;
        for (int j = 0; j < SYNTH_NSYM; j++) {
            acc += w[j];
            /* cdf in [1, 2^32]; last entry forced to 2^32-1 so every u32 maps */
            uint64_t c = (acc << 10) / (tot >> 22 ? tot >> 22 : 1);
            if (c > 0xFFFFFFFFull) c = 0xFFFFFFFFull;
            m->cdf[r][j] = (uint32_t)c;
        }
        m->cdf[r][SYNTH_NSYM - 1] = 0xFFFFFFFFu;
    }
}

SYNTH_HD int synth_markov_step(const synth_markov_t *m, int prev, uint32_t u)
{
    const uint32_t *c = m->cdf[prev];
    int j = 0;
    while (j < SYNTH_NSYM - 1 && c[j] <= u) j++;
    return j;
}

/* ---------------------------------------------------------------- block generators
 * Sequential generators keep a small state machine; a block starts from a state
 * derived from (seed, kind, block) alone. */
typedef struct {
    uint64_t key, ctr;
    int kind;
    /* markov */
    int prev;
    int span_left, tok_len, tok_pos;
    uint8_t tok[16];
    /* zeroheavy / rampmix */
    int piece_left, piece_type;
    uint8_t ramp_val;
    int ramp_dir;
} synth_state_t;

SYNTH_HD uint64_t synth_next(synth_state_t *s) { return synth_rng(s->key, s->ctr++); }

SYNTH_HD void synth_block_init(synth_state_t *s, int kind, uint64_t seed, uint64_t block)
{
    s->key = synth_key(seed, (uint64_t)kind, block);
    s->ctr = 0;
    s->kind = kind;
    s->prev = (int)(synth_next(s) % SYNTH_NSYM);
    s->span_left = 0; s->tok_len = 0; s->tok_pos = 0;
    s->piece_left = 0; s->piece_type = 0; s->ramp_val = 0; s->ramp_dir = 1;
}

/* Next byte of a sequential kind (MARKOV, ZEROHEAVY, RAMPMIX). */
SYNTH_HD uint8_t synth_block_byte(synth_state_t *s, const synth_markov_t *m)
{
    if (s->kind == SYNTH_MARKOV) {
        if (s->span_left > 0) {                       /* inside a repeated-token span */
            uint8_t b = s->tok[s->tok_pos];
            s->tok_pos = (s->tok_pos + 1 == s->tok_len) ? 0 : s->tok_pos + 1;
            s->span_left--;
            return b;
        }
        uint64_t r = synth_next(s);
        if ((r & 0xFFFFFull) < 171ull) {              /* p ~ 1/6132: start a span (~5% of bytes) */
            s->tok_len = 2 + (int)((r >> 20) % 15);   /* token 2..16 bytes from the chain */
            int rep = 8 + (int)((r >> 28) % 57);      /* repeated 8..64 times */
            for (int k = 0; k < s->tok_len; k++) {
                s->prev = synth_markov_step(m, s->prev, (uint32_t)(synth_next(s) >> 32));
                s->tok[k] = m->sym[s->prev];
            }
            s->span_left = s->tok_len * rep - 1;
            s->tok_pos = 1 % s->tok_len;
            return s->tok[0];
        }
        s->prev = synth_markov_step(m, s->prev, (uint32_t)(r >> 32));
        return m->sym[s->prev];
    }
    if (s->kind == SYNTH_ZEROHEAVY) {
        if (s->piece_left == 0) {
            uint64_t r = synth_next(s);
            s->piece_type ^= 1;                        /* alternate zero run / random block */
            s->piece_left = s->piece_type ? 64 + (int)(r % 4033)    /* zeros U[64,4096] */
                                          : 64 + (int)(r % 2647);   /* random U[64,2710] */
        }
        s->piece_left--;
        if (s->piece_type) return 0;
        return (uint8_t)(synth_next(s) >> 56);
    }
    /* SYNTH_RAMPMIX */
    if (s->piece_left == 0) {
        uint64_t r = synth_next(s);
        s->piece_left = 2 + (int)(r % 599);            /* U[2,600] */
        s->piece_type = (int)((r >> 32) & 1);          /* 1 = ramp, 0 = random */
        s->ramp_val = (uint8_t)(r >> 40);              /* U[0,255] */
        s->ramp_dir = ((r >> 48) & 1) ? 1 : -1;
    }
    s->piece_left--;
    if (s->piece_type) {
        uint8_t v = s->ramp_val;
        s->ramp_val = (uint8_t)(s->ramp_val + s->ramp_dir);
        return v;
    }
    return (uint8_t)(synth_next(s) >> 56);
}

#endif /* SYNTH_H_ */
