// seqcdc_dedup.cu -- the step after chunking (PAPER.md
// §2): a collision-resistant fingerprint per chunk (SHA-256),
// duplicate detection against the fingerprints already seen, and the
// stored ("unique") bytes that Eq. 1 turns into space savings.
//
//   k_sha256      one thread per chunk: FIPS 180-4 SHA-256 of d_in[c_{i-1}, c_i)
//                 (integer-ALU bound: ~22 ALU ops per byte)
//   k_dedup_*     open-addressing hash set in device memory keyed by the digest;
//                 each distinct digest keeps its smallest chunk index (atomicCAS),
//                 so "first occurrence" is deterministic; unique bytes = sum of
//                 the sizes of first occurrences.
// No host synchronisation: the number of chunks is read on the device
// (d_ncuts, e.g. straight from seqcdc_chunk); grids are sized by a host bound.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "../../include/seqcdc.h"

#define SEQCDC_API extern "C" __attribute__((visibility("default")))
// internal (seqcdc.cu): the library's memory pool (keeps its memory across syncs)
int seqcdc_internal_pool(cudaMemPool_t *pool);
void seqcdc_note_launches(int k);

namespace seqcdc {
namespace {

__constant__ uint32_t K256[64] = {
    0x428a2f98u, 0x71374491u, 0xb5c0fbcfu, 0xe9b5dba5u, 0x3956c25bu, 0x59f111f1u, 0x923f82a4u, 0xab1c5ed5u,
    0xd807aa98u, 0x12835b01u, 0x243185beu, 0x550c7dc3u, 0x72be5d74u, 0x80deb1feu, 0x9bdc06a7u, 0xc19bf174u,
    0xe49b69c1u, 0xefbe4786u, 0x0fc19dc6u, 0x240ca1ccu, 0x2de92c6fu, 0x4a7484aau, 0x5cb0a9dcu, 0x76f988dau,
    0x983e5152u, 0xa831c66du, 0xb00327c8u, 0xbf597fc7u, 0xc6e00bf3u, 0xd5a79147u, 0x06ca6351u, 0x14292967u,
    0x27b70a85u, 0x2e1b2138u, 0x4d2c6dfcu, 0x53380d13u, 0x650a7354u, 0x766a0abbu, 0x81c2c92eu, 0x92722c85u,
    0xa2bfe8a1u, 0xa81a664bu, 0xc24b8b70u, 0xc76c51a3u, 0xd192e819u, 0xd6990624u, 0xf40e3585u, 0x106aa070u,
    0x19a4c116u, 0x1e376c08u, 0x2748774cu, 0x34b0bcb5u, 0x391c0cb3u, 0x4ed8aa4au, 0x5b9cca4fu, 0x682e6ff3u,
    0x748f82eeu, 0x78a5636fu, 0x84c87814u, 0x8cc70208u, 0x90befffau, 0xa4506cebu, 0xbef9a3f7u, 0xc67178f2u};

__device__ __forceinline__ uint32_t rotr(uint32_t x, int n) { return __funnelshift_r(x, x, n); }
__device__ __forceinline__ uint32_t bswap(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

// a * one + b on the FMA pipe (IMAD): `one` is an opaque 1, so ptxas cannot
// turn it back into an ALU-pipe IADD3.  The compression is ALU-pipe bound
// (rotates and LOP3 xors); moving its additions to the otherwise idle FMA
// pipe raises throughput (profiles/r01: ALU pipe 90% busy, FMA 4%).
__device__ __forceinline__ uint32_t fadd(uint32_t a, uint32_t b, uint32_t one)
{
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(one), "r"(b));
    return r;
}

// One 64-byte block (FIPS 180-4 §6.2.2); w = the block's 16 big-endian words.
__device__ __forceinline__ void sha256_block(uint32_t st[8], uint32_t w[16], uint32_t one)
{
    uint32_t a = st[0], b = st[1], c = st[2], d = st[3], e = st[4], f = st[5], g = st[6], h = st[7];
#pragma unroll
    for (int i = 0; i < 64; i++) {
        if (i >= 16) {
            const uint32_t w15 = w[(i - 15) & 15], w2 = w[(i - 2) & 15];
            const uint32_t s0 = rotr(w15, 7) ^ rotr(w15, 18) ^ (w15 >> 3);
            const uint32_t s1 = rotr(w2, 17) ^ rotr(w2, 19) ^ (w2 >> 10);
            w[i & 15] = fadd(w[i & 15], fadd(s0, w[(i - 7) & 15] + s1, one), one);
        }
        const uint32_t S1 = rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25);
        const uint32_t ch = (e & f) ^ (~e & g);
        const uint32_t t1 = fadd(h + K256[i], fadd(S1, fadd(ch, w[i & 15], one), one), one);
        const uint32_t S0 = rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22);
        const uint32_t maj = (a & b) ^ (a & c) ^ (b & c);
        const uint32_t t2 = fadd(S0, maj, one);
        h = g;
        g = f;
        f = e;
        e = fadd(d, t1, one);
        d = c;
        c = b;
        b = a;
        a = fadd(t1, t2, one);
    }
    st[0] += a;
    st[1] += b;
    st[2] += c;
    st[3] += d;
    st[4] += e;
    st[5] += f;
    st[6] += g;
    st[7] += h;
}

// 4-byte aligned little-endian word at aligned address p (only called for words
// that start before the chunk end, so never past the buffer's last word)
__device__ __forceinline__ uint32_t ldw(const uint8_t *p) { return __ldg((const uint32_t *)p); }

// Message word j of block k of a chunk [s, e) (FIPS 180-4 §5.1.1 padding):
// the data bytes of the block, 0x80 right after the last data byte, zeros, and
// the 64-bit bit length in words 14-15 of the chunk's last block.  Words that
// start at or past the chunk end are never loaded.
__device__ __forceinline__ void load_block(uint32_t w[16], const uint8_t *in, uint64_t s, uint64_t e, uint64_t k,
                                           bool last)
{
    const uint64_t len = e - s;
    const uint64_t rest = len - 64 * k;                     // data bytes from this block on (wraps when past the end)
    const int32_t valid = 64 * k > len ? -1 : (rest > 64 ? 64 : (int32_t)rest);   // data bytes in this block
    const uintptr_t o = (uintptr_t)in + s + 64 * k;
    const uintptr_t endp = (uintptr_t)in + e;
    const uint8_t *base = (const uint8_t *)(o & ~(uintptr_t)3);
    const uint32_t sh = 8u * (uint32_t)(o & 3);
    uint32_t prev = (uintptr_t)base < endp ? ldw(base) : 0u;
#pragma unroll
    for (int j = 0; j < 16; j++) {
        const uint8_t *p = base + 4 * (j + 1);
        const uint32_t nx = (uintptr_t)p < endp ? ldw(p) : 0u;
        uint32_t v = bswap(__funnelshift_r(prev, nx, sh));
        prev = nx;
        const int32_t vb = valid - 4 * j;                     // message bytes in this word
        if (vb <= 0) v = 0;
        else if (vb < 4) v &= ~(0xffffffffu >> (8 * vb));
        if (vb >= 0 && vb < 4) v |= 0x80u << (24 - 8 * vb);
        w[j] = v;
    }
    if (last) {
        const uint64_t bits = len * 8;
        w[14] = (uint32_t)(bits >> 32);
        w[15] = (uint32_t)bits;
    }
}

// Persistent, load-balanced: every lane compresses one 64-byte block per
// iteration (data or padding, the same straight-line code), so the 64-round
// compression never diverges; a lane that finishes its chunk writes the digest
// and takes the next chunk index from a counter (one atomic per warp), so the
// lanes of a warp no longer wait for the longest of 32 fixed chunks.
// (Prefetching the next chunk's bounds one chunk ahead measured slower:
// profiles/r01/dedup_next1_v3.jsonl.)
__global__ void __launch_bounds__(128) k_sha256(const uint8_t *in, const uint64_t *cuts, const uint64_t *ncuts_p,
                                                uint64_t cap, uint8_t *digests, uint32_t one,
                                                unsigned long long *next)
{
    const uint64_t n = min(*ncuts_p, cap);
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t T = (uint64_t)gridDim.x * blockDim.x;    // the first T chunks are assigned statically
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool act = i < n;
    uint64_t s = 0, e = 0, k = 0, nblk = 0;
    uint32_t st[8];
    auto start = [&]() {
        s = i ? cuts[i - 1] : 0;
        e = cuts[i];
        const uint64_t len = e - s;
        nblk = (len >> 6) + ((len & 63) <= 55 ? 1 : 2);
        k = 0;
        st[0] = 0x6a09e667u; st[1] = 0xbb67ae85u; st[2] = 0x3c6ef372u; st[3] = 0xa54ff53au;
        st[4] = 0x510e527fu; st[5] = 0x9b05688cu; st[6] = 0x1f83d9abu; st[7] = 0x5be0cd19u;
    };
    if (act) start();
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll 1
    while (__any_sync(0xffffffffu, act)) {
        uint32_t w[16];
        load_block(w, in, act ? s : 0, act ? e : 0, k, act && k + 1 == nblk);
        sha256_block(st, w, one);
        const bool fin = act && ++k == nblk;
        if (fin) {
            uint4 *out = (uint4 *)(digests + 32 * i);
            out[0] = make_uint4(bswap(st[0]), bswap(st[1]), bswap(st[2]), bswap(st[3]));
            out[1] = make_uint4(bswap(st[4]), bswap(st[5]), bswap(st[6]), bswap(st[7]));
        }
        const uint32_t want = __ballot_sync(0xffffffffu, fin);
        if (want) {
            const int leader = __ffs(want) - 1;
            unsigned long long b = 0;
            if ((int)lane == leader) b = atomicAdd(next, (unsigned long long)__popc(want));
            b = __shfl_sync(0xffffffffu, b, leader);
            if (fin) {
                i = T + b + __popc(want & lt);
                act = i < n;
                if (act) start();
            }
        }
    }
}

// ---------------------------------------------------------------- dedup index
constexpr uint64_t EMPTY = ~0ull;

__device__ __forceinline__ bool same_digest(const uint8_t *dg, uint64_t a, uint64_t b)
{
    const uint4 *x = (const uint4 *)(dg + 32 * a), *y = (const uint4 *)(dg + 32 * b);
    const uint4 x0 = x[0], x1 = x[1], y0 = y[0], y1 = y[1];
    return x0.x == y0.x && x0.y == y0.y && x0.z == y0.z && x0.w == y0.w && x1.x == y1.x && x1.y == y1.y &&
           x1.z == y1.z && x1.w == y1.w;
}

__device__ __forceinline__ uint64_t slot_of(const uint8_t *dg, uint64_t i, uint64_t mask)
{
    const uint2 h = *(const uint2 *)(dg + 32 * i);              // digest bytes 0..7 (uniformly distributed)
    return (((uint64_t)h.y << 32) | h.x) & mask;
}

__global__ void k_dedup_clear(uint64_t *table, uint64_t cap, uint64_t *unique)
{
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cap; i += (uint64_t)gridDim.x * blockDim.x)
        table[i] = EMPTY;
    if (blockIdx.x == 0 && threadIdx.x == 0) *unique = 0;
}

__global__ void k_dedup_insert(const uint8_t *dg, const uint64_t *ncuts_p, uint64_t bound, uint64_t *table,
                               uint64_t mask)
{
    const uint64_t n = min(*ncuts_p, bound);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t h = slot_of(dg, i, mask);
        for (;;) {
            unsigned long long cur = table[h];
            if (cur == EMPTY) {
                cur = atomicCAS((unsigned long long *)(table + h), EMPTY, (unsigned long long)i);
                if (cur == EMPTY) break;                       // inserted: i represents its digest
            }
            if (same_digest(dg, cur, i)) {                     // keep the smallest index of the digest
                while (i < cur) {
                    const unsigned long long prev =
                        atomicCAS((unsigned long long *)(table + h), cur, (unsigned long long)i);
                    if (prev == cur) break;
                    cur = prev;                                // another index of the same digest won
                }
                break;
            }
            h = (h + 1) & mask;                                // a different digest: linear probing
        }
    }
}

__global__ void __launch_bounds__(256) k_dedup_mark(const uint8_t *dg, const uint64_t *cuts, const uint64_t *ncuts_p,
                                                    uint64_t bound, const uint64_t *table, uint64_t mask,
                                                    uint8_t *first, uint64_t *unique)
{
    const uint64_t n = min(*ncuts_p, bound);
    uint64_t acc = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t h = slot_of(dg, i, mask);
        uint64_t rep;
        for (;;) {
            rep = table[h];
            if (rep == i || same_digest(dg, rep, i)) break;
            h = (h + 1) & mask;
        }
        const bool f = rep == i;
        if (first) first[i] = f ? 1 : 0;
        if (f) acc += cuts[i] - (i ? cuts[i - 1] : 0);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd((unsigned long long *)unique, (unsigned long long)acc);
}

uint64_t table_cap(uint64_t max_cuts)
{
    uint64_t cap = 1024;
    while (cap < 2 * max_cuts) cap <<= 1;
    return cap;
}

}  // namespace
}  // namespace seqcdc

using namespace seqcdc;

SEQCDC_API int seqcdc_fingerprint(const uint8_t *d_in, const uint64_t *d_cuts, const uint64_t *d_ncuts,
                                  uint64_t max_cuts, uint8_t *d_digests, void *stream)
{
    if (!d_ncuts || (max_cuts && (!d_in || !d_cuts || !d_digests))) return SEQCDC_EINVAL;
    if (((uintptr_t)d_digests & 15) != 0) return SEQCDC_EINVAL;
    if (max_cuts == 0) return SEQCDC_OK;
    cudaStream_t st = (cudaStream_t)stream;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // persistent grid: exactly the resident CTAs (all of them start at once, so the
    // statically assigned first chunks do not wait for a second wave), never more
    // threads than chunks
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sha256, 128, 0) != cudaSuccess || occ < 1) occ = 4;
    if (const char *e = getenv("SEQCDC_SHA_CTAS_PER_SM")) occ = std::max(1, std::min(occ, atoi(e)));   // tuning
    const uint64_t grid = std::min<uint64_t>((max_cuts + 127) / 128, (uint64_t)sms * occ);
    unsigned long long *next = nullptr;               // chunk counter for the dynamic assignment
    cudaMemPool_t pool;
    if (seqcdc_internal_pool(&pool) != SEQCDC_OK) return SEQCDC_ECUDA;
    if (cudaMallocFromPoolAsync((void **)&next, 8, pool, st) != cudaSuccess) return SEQCDC_ENOMEM;
    cudaMemsetAsync(next, 0, 8, st);
    k_sha256<<<(unsigned)grid, 128, 0, st>>>(d_in, d_cuts, d_ncuts, max_cuts, d_digests, 1u, next);
    seqcdc_note_launches(1);
    cudaFreeAsync(next, st);
    return cudaGetLastError() == cudaSuccess ? SEQCDC_OK : SEQCDC_ECUDA;
}

SEQCDC_API size_t seqcdc_dedup_workspace_size(uint64_t max_cuts) { return 8 * table_cap(max_cuts); }

SEQCDC_API int seqcdc_dedup(const uint8_t *d_digests, const uint64_t *d_cuts, const uint64_t *d_ncuts,
                            uint64_t max_cuts, uint8_t *d_first, uint64_t *d_unique_bytes, void *d_ws,
                            size_t ws_bytes, void *stream)
{
    if (!d_ncuts || !d_unique_bytes || (max_cuts && (!d_digests || !d_cuts))) return SEQCDC_EINVAL;
    if (((uintptr_t)d_digests & 15) != 0) return SEQCDC_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    const uint64_t cap = table_cap(max_cuts);
    uint64_t *table = (uint64_t *)d_ws;
    bool owned = false;
    if (table) {
        if (ws_bytes < 8 * cap) return SEQCDC_ENOMEM;
    } else {
        cudaMemPool_t pool;
        if (seqcdc_internal_pool(&pool) != SEQCDC_OK) return SEQCDC_ECUDA;
        if (cudaMallocFromPoolAsync((void **)&table, 8 * cap, pool, st) != cudaSuccess) return SEQCDC_ENOMEM;
        owned = true;
    }
    k_dedup_clear<<<592, 256, 0, st>>>(table, cap, d_unique_bytes);
    seqcdc_note_launches(1);
    if (max_cuts) {
        k_dedup_insert<<<592, 256, 0, st>>>(d_digests, d_ncuts, max_cuts, table, cap - 1);
        k_dedup_mark<<<592, 256, 0, st>>>(d_digests, d_cuts, d_ncuts, max_cuts, table, cap - 1, d_first,
                                          d_unique_bytes);
        seqcdc_note_launches(2);
    }
    if (owned) cudaFreeAsync(table, st);
    return cudaGetLastError() == cudaSuccess ? SEQCDC_OK : SEQCDC_ECUDA;
}
