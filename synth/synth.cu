// synth.cu -- host and device entry points of the seeded input generators
// (see synth.h).  Built into libsynth.so; used by tests, bench.py and the
// smoke check for BOTH the CUDA path and the CPU oracle.  Nothing here
// implements any part of SeqCDC.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>
#include <stdlib.h>

#include "synth.h"

#define SYNTH_API extern "C" __attribute__((visibility("default")))

// ------------------------------------------------------------------ host
static void fill_seq_host(int kind, uint64_t seed, uint64_t pos, uint64_t len, uint8_t *out,
                          const synth_markov_t *m)
{
    uint64_t end = pos + len;
    for (uint64_t blk = pos >> SYNTH_BLOCK_SHIFT; (blk << SYNTH_BLOCK_SHIFT) < end; blk++) {
        synth_state_t s;
        synth_block_init(&s, kind, seed, blk);
        uint64_t b0 = blk << SYNTH_BLOCK_SHIFT;
        for (uint64_t i = b0; i < b0 + SYNTH_BLOCK && i < end; i++) {
            uint8_t v = synth_block_byte(&s, m);
            if (i >= pos) out[i - pos] = v;
        }
    }
}

SYNTH_API int synth_fill_host(int kind, uint64_t seed, uint64_t pos, uint64_t len, uint8_t *out)
{
    if (kind < 0 || kind >= SYNTH_NKINDS || (len && !out)) return 1;
    if (kind == SYNTH_UNIFORM) {
        uint64_t key = synth_key(seed, SYNTH_UNIFORM, 0);
        for (uint64_t i = pos; i < pos + len; i++)
            out[i - pos] = (uint8_t)(synth_rng(key, i >> 3) >> (8 * (i & 7)));
        return 0;
    }
    synth_markov_t *m = (synth_markov_t *)malloc(sizeof(synth_markov_t));
    if (!m) return 2;
    synth_markov_build(seed, m);
    fill_seq_host(kind, seed, pos, len, out, m);
    free(m);
    return 0;
}

// ------------------------------------------------------------------ device
__global__ void synth_uniform_kernel(uint64_t key, uint64_t pos, uint64_t len, uint8_t *out)
{
    uint64_t w0 = pos >> 3, w1 = (pos + len + 7) >> 3;
    for (uint64_t w = w0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < w1;
         w += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t v = synth_rng(key, w);
        uint64_t i0 = w << 3;
        if (i0 >= pos && i0 + 8 <= pos + len && (((uintptr_t)(out + (i0 - pos))) & 7) == 0) {
            *(uint64_t *)(out + (i0 - pos)) = v;
        } else {
            for (int k = 0; k < 8; k++) {
                uint64_t i = i0 + k;
                if (i >= pos && i < pos + len) out[i - pos] = (uint8_t)(v >> (8 * k));
            }
        }
    }
}

struct MarkovParam { synth_markov_t m; };

__global__ void synth_seq_kernel(int kind, uint64_t seed, uint64_t pos, uint64_t len, uint8_t *out,
                                 const __grid_constant__ MarkovParam mp)
{
    __shared__ synth_markov_t sm;
    if (kind == SYNTH_MARKOV) {
        const uint32_t *src = (const uint32_t *)&mp.m;
        uint32_t *dst = (uint32_t *)&sm;
        for (int i = threadIdx.x; i < (int)(sizeof(synth_markov_t) / 4); i += blockDim.x) dst[i] = src[i];
        __syncthreads();
    }
    uint64_t end = pos + len;
    uint64_t blk = (pos >> SYNTH_BLOCK_SHIFT) + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if ((blk << SYNTH_BLOCK_SHIFT) >= end) return;
    synth_state_t s;
    synth_block_init(&s, kind, seed, blk);
    uint64_t b0 = blk << SYNTH_BLOCK_SHIFT;
    uint64_t b1 = b0 + SYNTH_BLOCK < end ? b0 + SYNTH_BLOCK : end;
    uint64_t i = b0;
    for (; i < pos; i++) (void)synth_block_byte(&s, &sm);        // discard bytes before pos
    uint8_t *d = out + (i - pos);
    for (; i < b1 && ((uintptr_t)d & 3); i++) *d++ = synth_block_byte(&s, &sm);
    for (; i + 4 <= b1; i += 4, d += 4) {
        uint32_t w = synth_block_byte(&s, &sm);
        w |= (uint32_t)synth_block_byte(&s, &sm) << 8;
        w |= (uint32_t)synth_block_byte(&s, &sm) << 16;
        w |= (uint32_t)synth_block_byte(&s, &sm) << 24;
        *(uint32_t *)d = w;
    }
    for (; i < b1; i++) *d++ = synth_block_byte(&s, &sm);
}

SYNTH_API int synth_fill_device(int kind, uint64_t seed, uint64_t pos, uint64_t len, uint8_t *d_out,
                                cudaStream_t stream)
{
    if (kind < 0 || kind >= SYNTH_NKINDS || (len && !d_out)) return 1;
    if (len == 0) return 0;
    if (kind == SYNTH_UNIFORM) {
        uint64_t words = ((pos + len + 7) >> 3) - (pos >> 3);
        uint64_t grid = (words + 255) / 256;
        if (grid > 148 * 64) grid = 148 * 64;
        synth_uniform_kernel<<<(unsigned)grid, 256, 0, stream>>>(synth_key(seed, SYNTH_UNIFORM, 0),
                                                                pos, len, d_out);
    } else {
        MarkovParam mp;
        memset(&mp, 0, sizeof(mp));
        if (kind == SYNTH_MARKOV) synth_markov_build(seed, &mp.m);
        uint64_t nblk = ((pos + len - 1) >> SYNTH_BLOCK_SHIFT) - (pos >> SYNTH_BLOCK_SHIFT) + 1;
        unsigned grid = (unsigned)((nblk + 63) / 64);
        synth_seq_kernel<<<grid, 64, 0, stream>>>(kind, seed, pos, len, d_out, mp);
    }
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

// ------------------------------------------------------------------ batch layout (config 3)
// Stream j: size round(mean * U[1-jit, 1+jit]) forced odd (never a multiple of 16),
// kind 50% uniform / 30% Markov / 20% zero-heavy, its own seed.
SYNTH_API int synth_batch_layout(uint64_t seed, uint32_t nstreams, uint64_t mean_size,
                                 double jitter, uint64_t *offsets, int32_t *kinds, uint64_t *seeds)
{
    uint64_t key = synth_key(seed, 99, 0);
    offsets[0] = 0;
    for (uint32_t j = 0; j < nstreams; j++) {
        double u = (double)(synth_rng(key, 3ull * j) >> 11) * (1.0 / 9007199254740992.0);
        uint64_t sz = (uint64_t)((double)mean_size * (1.0 - jitter + 2.0 * jitter * u) + 0.5);
        sz |= 1;
        uint64_t t = synth_rng(key, 3ull * j + 1) % 10;
        kinds[j] = t < 5 ? SYNTH_UNIFORM : (t < 8 ? SYNTH_MARKOV : SYNTH_ZEROHEAVY);
        seeds[j] = synth_rng(key, 3ull * j + 2);
        offsets[j + 1] = offsets[j] + sz;
    }
    return 0;
}

// ------------------------------------------------------------------ gather (config 4 versions)
// dst[dst_off .. +len) = (sel ? src1 : src0)[src_off .. +len) for every slice
// (slices: uint64[n][4] = sel, src_off, dst_off, len; each <= 64 KiB).  Pure
// byte movement: builds a version of the versioned-backup stream from the
// previous version and a pool of fresh random bytes.
__global__ void synth_gather_kernel(uint8_t *dst, const uint8_t *src0, const uint8_t *src1,
                                    const uint64_t *slices, uint64_t n)
{
    for (uint64_t i = blockIdx.x; i < n; i += gridDim.x) {
        const uint64_t *s = slices + 4 * i;
        const uint8_t *src = (s[0] ? src1 : src0) + s[1];
        uint8_t *d = dst + s[2];
        const uint64_t len = s[3];
        for (uint64_t k = threadIdx.x; k < len; k += blockDim.x) d[k] = src[k];
    }
}

SYNTH_API int synth_gather_device(uint8_t *dst, const uint8_t *src0, const uint8_t *src1,
                                  const uint64_t *d_slices, uint64_t n, cudaStream_t stream)
{
    if (n == 0) return 0;
    unsigned grid = (unsigned)(n < 148 * 16 ? n : 148 * 16);
    synth_gather_kernel<<<grid, 512, 0, stream>>>(dst, src0, src1, d_slices, n);
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
}
