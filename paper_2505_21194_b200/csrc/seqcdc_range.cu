// seqcdc_range.cu -- the seam re-synchronisation step of the multi-GPU layer
// (include/seqcdc.h "Range calls").
//
// A stream sharded over P ranks is chunked by every rank speculatively from its
// range start (seqcdc_range_chunk, in seqcdc.cu).  Rank r's true first chunk
// starts at the overhang of rank r-1 (its first cut >= R_r), which is only
// known after an exchange.  seqcdc_range_resync re-walks rank r's chain from
// that true entry until it reaches a cut that is also in the speculative list:
// "the next cut depends only on the previous cut" (f(base)
// reads only [base, f(base)) and the stream end), so from a common cut on both
// chains are identical and the speculative suffix is reused as is.
//
// One warp walks (latency-bound; typically tens of chunks, SURVEY.md [MC-3]);
// a grid-stride kernel then appends the reused suffix.  No host sync.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "../../include/seqcdc.h"
#include "seqcdc_device.cuh"

#define SEQCDC_API extern "C" __attribute__((visibility("default")))

// internal (seqcdc.cu): the ring geometry every walker of a call uses
void seqcdc_ring_geometry(const seqcdc_params_t *p, uint32_t *bs, uint32_t *nb, uint32_t *ah);
void seqcdc_note_launches(int k);

namespace seqcdc {
namespace {

enum { ST_MERGED = 0, ST_M = 1, ST_J = 2, ST_OVERHANG = 3 };

struct ResyncArgs {
    const uint8_t *buf;
    uint64_t buf_len, stop, entry, gofs;
    const uint64_t *d_entry;  // if set: the entry as a GLOBAL offset, read on the device
    const uint64_t *skip;     // if set and *skip != 0: a merge already settled the result
    uint64_t *sum3;           // optional: [final overhang, number of cuts, *spec_ov] (k_resync_tail)
    const uint64_t *spec_ov;
    const uint64_t *spec;     // speculative cut list (global offsets, ascending)
    const uint64_t *spec_n;   // its length (device)
    uint64_t *out, *ncuts, *status;
    DevParams p;
};

struct Spec {                 // a 32-entry window of the speculative list, one entry per lane
    uint64_t j, k;            // index of window entry 0; list length
    uint32_t nv;
    uint64_t v;
};

__device__ __forceinline__ void spec_load(const ResyncArgs &a, Spec &s, int lane)
{
    s.nv = (uint32_t)(s.k - s.j < 32 ? s.k - s.j : 32);
    s.v = lane < (int)s.nv ? __ldcg(a.spec + s.j + lane) : 0;
}

// index of `cut` in the speculative list, or -1 (cuts are queried in ascending order)
__device__ __forceinline__ int64_t spec_find(const ResyncArgs &a, Spec &s, uint64_t cut, int lane)
{
#pragma unroll 1
    while (s.nv) {
        const uint64_t last = __shfl_sync(FULL, s.v, s.nv - 1);
        if (last < cut) {
            s.j += s.nv;
            spec_load(a, s, lane);
            continue;
        }
        const uint32_t hit = __ballot_sync(FULL, lane < (int)s.nv && s.v == cut);
        return hit ? (int64_t)(s.j + __ffs(hit) - 1) : -1;
    }
    return -1;
}

template <int MODE, int MSPEC>
__global__ void __launch_bounds__(32) k_resync(ResyncArgs a)
{
    __shared__ __align__(128) uint8_t ring[RING];
    const int lane = threadIdx.x;
    if (a.skip && *a.skip != 0) return;
    Walker wk;
    walker_init(wk, ring, a.p, lane);
    const uint64_t abase = (uint64_t)(uintptr_t)a.buf;
    uint64_t entry = a.entry;
    if (a.d_entry) {              // device-side entry: the predecessor's overhang (global)
        const uint64_t g = *a.d_entry;
        entry = g < a.gofs ? 0 : (g - a.gofs > a.stop ? a.stop : g - a.gofs);
    }
    if (entry >= a.stop) {        // no chunk starts in the range
        if (lane == 0) {
            *a.ncuts = 0;
            a.status[ST_MERGED] = 2;                    // 2 = empty (k_resync_tail leaves it alone)
            a.status[ST_M] = 0;
            a.status[ST_J] = 0;
            a.status[ST_OVERHANG] = a.gofs + entry;
        }
        return;
    }
    Spec sp{0, *a.spec_n, 0, 0};
    spec_load(a, sp, lane);
    uint64_t vbuf = 0;            // 32 output cuts buffered in lanes
    uint32_t m = 0;
    int64_t j = -1;
    uint64_t pos = entry, last = entry;
#pragma unroll 1
    while (pos < a.stop && j < 0) {
        uint32_t base = walker_begin(wk, abase + pos, abase + a.buf_len);
        const uint64_t off = wk.rb - abase;
        const uint32_t stop_at = base + JOB_SPAN;
#pragma unroll 1
        while (base < wk.end_rel && base < stop_at) {
            const uint32_t c = resolve<MODE, MSPEC>(wk, a.p, base, lane);
            last = off + c;
            const uint64_t g = a.gofs + last;
            if (lane == (int)(m & 31)) vbuf = g;
            m++;
            if ((m & 31) == 0) a.out[m - 32 + lane] = vbuf;
            j = spec_find(a, sp, g, lane);
            base = c;
            if (j >= 0 || last >= a.stop) break;
        }
        pos = off + base;
        if (last >= a.stop) break;
    }
    walker_finish(wk);
    const uint32_t r = m & 31;
    if (lane < (int)r) a.out[m - r + lane] = vbuf;
    if (lane == 0) {
        a.status[ST_MERGED] = j >= 0 ? 1 : 0;
        a.status[ST_M] = m;
        a.status[ST_J] = (uint64_t)j;
        a.status[ST_OVERHANG] = a.gofs + last;
    }
}

// Append the reused speculative suffix spec[j+1 .. k) after the m re-walked cuts.
__global__ void __launch_bounds__(256) k_resync_tail(ResyncArgs a)
{
    const uint64_t merged = a.status[ST_MERGED], m = a.status[ST_M];
    if (merged == 2) {                                // empty range (written by k_resync / k_merge_tail)
        if (a.sum3 && blockIdx.x == 0 && threadIdx.x == 0) {
            a.sum3[0] = a.status[ST_OVERHANG];
            a.sum3[1] = 0;
            a.sum3[2] = *a.spec_ov;
        }
        return;
    }
    const uint64_t k = *a.spec_n;
    const uint64_t j = a.status[ST_J];
    const uint64_t ns = merged ? k - (j + 1) : 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += stride)
        a.out[m + i] = __ldcg(a.spec + j + 1 + i);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *a.ncuts = m + ns;
        if (merged) a.status[ST_OVERHANG] = k ? __ldcg(a.spec + k - 1) : a.status[ST_OVERHANG];
        if (a.sum3) {
            a.sum3[0] = a.status[ST_OVERHANG];
            a.sum3[1] = m + ns;
            a.sum3[2] = *a.spec_ov;
        }
    }
}

// Rank r's local merge with rank r-1's tail: blk = [overhang, count, n, e_0 .. e_{n-1}],
// the true chain from rank r's entry (e_0 = the overhang).  The first e_i that
// is also a speculative cut of this range is a merge: the result is e_1..e_i
// followed by the speculative cuts after it (k_resync_tail).  No merge within
// the tail (or no tail) leaves status merged = 0 for the re-walk fallback.
//
// Fused-exchange form (wait_flag set): blk is this range's mailbox, filled over
// peer memory by the previous range's k_post; thread 0 first acquires the flag
// (system scope) until it reaches wait_value.  After timeout_ns without it the
// range reports itself empty with overhang ~0 (sum3 then differs from the
// speculative overhang, so the caller falls back to the collective protocol).
__global__ void __launch_bounds__(128) k_merge_tail(const uint64_t *blk, uint32_t tail_max, ResyncArgs a,
                                                    const uint64_t *wait_flag, uint64_t wait_value,
                                                    uint64_t timeout_ns)
{
    __shared__ unsigned long long best;                  // (i << 32) | j of the first merge
    __shared__ unsigned long long tcap_s;                // first tail entry at or past the range end
    __shared__ int timed_out;
    if (wait_flag) {
        if (threadIdx.x == 0) {
            uint64_t t0, t, v;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
            int to = 0;
#pragma unroll 1
            for (;;) {
                asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(wait_flag) : "memory");
                if (v >= wait_value) break;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                if (t - t0 > timeout_ns) {
                    to = 1;
                    break;
                }
                __nanosleep(500);
            }
            timed_out = to;
        }
        __syncthreads();
        if (timed_out) {
            if (threadIdx.x == 0) {
                *a.ncuts = 0;
                a.status[ST_MERGED] = 2;
                a.status[ST_M] = 0;
                a.status[ST_J] = 0;
                a.status[ST_OVERHANG] = ~0ull;
            }
            return;
        }
    }
    const uint64_t n = min(__ldcg(blk + 2), (uint64_t)tail_max);
    const uint64_t *e = blk + 3;
    const uint64_t k = *a.spec_n;
    const uint64_t ov = __ldcg(blk);
    if (threadIdx.x == 0) best = ~0ull;
    __syncthreads();
    if (ov >= a.gofs + a.stop) {                         // no chunk starts in this range
        if (threadIdx.x == 0) {
            *a.ncuts = 0;
            a.status[ST_MERGED] = 2;
            a.status[ST_M] = 0;
            a.status[ST_J] = 0;
            a.status[ST_OVERHANG] = ov;
        }
        return;
    }
    // the true chain's first cut at or past this range's end caps the search: a
    // merge found only beyond it would hand this range cuts of the next one, so
    // then the re-walk decides (and reports the changed overhang)
    if (threadIdx.x == 0) tcap_s = ~0ull;
    __syncthreads();
    for (uint64_t i = threadIdx.x; i < n; i += blockDim.x)
        if (__ldcg(e + i) >= a.gofs + a.stop) atomicMin(&tcap_s, (unsigned long long)i);
    __syncthreads();
    const uint64_t lim = min(n, (uint64_t)tcap_s + 1);
    for (uint64_t i = threadIdx.x; i < lim; i += blockDim.x) {
        const uint64_t x = __ldcg(e + i);
        uint64_t lo = 0, hi = k;                         // binary search in the ascending spec list
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (__ldcg(a.spec + mid) < x) lo = mid + 1; else hi = mid;
        }
        if (lo < k && __ldcg(a.spec + lo) == x) atomicMin(&best, ((unsigned long long)i << 32) | lo);
    }
    __syncthreads();
    const unsigned long long b = best;
    if (b == ~0ull) {
        if (threadIdx.x == 0) a.status[ST_MERGED] = 0;   // fallback: re-walk from the overhang
        return;
    }
    const uint64_t im = b >> 32, jm = b & 0xffffffffull;
    for (uint64_t t = threadIdx.x; t < im; t += blockDim.x) a.out[t] = __ldcg(e + t + 1);
    if (threadIdx.x == 0) {
        a.status[ST_MERGED] = 1;
        a.status[ST_M] = im;
        a.status[ST_J] = jm;
        a.status[ST_OVERHANG] = ov;
    }
}

__global__ void k_resync_empty(uint64_t *ncuts, uint64_t *status, uint64_t overhang)
{
    *ncuts = 0;
    status[ST_MERGED] = 1;
    status[ST_M] = 0;
    status[ST_J] = 0;
    status[ST_OVERHANG] = overhang;
}

template <int MODE, int MSPEC>
void launch(const ResyncArgs &a, cudaStream_t st)
{
    k_resync<MODE, MSPEC><<<1, 32, 0, st>>>(a);
    k_resync_tail<<<148, 256, 0, st>>>(a);
    seqcdc_note_launches(2);
}

template <int MODE>
void launch_ms(int ms, const ResyncArgs &a, cudaStream_t st)
{
    if (ms == 4) launch<MODE, 4>(a, st);
    else if (ms == 0) launch<MODE, 0>(a, st);
    else launch<MODE, -1>(a, st);
}

}  // namespace
}  // namespace seqcdc

using namespace seqcdc;

static int resync_impl(const uint8_t *d_buf, uint64_t buf_len, uint64_t range_len, uint64_t entry,
                       const uint64_t *d_entry, uint64_t global_offset, const seqcdc_params_t *p,
                       const uint64_t *d_spec, const uint64_t *d_spec_n, uint64_t *d_cuts, uint64_t *d_ncuts,
                       uint64_t *d_status, void *stream, const uint64_t *merge_blk = nullptr,
                       uint32_t tail_max = 0);
static thread_local uint64_t *g_sum3 = nullptr;          // merge_tail's optional summary outputs
static thread_local const uint64_t *g_spec_ov = nullptr;
static thread_local const uint64_t *g_wait_flag = nullptr; // merge_tail_wait: mailbox flag, value, timeout
static thread_local uint64_t g_wait_value = 0, g_wait_timeout = 0;

SEQCDC_API int seqcdc_range_merge_tail(const uint8_t *d_buf, uint64_t buf_len, uint64_t range_len,
                                       uint64_t global_offset, const seqcdc_params_t *p, const uint64_t *d_prev,
                                       uint32_t tail_max, const uint64_t *d_spec, const uint64_t *d_spec_n,
                                       uint64_t *d_cuts, uint64_t *d_ncuts, uint64_t *d_status,
                                       const uint64_t *d_spec_ov, uint64_t *d_sum3, void *stream)
{
    if (!d_prev || (d_sum3 && !d_spec_ov)) return SEQCDC_EINVAL;
    g_sum3 = d_sum3;
    g_spec_ov = d_spec_ov;
    const int rc = resync_impl(d_buf, buf_len, range_len, 0, d_prev, global_offset, p, d_spec, d_spec_n, d_cuts,
                               d_ncuts, d_status, stream, d_prev, tail_max);
    g_sum3 = nullptr;
    g_spec_ov = nullptr;
    return rc;
}

SEQCDC_API int seqcdc_range_merge_tail_wait(const uint8_t *d_buf, uint64_t buf_len, uint64_t range_len,
                                            uint64_t global_offset, const seqcdc_params_t *p,
                                            const uint64_t *d_mailbox, uint32_t tail_max, const uint64_t *d_spec,
                                            const uint64_t *d_spec_n, uint64_t *d_cuts, uint64_t *d_ncuts,
                                            uint64_t *d_status, const uint64_t *d_spec_ov, uint64_t *d_sum3,
                                            const uint64_t *d_flag, uint64_t flag_value, uint64_t timeout_ns,
                                            void *stream)
{
    if (!d_flag) return SEQCDC_EINVAL;
    g_wait_flag = d_flag;
    g_wait_value = flag_value;
    g_wait_timeout = timeout_ns;
    const int rc = seqcdc_range_merge_tail(d_buf, buf_len, range_len, global_offset, p, d_mailbox, tail_max, d_spec,
                                           d_spec_n, d_cuts, d_ncuts, d_status, d_spec_ov, d_sum3, stream);
    g_wait_flag = nullptr;
    g_wait_value = g_wait_timeout = 0;
    return rc;
}

SEQCDC_API int seqcdc_range_resync_dev(const uint8_t *d_buf, uint64_t buf_len, uint64_t range_len,
                                       const uint64_t *d_entry, uint64_t global_offset, const seqcdc_params_t *p,
                                       const uint64_t *d_spec, const uint64_t *d_spec_n, uint64_t *d_cuts,
                                       uint64_t *d_ncuts, uint64_t *d_status, void *stream)
{
    if (!d_entry) return SEQCDC_EINVAL;
    return resync_impl(d_buf, buf_len, range_len, 0, d_entry, global_offset, p, d_spec, d_spec_n, d_cuts, d_ncuts,
                       d_status, stream);
}

SEQCDC_API int seqcdc_range_resync(const uint8_t *d_buf, uint64_t buf_len, uint64_t range_len, uint64_t entry,
                                   uint64_t global_offset, const seqcdc_params_t *p, const uint64_t *d_spec,
                                   const uint64_t *d_spec_n, uint64_t *d_cuts, uint64_t *d_ncuts,
                                   uint64_t *d_status, void *stream)
{
    return resync_impl(d_buf, buf_len, range_len, entry, nullptr, global_offset, p, d_spec, d_spec_n, d_cuts,
                       d_ncuts, d_status, stream);
}

static int resync_impl(const uint8_t *d_buf, uint64_t buf_len, uint64_t range_len, uint64_t entry,
                       const uint64_t *d_entry, uint64_t global_offset, const seqcdc_params_t *p,
                       const uint64_t *d_spec, const uint64_t *d_spec_n, uint64_t *d_cuts, uint64_t *d_ncuts,
                       uint64_t *d_status, void *stream, const uint64_t *merge_blk, uint32_t tail_max)
{
    if (seqcdc_validate_params(p)) return SEQCDC_EINVAL;
    if (!d_ncuts || !d_status || !d_spec_n || range_len > buf_len || entry > range_len) return SEQCDC_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    if (!d_entry && entry >= range_len) {
        k_resync_empty<<<1, 1, 0, st>>>(d_ncuts, d_status, global_offset + entry);
        seqcdc_note_launches(1);
        return cudaGetLastError() == cudaSuccess ? SEQCDC_OK : SEQCDC_ECUDA;
    }
    if (!d_buf || !d_cuts || !d_spec) return SEQCDC_EINVAL;
    ResyncArgs a;
    memset(&a, 0, sizeof(a));
    a.buf = d_buf;
    a.buf_len = buf_len;
    a.stop = range_len;
    a.entry = entry;
    a.d_entry = d_entry;
    a.sum3 = g_sum3;
    a.spec_ov = g_spec_ov;
    a.gofs = global_offset;
    a.spec = d_spec;
    a.spec_n = d_spec_n;
    a.out = d_cuts;
    a.ncuts = d_ncuts;
    a.status = d_status;
    a.p.L = p->seq_length;
    a.p.T = p->skip_trigger;
    a.p.S = p->skip_size;
    a.p.M = p->seq_length - ((p->flags & SEQCDC_FLAG_PAIRS) ? 0u : 1u);
    a.p.mn = (uint32_t)p->min_size;
    a.p.mx = (uint32_t)p->max_size;
    a.p.mnL = (uint32_t)p->min_size - p->seq_length;
    seqcdc_ring_geometry(p, &a.p.bs, &a.p.nb, &a.p.ah);
    if (merge_blk) {              // local merge first; the re-walk runs only if it found none
        k_merge_tail<<<1, 128, 0, st>>>(merge_blk, tail_max, a, g_wait_flag, g_wait_value, g_wait_timeout);
        seqcdc_note_launches(1);
        a.skip = d_status;
    }
    const int ms = a.p.M == 4 ? 4 : (a.p.M < 4 ? 0 : -1);
    switch (p->mode | ((p->flags & SEQCDC_FLAG_SIGNED) ? 2u : 0u)) {
    case 0: launch_ms<0>(ms, a, st); break;
    case 1: launch_ms<1>(ms, a, st); break;
    case 2: launch_ms<2>(ms, a, st); break;
    default: launch_ms<3>(ms, a, st); break;
    }
    return cudaGetLastError() == cudaSuccess ? SEQCDC_OK : SEQCDC_ECUDA;
}
