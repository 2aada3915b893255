// Dependent-chain latency of warp primitives on this GPU (design evidence for
// the walker's per-round critical path).  nvcc -arch=sm_100a lat.cu -o lat
#include <cstdio>
#include <cstdint>
#define N 256
__global__ void k(uint32_t *out, uint32_t seed, long long *cyc)
{
    uint32_t x = seed + threadIdx.x, y = 0;
    long long t0, t1;
#define BENCH(idx, body)                                        \
    __syncwarp();                                               \
    t0 = clock64();                                             \
    _Pragma("unroll 1") for (int i = 0; i < N; i++) { body; }   \
    t1 = clock64();                                             \
    if (threadIdx.x == 0) cyc[idx] = t1 - t0;
    BENCH(0, x = x * 3u + 1u)                                   // IMAD chain
    BENCH(1, x = (x ^ 0x1234u) + 7u)                            // LOP3 + IADD
    BENCH(2, x = __shfl_sync(0xffffffffu, x, (x + 1) & 31))    // SHFL.IDX
    BENCH(3, x = __shfl_up_sync(0xffffffffu, x, 1) + 1u)       // SHFL.UP + add
    BENCH(4, x = __ballot_sync(0xffffffffu, x & 1) + x)        // VOTE + add
    BENCH(5, x = __reduce_add_sync(0xffffffffu, x) + 1u)       // REDUX
    BENCH(6, x = __popc(x) + x)                                 // POPC + add
    BENCH(7, x = __ffs(x) + x)                                  // BREV/FLO + add
    BENCH(8, x = __reduce_or_sync(0xffffffffu, x) + 1u)        // REDUX.OR
    BENCH(9, x = __funnelshift_l(x, y, x & 7) + 1u)             // SHF + add
    BENCH(10, x = __fns(x | 1u, 0, 1) + x)                      // FNS
    out[threadIdx.x] = x + y;
}
int main()
{
    uint32_t *o; long long *c, h[16];
    cudaMalloc(&o, 128 * 4); cudaMalloc(&c, 16 * 8);
    for (int r = 0; r < 2; r++) k<<<1, 32>>>(o, r, c);
    cudaMemcpy(h, c, 16 * 8, cudaMemcpyDeviceToHost);
    const char *nm[] = {"imad", "lop3+iadd", "shfl.idx", "shfl.up+add", "vote+add", "redux.sum", "popc+add", "ffs+add", "redux.or", "shf+add", "fns+add"};
    for (int i = 0; i < 11; i++) printf("%-12s %6.1f cycles/iter\n", nm[i], (double)h[i] / N);
    return 0;
}
