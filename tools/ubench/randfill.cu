// Latency of dependent random 128-B fills (8 x 16-B cp.async, wait) per thread,
// for a region of R bytes: does the latency grow with the number of 2 MB pages
// touched (TLB reach)?   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o randfill randfill.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// mode 0: cp.async 8x16 B + wait; mode 1: ld.global.v4 x1 (16 B), dependent
// local: each thread stays within its own window of `win` bytes (like a lane's segment)
__global__ void k(const uint8_t *base, uint64_t R, uint64_t win, int iters, int mode, unsigned long long *out)
{
    __shared__ __align__(16) uint8_t buf[256 * 128];
    const uint32_t tid = threadIdx.x;
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(buf + tid * 128);
    const uint64_t gid = blockIdx.x * blockDim.x + tid;
    uint64_t lo = win ? (gid * win) % (R - win) : 0, span = win ? win : R;
    uint64_t acc = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        uint64_t off = lo + ((mix(gid * 1000003ull + i + acc) % span) & ~127ull);
        if (mode == 0) {
            const uint8_t *src = base + off;
#pragma unroll
            for (int j = 0; j < 8; j++)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16 * j), "l"(src + 16 * j) : "memory");
            asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
            uint32_t v;
            asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(dst));
            acc += v & 1;
        } else {
            uint32_t a0, a1, a2, a3;
            asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3) : "l"(base + off));
            acc += (a0 ^ a3) & 1;
        }
    }
    long long t1 = clock64();
    atomicAdd(&out[0], (unsigned long long)(t1 - t0));
    atomicAdd(&out[1], (unsigned long long)iters);
    if (acc == 12345678) out[2] = acc;
}

int main(int argc, char **argv)
{
    const uint64_t maxR = 64ull << 30;
    uint8_t *d;
    if (cudaMalloc(&d, maxR) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaMemset(d, 1, maxR);
    unsigned long long *o;
    cudaMalloc(&o, 32);
    const uint64_t Rs[] = {32ull << 20, 256ull << 20, 1ull << 30, 4ull << 30, 16ull << 30, 64ull << 30};
    const int grids[] = {148, 148 * 4};
    for (int mode = 0; mode < 2; mode++)
        for (int gi = 0; gi < 2; gi++)
            for (int win = 0; win < 2; win++)
                for (uint64_t R : Rs) {
                    cudaMemset(o, 0, 32);
                    const uint64_t w = win ? (1ull << 20) : 0;
                    if (w && R <= w) continue;
                    k<<<grids[gi], 128>>>(d, R, w, 200, mode, o);
                    cudaDeviceSynchronize();
                    unsigned long long h[2];
                    cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
                    printf("{\"mode\": \"%s\", \"threads\": %d, \"window\": %llu, \"R_MiB\": %llu, \"cycles_per_fill\": %.0f}\n",
                           mode ? "ldg16" : "cp.async128", grids[gi] * 128, (unsigned long long)w,
                           (unsigned long long)(R >> 20), (double)h[0] / h[1]);
                }
    return 0;
}
