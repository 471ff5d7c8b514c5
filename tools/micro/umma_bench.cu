// Microbenchmark (tooling, not product): cycles per tcgen05.mma kind::i8 (M = 128, K = 32) for
// N = 64 / 128 / 256 on one SM, operands in shared memory (contents irrelevant), accumulator in TMEM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)32 << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)4 << 61;
    return d;
}
template <int N>
__global__ void bench(long long *out, int iters) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(s_addr(&tslot)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_addr(&bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    if (threadIdx.x == 0) {
        const uint64_t da = sdesc(s_addr(sm)), db = sdesc(s_addr(sm + 16384));
        const uint32_t m0 = 0;
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %5, %5, %5}, p;\n\t}\n" ::"r"(tmem),
                "l"(da), "l"(db), "r"(idesc), "r"(it), "r"(m0));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s_addr(&bar)) : "memory");
        uint32_t ok = 0;
        while (!ok) {
            asm volatile("{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], 0;\n\tselp.u32 %0, 1, 0, q;\n}"
                         : "=r"(ok) : "r"(s_addr(&bar)) : "memory");
        }
        long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}
template <int N>
void run() {
    long long *d, h[148];
    cudaMalloc(&d, 148 * sizeof(long long));
    const int iters = 4096;
    cudaFuncSetAttribute(bench<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    bench<N><<<148, 128, 64 * 1024>>>(d, iters);
    cudaDeviceSynchronize();
    bench<N><<<148, 128, 64 * 1024>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double cyc = (double)h[0] / iters;
    double macs = 128.0 * N * 32;
    printf("N=%d: %s, %.1f cycles per MMA (%.0f MAC/clk/SM; %.0f TOPS at 148 SMs x 1.965 GHz)\n", N,
           cudaGetErrorString(e), cyc, macs / cyc, 2 * macs / cyc * 148 * 1.965e9 / 1e12);
    cudaFree(d);
}
int main() {
    run<64>();
    run<128>();
    run<256>();
    return 0;
}
