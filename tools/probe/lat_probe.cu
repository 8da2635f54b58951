// Cold-load latency probe: after a 256 MiB fill (the bench's L2 flush), one
// thread does dependent loads from a cold buffer; %globaltimer deltas.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void fill(unsigned *p, size_t n, unsigned v) {
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}
__device__ __forceinline__ unsigned long long gt_after(unsigned dep) {
    unsigned x;
    asm volatile("mov.b32 %0, %1;" : "=r"(x) : "r"(dep));  // in-order issue: waits for dep
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
    return t + (x & 0);
}
__global__ void chase(const unsigned *cold, unsigned long long *out, int stride_words) {
    unsigned idx = 0;
    unsigned long long t[9];
    t[0] = gt_after(0);
    for (int k = 0; k < 8; ++k) {
        idx = *(const volatile unsigned *)(cold + idx + (unsigned)stride_words * (k + 1));  // dependent (zero buffer)
        t[k + 1] = gt_after(idx);
    }
    for (int k = 0; k < 9; ++k) out[k] = t[k];
    out[9] = idx;
}
int main() {
    size_t n = 64 << 20;
    unsigned *buf, *cold;
    cudaMalloc(&buf, n * 4);
    cudaMalloc(&cold, 512 << 20);
    cudaMemset(cold, 0, 512 << 20);
    unsigned long long *out, h[9];
    cudaMalloc(&out, 10 * 8);
    int strides[] = {32, 1 << 16, 1 << 19, 1 << 22};  // 128 B, 256 KiB, 2 MiB, 16 MiB apart
    for (int si = 0; si < 4; ++si) {
        for (int rep = 0; rep < 3; ++rep) {
            fill<<<592, 1024>>>(buf, n, rep);
            chase<<<1, 1>>>(cold, out, strides[si]);
            cudaMemcpy(h, out, 72, cudaMemcpyDeviceToHost);
            if (rep == 2) {
                printf("stride %8d words: per dependent load (ns):", strides[si]);
                for (int k = 1; k < 9; ++k) printf(" %llu", h[k] - h[k - 1]);
                printf("\n");
            }
        }
    }
    return 0;
}
