// Launch-overhead probe: event time of empty kernels in various launch modes,
// each preceded by a memset-like kernel (as the bench's L2 flush).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void fill(unsigned *p, size_t n, unsigned v) {
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}
__global__ void __launch_bounds__(1024, 1) empty_k(int *out) {
    extern __shared__ unsigned char sm[];
    if (threadIdx.x == 0 && out) { sm[0] = 1; out[blockIdx.x] = sm[0]; }
}
int main() {
    size_t n = 64 << 20;
    unsigned *buf; cudaMalloc(&buf, n * 4);
    int *out; cudaMalloc(&out, 4096);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(empty_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int mode = 0; mode < 6; ++mode) {
        float tot = 0; int cnt = 0;
        for (int rep = 0; rep < 20; ++rep) {
            fill<<<sms * 4, 1024>>>(buf, n, rep);
            cudaEventRecord(a);
            size_t smem = (mode & 1) ? 225 * 1024 : 16;
            if (mode < 2) {
                empty_k<<<sms, 1024, smem>>>(out);
            } else if (mode < 4) {
                void *args[] = {&out};
                cudaLaunchCooperativeKernel((void *)empty_k, dim3(sms), dim3(1024), args, smem, 0);
            } else {
                empty_k<<<1, 1024, smem>>>(out);
            }
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0; cudaError_t e = cudaEventElapsedTime(&ms, a, b);
            if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) { printf("err mode %d: %s\n", mode, cudaGetErrorString(e)); return 1; }
            if (rep >= 5) { tot += ms; cnt++; }
        }
        const char *names[] = {"normal grid=SMs smem 0", "normal grid=SMs smem 225K", "coop grid=SMs smem 0",
                               "coop grid=SMs smem 225K", "normal grid=1 smem 0", "normal grid=1 smem 225K"};
        printf("%-28s %8.2f us\n", names[mode], tot / cnt * 1e3);
        fflush(stdout);
    }
    return 0;
}
