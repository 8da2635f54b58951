// KB0: pure read stream (the read-only ceiling BASELINE.md asks to report next
// to the copy-based MEASURED_PEAKS figure).  Each thread reads 16-byte words
// (non-coherent, no L1 allocation), 8 loads in flight, XOR-reduces them and
// writes one word, so the kernel moves `bytes` of HBM reads.
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) kb0_read(const uint4 *__restrict__ p, uint64_t n16, uint4 *sink) {
    uint4 acc = make_uint4(0, 0, 0, 0);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 7 * stride < n16; i += 8 * stride) {
        uint4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k)
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w)
                         : "l"(p + i + k * stride));
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            acc.x ^= v[k].x; acc.y ^= v[k].y; acc.z ^= v[k].z; acc.w ^= v[k].w;
        }
    }
    for (; i < n16; i += stride) {
        const uint4 v = p[i];
        acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
    if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x9E3779B9u) sink[blockIdx.x] = acc;  // keeps the loads
}

extern "C" int kb0_launch(const void *d, uint64_t bytes, void *d_sink, int sms, void *stream) {
    kb0_read<<<sms * 4, 512, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        reinterpret_cast<const uint4 *>(d), bytes / 16, reinterpret_cast<uint4 *>(d_sink));
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}
