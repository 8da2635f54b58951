// Prints the shared-window address of dynamic shared memory (no static smem),
// for a few dynamic sizes: the filter addressing (scan.cu) ORs lane terms into
// addresses and needs to know which low bits of the base are zero.
#include <cstdio>
__global__ void k(unsigned *out) {
    extern __shared__ __align__(128) unsigned char sm[];
    if (threadIdx.x == 0) out[blockIdx.x] = (unsigned)__cvta_generic_to_shared(sm);
}
int main() {
    unsigned *d, h[2];
    cudaMalloc(&d, 8);
    for (int bytes : {1024, 65536, 200 * 1024, 232448}) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
        k<<<2, 32, bytes>>>(d);
        cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
        printf("dyn %d: base 0x%x 0x%x (%s)\n", bytes, h[0], h[1], cudaGetErrorString(cudaGetLastError()));
    }
    int r = 0;
    cudaDeviceGetAttribute(&r, cudaDevAttrReservedSharedMemoryPerBlock, 0);
    printf("reserved per block %d\n", r);
}
