// Experiment helper: a rate-limited SM copy into host-mapped memory (one CTA), to test
// whether low-intensity device->host traffic interferes less with other GPU work than
// full-speed copy-engine bursts.  nvcc -shared -Xcompiler -fPIC -gencode arch=compute_100a,code=sm_100a
#include <cuda_runtime.h>
#include <stdint.h>
__global__ void trickle(const uint4* __restrict__ src, uint4* dst, int64_t nvec, int gap_ns, int chunk_vec) {
    for (int64_t base = 0; base < nvec; base += chunk_vec) {
        for (int64_t q = base + threadIdx.x; q < base + chunk_vec && q < nvec; q += blockDim.x) {
            uint4 v = src[q];
            asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(dst + q), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
        }
        __syncthreads();
        if (gap_ns > 0) {
            for (int g = gap_ns; g > 0; g -= 1000) __nanosleep(g > 1000 ? 1000 : g);
        }
        __syncthreads();
    }
}
extern "C" int launch_trickle(const void* src, void* dst, long long bytes, int gap_ns, int chunk_bytes, void* stream) {
    trickle<<<1, 256, 0, (cudaStream_t)stream>>>((const uint4*)src, (uint4*)dst, bytes / 16, gap_ns, chunk_bytes / 16);
    return (int)cudaGetLastError();
}
