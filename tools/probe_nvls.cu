// probe_nvls.cu -- does this box support NVLink SHARP multicast (NVLS) for the f2 row?
// Single process, all visible GPUs: query CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, create a
// multicast object over every device, bind one physical allocation per device, map the
// multicast address, store through it with multimem.st from GPU 0 and check that every
// device's unicast view received the data; then time multimem.st vs n unicast peer stores.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/probe_nvls tools/probe_nvls.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <vector>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s; cuGetErrorString(r_, &s); \
    printf("FAIL %s: %s\n", #x, s); return 1; } } while (0)
#define CR(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("FAIL %s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

__global__ void mc_store(float* mc, int64_t nvec, float base) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nvec; q += (int64_t)gridDim.x * blockDim.x) {
        float a = base + (float)(q * 4), b = a + 1, c = a + 2, d = a + 3;
        asm volatile("multimem.st.global.v4.f32 [%0], {%1,%2,%3,%4};" :: "l"(mc + q * 4), "f"(a), "f"(b), "f"(c), "f"(d)
                     : "memory");
    }
}
__global__ void uc_store(float* const* dst, int n, int64_t nvec, float base) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nvec; q += (int64_t)gridDim.x * blockDim.x) {
        float4 v = make_float4(base + (float)(q * 4), base + (float)(q * 4 + 1), base + (float)(q * 4 + 2), base + (float)(q * 4 + 3));
        for (int k = 0; k < n; ++k) reinterpret_cast<float4*>(dst[k])[q] = v;
    }
}

int main() {
    CK(cuInit(0));
    int n = 0;
    CR(cudaGetDeviceCount(&n));
    printf("devices %d\n", n);
    for (int d = 0; d < n; ++d) {
        int mc = 0, fd = 0, fab = 0;
        CK(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d));
        CK(cuDeviceGetAttribute(&fd, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED, d));
        CK(cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, d));
        printf("dev %d multicast %d posix_fd %d fabric %d\n", d, mc, fd, fab);
        if (!mc) { printf("RESULT no-multicast\n"); return 0; }
    }
    const size_t want = 256ull << 20;
    CUmulticastObjectProp mp = {};
    mp.numDevices = n;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    mp.size = want;
    size_t gran = 0;
    CK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    const size_t size = (want + gran - 1) / gran * gran;
    mp.size = size;
    printf("mc granularity %zu size %zu\n", gran, size);
    CUmemGenericAllocationHandle mc;
    CK(cuMulticastCreate(&mc, &mp));
    for (int d = 0; d < n; ++d) CK(cuMulticastAddDevice(mc, d));
    std::vector<CUmemGenericAllocationHandle> phys(n);
    std::vector<CUdeviceptr> uc(n);
    for (int d = 0; d < n; ++d) {
        CUmemAllocationProp ap = {};
        ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
        ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        ap.location.id = d;
        ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
        CK(cuMemCreate(&phys[d], size, &ap, 0));
        CK(cuMulticastBindMem(mc, 0, phys[d], 0, size, 0));
        CK(cuMemAddressReserve(&uc[d], size, gran, 0, 0));
        CK(cuMemMap(uc[d], size, 0, phys[d], 0));
        CUmemAccessDesc ad = {};
        ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        std::vector<CUmemAccessDesc> all(n, ad);
        for (int k = 0; k < n; ++k) all[k].location.id = k;   // every device may access (peer stores)
        CK(cuMemSetAccess(uc[d], size, all.data(), n));
    }
    CUdeviceptr mcva;
    CK(cuMemAddressReserve(&mcva, size, gran, 0, 0));
    CK(cuMemMap(mcva, size, 0, mc, 0));
    {
        std::vector<CUmemAccessDesc> all(n);
        for (int k = 0; k < n; ++k) {
            all[k].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
            all[k].location.id = k;
            all[k].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        }
        CK(cuMemSetAccess(mcva, size, all.data(), n));
    }
    CR(cudaSetDevice(0));
    const int64_t nvec = size / 16;
    mc_store<<<592, 512>>>((float*)mcva, nvec, 1.0f);
    CR(cudaDeviceSynchronize());
    bool ok = true;
    for (int d = 0; d < n; ++d) {
        std::vector<float> h(4096);
        CR(cudaMemcpy(h.data(), (void*)(uc[d] + size - h.size() * 4), h.size() * 4, cudaMemcpyDefault));
        const int64_t e0 = size / 4 - 4096;
        for (int i = 0; i < 4096; ++i)
            if (h[i] != 1.0f + (float)(e0 + i)) { ok = false; printf("dev %d mismatch at %d: %f\n", d, i, h[i]); break; }
    }
    printf("multimem.st broadcast %s\n", ok ? "ok" : "WRONG");
    // timing: multimem.st (1 store/vector) vs n unicast stores over NVLink, from GPU 0
    float** dptr;
    CR(cudaMalloc(&dptr, n * sizeof(float*)));
    CR(cudaMemcpy(dptr, uc.data(), n * sizeof(float*), cudaMemcpyHostToDevice));
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int mode = 0; mode < 2; ++mode) {
        for (int w = 0; w < 3; ++w) {
            if (mode == 0) mc_store<<<592, 512>>>((float*)mcva, nvec, 2.0f);
            else uc_store<<<592, 512>>>(dptr, n, nvec, 2.0f);
        }
        cudaEventRecord(a);
        const int reps = 10;
        for (int w = 0; w < reps; ++w) {
            if (mode == 0) mc_store<<<592, 512>>>((float*)mcva, nvec, 3.0f);
            else uc_store<<<592, 512>>>(dptr, n, nvec, 3.0f);
        }
        cudaEventRecord(b);
        CR(cudaEventSynchronize(b));
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        ms /= reps;
        printf("%s: %zu MiB to %d devices in %.3f ms = %.1f GB/s egress-equivalent (bytes x (n-1) / t)\n",
               mode == 0 ? "multimem.st" : "unicast x n", size >> 20, n, ms,
               (double)size * (n - 1) / (ms * 1e-3) / 1e9);
    }
    printf("RESULT multicast-%s\n", ok ? "ok" : "wrong");
    return 0;
}
