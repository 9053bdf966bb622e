// Random fp64 atomic throughput vs working-set size (returning ATOMG vs RED).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL; z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL; return z ^ (z >> 31);
}
template <bool RET, int U>
__global__ void k(double *a, uint64_t mask, int64_t per, double *sink, int skew) {
    uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    double acc = 0;
    for (int64_t i = 0; i < per; i += U) {
        double o[U];
#pragma unroll
        for (int q = 0; q < U; q++) {
            uint64_t h = mix(t * 1000003ULL + i + q);
            uint64_t idx = h & mask;
            if (skew) idx = (idx * (h >> 40 & 0xff)) >> 8 & mask;   // skewed toward low ids
            if (RET) o[q] = atomicAdd(a + idx, 1.0); else { atomicAdd(a + idx, 1.0); o[q] = 0; }
        }
#pragma unroll
        for (int q = 0; q < U; q++) acc += o[q];
    }
    if (acc == -1.0) sink[0] = acc;
}
int main() {
    double *a, *sink; cudaMalloc(&a, 1ULL << 33); cudaMalloc(&sink, 8);
    cudaMemset(a, 0, 1ULL << 33);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int skew = 0; skew < 2; skew++)
    for (uint64_t mb : {4ULL, 16ULL, 64ULL, 256ULL, 1024ULL, 8192ULL}) {
        uint64_t n = mb * (1ULL << 20) / 8, mask = n - 1;
        int blocks = sms * 4, th = 512; int64_t per = 256;
        for (int ret = 0; ret < 2; ret++) {
            for (int rep = 0; rep < 2; rep++) {
                cudaEventRecord(e0);
                if (ret) k<true, 4><<<blocks, th>>>(a, mask, per, sink, skew);
                else k<false, 4><<<blocks, th>>>(a, mask, per, sink, skew);
                cudaEventRecord(e1); cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                if (rep) printf("skew %d  ws %6llu MB  %s  %.1f G atomics/s\n", skew, (unsigned long long)mb,
                                ret ? "ATOMG(ret)" : "RED      ", (double)blocks * th * per / ms / 1e6);
            }
        }
    }
    return 0;
}
