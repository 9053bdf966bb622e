// generate.cu -- counter-based R-MAT candidate edges on the device.
//
// Bit-identical to paper_2410_21634_b200.synth.rmat_edges/permute_ids: the
// random stream is splitmix64(base ^ (edge * nchunks + chunk)), 16 bits per
// recursion level, integer thresholds.  Output is the undirected key
// min*n+max of each kept candidate, -1 for dropped ones (id >= n, self loop);
// deduplication and CSR construction happen on the device in the caller.
#include "common.cuh"

namespace gd {
namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t permute(uint64_t z, int scale, uint64_t key) {
    const uint64_t mask = (scale >= 64) ? ~0ULL : ((1ULL << scale) - 1ULL);
    const uint64_t sh = scale / 2 > 1 ? scale / 2 : 1;
    for (int rnd = 0; rnd < 3; rnd++) {
        uint64_t mult = ((key >> (rnd * 16)) & 0xFFFFULL) * 2ULL + 0x9E37ULL * 2ULL + 1ULL;
        z = (z * mult) & mask;
        z = z ^ (z >> sh);
    }
    return z;
}

__global__ void k_rmat(int scale, int64_t n, int64_t first, int64_t count, uint64_t base,
                       uint64_t pkey, uint32_t ta, uint32_t tb, uint32_t tc,
                       int64_t *__restrict__ keys) {
    const int nchunks = (scale + 3) / 4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t e = (uint64_t)(first + i);
        uint64_t u = 0, v = 0;
        for (int k = 0; k < nchunks; k++) {
            const uint64_t h = splitmix64(base ^ (e * (uint64_t)nchunks + (uint64_t)k));
            for (int q = 0; q < 4; q++) {
                const int lvl = 4 * k + q;
                if (lvl >= scale) break;
                const uint32_t f = (uint32_t)((h >> (16 * q)) & 0xFFFFULL);
                const int bit = scale - 1 - lvl;
                const uint64_t ub = f >= tb;
                const uint64_t vb = (f >= ta && f < tb) || f >= tc;
                u |= ub << bit;
                v |= vb << bit;
            }
        }
        const int64_t a = (int64_t)permute(u, scale, pkey);
        const int64_t b = (int64_t)permute(v, scale, pkey);
        keys[i] = (a < n && b < n && a != b) ? (a < b ? a * n + b : b * n + a) : -1;
    }
}

}  // namespace
}  // namespace gd

using namespace gd;

extern "C" int gd_rmat_keys_device(int32_t scale, int64_t n, int64_t first, int64_t count,
                                   uint64_t seed, double a, double b, double c, int64_t *d_keys,
                                   void *stream) {
    return guarded([&] {
        GD_CHECK_ARG(scale >= 1 && scale <= 40 && d_keys, "bad arguments");
        const uint32_t ta = (uint32_t)llround(a * 65536.0);
        const uint32_t tb = ta + (uint32_t)llround(b * 65536.0);
        const uint32_t tc = tb + (uint32_t)llround(c * 65536.0);
        const uint64_t base = seed * 0x632BE59BD9B4E019ULL;
        // key of the id permutation: splitmix64(seed ^ 0x5EED)
        uint64_t z = (seed ^ 0x5EEDULL) + 0x9E3779B97F4A7C15ULL;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        const uint64_t pkey = z ^ (z >> 31);
        int dev = 0;
        cudaGetDevice(&dev);
        k_rmat<<<8 * n_sms(dev), 256, 0, (cudaStream_t)stream>>>(scale, n, first, count, base,
                                                                 pkey, ta, tb, tc, d_keys);
        GD_LAUNCH_CHECK();
    });
}
