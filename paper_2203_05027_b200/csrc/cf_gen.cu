// Counter-based instance generator: the device half of paper_2203_05027_b200/cfgen.py.
//
// Every draw k of stream s is H(seed, s, k) = mix(base(seed, s) + (k + 1) * golden), the
// splitmix64 finaliser over a Weyl sequence, so a thread computes its own draws with no
// state. Normals are Wichura's AS241 inverse CDF with a log built from frexp and an
// atanh series; every floating-point operation is an explicit round-to-nearest
// intrinsic (no FMA contraction), in the same order as the numpy restatement, so the
// host and device generators return bit-identical arrays (tests/test_gpu_gen.py).
// Used by bench tooling only (the large-config instances); not on the solve path.
#include "cf_common.h"

namespace cf {
namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kM1 = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t kM2 = 0x94D049BB133111EBull;
constexpr uint64_t kStreamMul = 0xD1B54A32D192ED03ull;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z ^= z >> 30;
    z *= kM1;
    z ^= z >> 27;
    z *= kM2;
    z ^= z >> 31;
    return z;
}

uint64_t stream_base(uint64_t seed, uint64_t stream) { return mix64(seed ^ (stream * kStreamMul)); }

__device__ __forceinline__ uint64_t draw(uint64_t base, int64_t k) {
    return mix64(base + (uint64_t)(k + 1) * kGolden);
}

// Horner with one rounded multiply and one rounded add per step: ((c7 r + c6) r + ...) + c0
__device__ __forceinline__ double horner8(const double* c, double r) {
    double acc = c[7];
#pragma unroll
    for (int i = 6; i >= 0; --i) acc = __dadd_rn(__dmul_rn(acc, r), c[i]);
    return acc;
}

__constant__ double kA[8] = {3.3871328727963666080e0, 1.3314166789178437745e+2, 1.9715909503065514427e+3,
                             1.3731693765509461125e+4, 4.5921953931549871457e+4, 6.7265770927008700853e+4,
                             3.3430575583588128105e+4, 2.5090809287301226727e+3};
__constant__ double kB[8] = {1.0,
                             4.2313330701600911252e+1, 6.8718700749205790830e+2, 5.3941960214247511077e+3,
                             2.1213794301586595867e+4, 3.9307895800092710610e+4, 2.8729085735721942674e+4,
                             5.2264952788528545610e+3};
__constant__ double kC[8] = {1.42343711074968357734e0, 4.63033784615654529590e0, 5.76949722146069140550e0,
                             3.64784832476320460504e0, 1.27045825245236838258e0, 2.41780725177450611770e-1,
                             2.27238449892691845833e-2, 7.74545014278341407640e-4};
__constant__ double kD[8] = {1.0,
                             2.05319162663775882187e0, 1.67638483018380384940e0, 6.89767334985100004550e-1,
                             1.48103976427480074590e-1, 1.51986665636164571966e-2, 5.47593808499534494600e-4,
                             1.05075007164441684324e-9};
__constant__ double kE[8] = {6.65790464350110377720e0, 5.46378491116411436990e0, 1.78482653991729133580e0,
                             2.96560571828504891230e-1, 2.65321895265761230930e-2, 1.24266094738807843860e-3,
                             2.71155556874348757815e-5, 2.01033439929228813265e-7};
__constant__ double kF[8] = {1.0,
                             5.99832206555887937690e-1, 1.36929880922735805310e-1, 1.48753612908506148525e-2,
                             7.86869131145613259100e-4, 1.84631831751005468180e-5, 1.42151175831644588870e-7,
                             2.04426310338993978564e-15};
// 1 / (2k + 1), k = 0..12, set from the host (the same correctly rounded quotients as cfgen.py)
__constant__ double kLogSeries[13];

__device__ __forceinline__ double det_log(double x) {
    int e = 0;
    double m = frexp(x, &e);   // exact
    if (m < 0.7071067811865476) {
        m = __dmul_rn(m, 2.0);
        e -= 1;
    }
    const double f = __dsub_rn(m, 1.0);
    const double s = __ddiv_rn(f, __dadd_rn(2.0, f));
    const double z = __dmul_rn(s, s);
    double acc = kLogSeries[12];
#pragma unroll
    for (int i = 11; i >= 0; --i) acc = __dadd_rn(__dmul_rn(acc, z), kLogSeries[i]);
    return __dadd_rn(__dmul_rn((double)e, 0.6931471805599453), __dmul_rn(__dmul_rn(2.0, s), acc));
}

__device__ __forceinline__ double normal_from_raw(uint64_t r) {
    const double p = __dmul_rn(__dadd_rn((double)(r >> 12), 0.5), 1.0 / 4503599627370496.0);
    const double q = __dsub_rn(p, 0.5);
    if (fabs(q) <= 0.425) {
        const double rr = __dsub_rn(0.180625, __dmul_rn(q, q));
        return __ddiv_rn(__dmul_rn(q, horner8(kA, rr)), horner8(kB, rr));
    }
    double rt = q < 0.0 ? p : __dsub_rn(1.0, p);
    rt = __dsqrt_rn(-det_log(rt));
    double val;
    if (rt <= 5.0) {
        const double r1 = __dsub_rn(rt, 1.6);
        val = __ddiv_rn(horner8(kC, r1), horner8(kD, r1));
    } else {
        const double r2 = __dsub_rn(rt, 5.0);
        val = __ddiv_rn(horner8(kE, r2), horner8(kF, r2));
    }
    return q < 0.0 ? -val : val;
}

__global__ void k_gen_normal(uint64_t base, int64_t start, int64_t count, double* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = normal_from_raw(draw(base, start + i));
}

__global__ void k_gen_cells(uint64_t base, int64_t start, int64_t count, uint64_t total,
                            int64_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int64_t)(draw(base, start + i) % total);
}

__global__ void k_gen_keys(uint64_t base, int64_t start, int64_t count, int64_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int64_t)(draw(base, start + i) >> 1);
}

int set_log_series() {
    static bool done = false;
    if (done) return CF_OK;
    double h[13];
    for (int k = 0; k < 13; ++k) h[k] = 1.0 / (double)(2 * k + 1);
    CF_CUDA(cudaMemcpyToSymbol(kLogSeries, h, sizeof(h)));
    done = true;
    return CF_OK;
}

dim3 gen_grid(int64_t count) {
    const int64_t blocks = (count + 255) / 256;
    return dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>(blocks, 148 * 32)));
}

}  // namespace
}  // namespace cf

using namespace cf;

extern "C" int cf_gen_normal(uint64_t seed, uint64_t stream, int64_t start, int64_t count, double* out_dev,
                             void* cuda_stream) {
    if (count < 0 || start < 0 || (count > 0 && !out_dev)) {
        set_error("cf_gen_normal: bad arguments");
        return CF_EINVAL;
    }
    if (count == 0) return CF_OK;
    CF_TRY(set_log_series());
    k_gen_normal<<<gen_grid(count), 256, 0, (cudaStream_t)cuda_stream>>>(stream_base(seed, stream), start, count,
                                                                        out_dev);
    CF_LAUNCHED();
    return CF_OK;
}

extern "C" int cf_gen_cells(uint64_t seed, int64_t start, int64_t count, int64_t total, int64_t* out_dev,
                            void* cuda_stream) {
    if (count < 0 || start < 0 || total < 1 || (count > 0 && !out_dev)) {
        set_error("cf_gen_cells: bad arguments");
        return CF_EINVAL;
    }
    if (count == 0) return CF_OK;
    k_gen_cells<<<gen_grid(count), 256, 0, (cudaStream_t)cuda_stream>>>(stream_base(seed, 0), start, count,
                                                                       (uint64_t)total, out_dev);
    CF_LAUNCHED();
    return CF_OK;
}

extern "C" int cf_gen_keys(uint64_t seed, uint64_t stream, int64_t start, int64_t count, int64_t* out_dev,
                           void* cuda_stream) {
    if (count < 0 || start < 0 || (count > 0 && !out_dev)) {
        set_error("cf_gen_keys: bad arguments");
        return CF_EINVAL;
    }
    if (count == 0) return CF_OK;
    k_gen_keys<<<gen_grid(count), 256, 0, (cudaStream_t)cuda_stream>>>(stream_base(seed, stream), start, count,
                                                                      out_dev);
    CF_LAUNCHED();
    return CF_OK;
}
