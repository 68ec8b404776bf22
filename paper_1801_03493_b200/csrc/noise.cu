// noise.cu -- the cheap CNN's feature noise on the device (SURVEY.md §8f row
// 4): extract_feature (classifiers.py:152-158)
//     f' = obj.feature + sigma * default_rng([seed, oid, 1]).standard_normal(D)
// bit for bit.  numpy's pieces, restated (numpy 2.3.5, the pinned oracle
// version; tables from numpy's ziggurat_constants.h via tools/gen_ziggurat.py):
//   * SeedSequence + PCG64 XSL-RR (fx_internal.cuh pcg64_seed / pcg64_out);
//   * random_standard_normal (numpy/random/src/distributions/distributions.c):
//     256-layer ziggurat, one next_uint64 per normal on the fast path,
//     next_double uniforms on the slow paths;
//   * npy_log1p = glibc 2.39 log1p, x86_64 FMA variant (__log1p_fma, the ifunc
//     the image's CPUs select): the fdlibm algorithm with its FMA contractions
//     transcribed from the shipped machine code (tools/.. notes in DESIGN.md);
//   * exp: used only in a comparison (u-layer rejection test), decided with
//     CUDA's exp when the two sides are > 2 ulp apart, else with a double-
//     double exp whose correctly rounded value glibc returns (its error is
//     < 0.51 ulp); a case where the true value sits within 0.01 ulp of a
//     rounding midpoint is counted in *n_flagged (expected 0 per ~10^14 draws).
//
// Layout: one warp per object (grid-stride).  Lane l holds the PCG64 state of
// draw base + l; a 32-draw window is advanced with the jump (mult^32, inc *
// sum mult^i) so the 32 lanes produce 32 consecutive draws per step.  The
// ziggurat's fast path (99.3 %) is decided per lane; runs of fast draws are
// written by their lanes at once (ballot), slow draws are consumed by the
// warp in order (uniform control flow, values fetched by shuffles), so the
// number of draws each normal consumes -- and the stream position of every
// later normal -- is exactly numpy's.
#include <cmath>

#include "fx_internal.cuh"
#include "ziggurat_tables.cuh"

namespace fx {

namespace {
__constant__ U128 c_jump_a[33];  // mult^j
__constant__ U128 c_jump_g[33];  // sum_{i<j} mult^i

constexpr double kZigR = 3.6541528853610087963519472518;     // ziggurat_nor_r
constexpr double kZigInvR = 0.27366123732975827203338247596;  // ziggurat_nor_inv_r

__device__ __forceinline__ double hi_word_set(double x, uint32_t hi) {
    const uint64_t b = (uint64_t)__double_as_longlong(x);
    return __longlong_as_double((long long)(((uint64_t)hi << 32) | (b & 0xffffffffull)));
}

// glibc 2.39 __log1p_fma (sysdeps/ieee754/dbl-64/s_log1p.c built with -mfma):
// every fused multiply-add below is one vfmadd/vfnmadd/vfmsub of the shipped
// code, every other operation is a separately rounded SSE operation.
__device__ double glibc_log1p(double x) {
    const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
    const double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01, Lp3 = 2.857142874366239149e-01,
                 Lp4 = 2.222219843214978396e-01, Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
                 Lp7 = 1.479819860511658591e-01;
    const int32_t hx = (int32_t)((uint64_t)__double_as_longlong(x) >> 32);
    const int32_t ax = hx & 0x7fffffff;
    int k = 1, hu = 0;
    double f = 0.0, c = 0.0;
    if (hx < 0x3FDA827A) {
        if (ax >= 0x3ff00000) return x == -1.0 ? -INFINITY : __longlong_as_double(0x7ff8000000000000ll);
        if (ax < 0x3e200000) {
            if (ax < 0x3c900000) return x;
            return __fma_rn(-__dmul_rn(x, x), 0.5, x);
        }
        if (hx > 0 || hx <= (int32_t)0xbfd2bec3) {
            k = 0;
            f = x;
            hu = 1;
        }
    } else if (hx >= 0x7ff00000) {
        return __dadd_rn(x, x);
    }
    if (k != 0) {
        double u;
        if (hx < 0x43400000) {
            u = __dadd_rn(x, 1.0);
            hu = (int32_t)((uint64_t)__double_as_longlong(u) >> 32);
            k = (hu >> 20) - 1023;
            c = k > 0 ? __dsub_rn(1.0, __dsub_rn(u, x)) : __dsub_rn(x, __dsub_rn(u, 1.0));
            c = __ddiv_rn(c, u);
        } else {
            u = x;
            hu = (int32_t)((uint64_t)__double_as_longlong(u) >> 32);
            k = (hu >> 20) - 1023;
            c = 0.0;
        }
        hu &= 0x000fffff;
        if (hu < 0x6a09e) {
            u = hi_word_set(u, (uint32_t)hu | 0x3ff00000u);
        } else {
            k += 1;
            u = hi_word_set(u, (uint32_t)hu | 0x3fe00000u);
            hu = (0x00100000 - hu) >> 2;
        }
        f = __dsub_rn(u, 1.0);
    }
    const double kd = (double)k;
    const double hfsq = __dmul_rn(__dmul_rn(f, 0.5), f);
    if (hu == 0) {
        if (f == 0.0) {
            if (k == 0) return 0.0;
            return __fma_rn(kd, ln2_hi, __fma_rn(kd, ln2_lo, c));
        }
        const double R = __dmul_rn(__fma_rn(-f, 0.6666666666666666, 1.0), hfsq);
        if (k == 0) return __dsub_rn(f, R);
        return __fma_rn(kd, ln2_hi, -__dsub_rn(__dsub_rn(R, __fma_rn(kd, ln2_lo, c)), f));
    }
    const double s = __ddiv_rn(f, __dadd_rn(f, 2.0));
    const double z = __dmul_rn(s, s);
    const double R2 = __fma_rn(z, Lp3, Lp2), R3 = __fma_rn(z, Lp5, Lp4), R4 = __fma_rn(z, Lp7, Lp6);
    const double z2 = __dmul_rn(z, z), z4 = __dmul_rn(z2, z2), z6 = __dmul_rn(z2, z4);
    double t = __dmul_rn(z2, R2);
    t = __fma_rn(z, Lp1, t);
    t = __fma_rn(z4, R3, t);
    const double R = __fma_rn(z6, R4, t);
    const double w = __dmul_rn(__dadd_rn(R, hfsq), s);
    if (k == 0) return __dsub_rn(f, __dsub_rn(hfsq, w));
    return __fma_rn(kd, ln2_hi, -__dsub_rn(__dsub_rn(hfsq, __dadd_rn(__fma_rn(kd, ln2_lo, c), w)), f));
}

// double-double helpers (error-free transforms; explicit roundings)
struct DD {
    double hi, lo;
};
__device__ __forceinline__ DD two_sum(double a, double b) {
    const double s = __dadd_rn(a, b), bb = __dsub_rn(s, a);
    return DD{s, __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb))};
}
__device__ __forceinline__ DD quick_two_sum(double a, double b) {
    const double s = __dadd_rn(a, b);
    return DD{s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ __forceinline__ DD dd_mul(DD x, DD y) {
    const double p = __dmul_rn(x.hi, y.hi);
    double e = __fma_rn(x.hi, y.hi, -p);
    e = __dadd_rn(e, __dadd_rn(__dmul_rn(x.hi, y.lo), __dmul_rn(x.lo, y.hi)));
    return quick_two_sum(p, e);
}
__device__ __forceinline__ DD dd_add(DD x, DD y) {
    DD s = two_sum(x.hi, y.hi);
    s.lo = __dadd_rn(s.lo, __dadd_rn(x.lo, y.lo));
    return quick_two_sum(s.hi, s.lo);
}

// exp(v) to ~2^-100 relative, |v| < 700: v = k ln2 + r, exp(r) =
// (Taylor_10(r / 256))^(2^8), scaled by 2^k.
__device__ DD dd_exp(double v) {
    const double ln2_hi = 6.93147180559945286227e-01, ln2_lo = 2.31904681384629955842e-17;
    const double kd = rint(v * 1.4426950408889634);
    DD r = two_sum(v, -__dmul_rn(kd, ln2_hi));
    r.lo = __dadd_rn(r.lo, -__fma_rn(kd, ln2_hi, -__dmul_rn(kd, ln2_hi)));  // kd*ln2_hi's rounding error
    r = dd_add(r, DD{-__dmul_rn(kd, ln2_lo), -__fma_rn(kd, ln2_lo, -__dmul_rn(kd, ln2_lo))});
    const DD rs{ldexp(r.hi, -8), ldexp(r.lo, -8)};
    // Horner: 1 + rs (1 + rs/2 (1 + rs/3 (...)))
    DD acc{1.0, 0.0};
    for (int n = 10; n >= 1; n--) {
        DD q = dd_mul(acc, rs);
        // q / n in double-double
        const double qh = __ddiv_rn(q.hi, (double)n);
        const double rem = __fma_rn(-qh, (double)n, q.hi);
        const double ql = __ddiv_rn(__dadd_rn(rem, q.lo), (double)n);
        acc = dd_add(DD{1.0, 0.0}, quick_two_sum(qh, ql));
    }
    for (int i = 0; i < 8; i++) acc = dd_mul(acc, acc);
    const int k = (int)kd;
    return DD{ldexp(acc.hi, k), ldexp(acc.lo, k)};
}

// lhs < glibc exp(v)?  (distributions.c: the u-layer test of the ziggurat)
__device__ __forceinline__ bool exp_greater(double lhs, double v, unsigned long long *nflag) {
    const double e = exp(v);
    const double ulp = __dmul_rn(e, 2.220446049250313e-16);
    if (lhs < __dsub_rn(e, __dmul_rn(2.5, ulp))) return true;
    if (lhs > __dadd_rn(e, __dmul_rn(2.5, ulp))) return false;
    DD t = dd_exp(v);
    t = quick_two_sum(t.hi, t.lo);
    const double hu = __dmul_rn(fabs(t.hi), 1.1102230246251565e-16);  // half an ulp of t.hi (normal range)
    if (fabs(t.lo) > __dmul_rn(0.98, hu) && nflag) atomicAdd(nflag, 1ull);
    return lhs < t.hi;
}

__device__ __forceinline__ double f_at(const float *p, int64_t j) { return (double)p[j]; }
__device__ __forceinline__ double f_at(const double *p, int64_t j) { return p[j]; }

}  // namespace

// One warp per object; out rows are float64 (numpy promotes feature +
// float64 noise to float64).
template <typename TIn>
__global__ void __launch_bounds__(256) k_extract(int64_t n, int D, const int64_t *__restrict__ oids,
                                                 const TIn *__restrict__ fin, int64_t ld_in, double sigma,
                                                 uint64_t seed, double *__restrict__ out, int64_t ld_out,
                                                 unsigned long long *__restrict__ nflag) {
    __shared__ uint64_t ki[256];
    __shared__ double wi[256], fi[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        ki[i] = kZigKi[i];
        wi[i] = __longlong_as_double((long long)kZigWi[i]);
        fi[i] = __longlong_as_double((long long)kZigFi[i]);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const U128 al = c_jump_a[lane + 1], gl = c_jump_g[lane + 1], a32 = c_jump_a[32], g32 = c_jump_g[32];
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t obj = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); obj < n; obj += nw) {
        const TIn *frow = fin + obj * ld_in;
        double *orow = out + obj * ld_out;
        if (sigma == 0.0) {  // extract_feature returns a copy
            for (int j = lane; j < D; j += 32) orow[j] = f_at(frow, j);
            continue;
        }
        U128 s0, inc;
        pcg64_seed(seed, (uint64_t)oids[obj], 1ull, s0, inc);
        U128 st = add128(mul128(al, s0), mul128(gl, inc));  // state of draw `lane`
        const U128 c32 = mul128(g32, inc);
        int emitted = 0, state = 0, pidx = 0;
        uint64_t prabs = 0;
        double px = 0.0, pxx = 0.0;
        auto emit1 = [&](double nv) {  // one normal from the warp's slow path (lane 0 writes)
            if (lane == 0) orow[emitted] = __dadd_rn(f_at(frow, emitted), __dmul_rn(sigma, nv));
            emitted++;
        };
        while (emitted < D) {
            const uint64_t r = pcg64_out(st);
            st = add128(mul128(a32, st), c32);
            // this draw read as the first draw of a normal
            const int idx = (int)(r & 0xff);
            const uint64_t rr = r >> 8;
            const uint64_t rabs = (rr >> 1) & 0x000fffffffffffffull;
            double x = __dmul_rn((double)rabs, wi[idx]);
            if (rr & 1) x = -x;
            const bool fast = rabs < ki[idx];
            const unsigned fm = __ballot_sync(0xffffffffu, fast);
            int q = 0;
            while (q < 32 && emitted < D) {
                if (state == 0) {
                    const unsigned slow = ~fm & (0xffffffffu << q);
                    const int stop = slow ? __ffs(slow) - 1 : 32;
                    const int run = min(stop - q, D - emitted);
                    if (lane >= q && lane < q + run) {
                        const int j = emitted + lane - q;
                        orow[j] = __dadd_rn(f_at(frow, j), __dmul_rn(sigma, x));
                    }
                    emitted += run;
                    q += run;
                    if (q >= 32 || emitted >= D) break;
                    px = __shfl_sync(0xffffffffu, x, q);
                    prabs = __shfl_sync(0xffffffffu, rabs, q);
                    pidx = __shfl_sync(0xffffffffu, idx, q);
                    state = pidx == 0 ? 2 : 1;
                    q++;
                } else {
                    const uint64_t rq = __shfl_sync(0xffffffffu, r, q);
                    const double u = __dmul_rn((double)(rq >> 11), 1.0 / 9007199254740992.0);  // next_double
                    q++;
                    if (state == 1) {
                        const double lhs = __dadd_rn(__dmul_rn(__dsub_rn(fi[pidx - 1], fi[pidx]), u), fi[pidx]);
                        const double v = __dmul_rn(__dmul_rn(-0.5, px), px);
                        if (exp_greater(lhs, v, lane == 0 ? nflag : nullptr)) emit1(px);
                        state = 0;
                    } else if (state == 2) {
                        pxx = __dmul_rn(-kZigInvR, glibc_log1p(-u));
                        state = 3;
                    } else {
                        const double yy = -glibc_log1p(-u);
                        if (__dadd_rn(yy, yy) > __dmul_rn(pxx, pxx)) {
                            const double z = __dadd_rn(kZigR, pxx);
                            emit1(((prabs >> 8) & 1) ? -z : z);
                            state = 0;
                        } else {
                            state = 2;
                        }
                    }
                }
            }
        }
    }
}

namespace {
void ensure_jump_tables(int dev) {
    static bool done[64] = {};
    if (done[dev & 63]) return;
    const unsigned __int128 mult = ((unsigned __int128)0x2360ed051fc65da4ull << 64) | 0x4385df649fccf645ull;
    U128 a[33], g[33];
    unsigned __int128 pa = 1, pg = 0;
    for (int j = 0; j <= 32; j++) {
        a[j] = U128{(uint64_t)(pa >> 64), (uint64_t)pa};
        g[j] = U128{(uint64_t)(pg >> 64), (uint64_t)pg};
        pg += pa;
        pa *= mult;
    }
    FX_CUDA(cudaMemcpyToSymbol(c_jump_a, a, sizeof(a)));
    FX_CUDA(cudaMemcpyToSymbol(c_jump_g, g, sizeof(g)));
    done[dev & 63] = true;
}
}  // namespace

void launch_extract(int dev, int64_t n, int D, const int64_t *d_oid, const void *d_in, int in_type, int64_t ld_in,
                    double sigma, uint64_t seed, double *d_out, int64_t ld_out, unsigned long long *d_flag,
                    cudaStream_t st) {
    if (n <= 0) return;
    ensure_jump_tables(dev);
    const unsigned grid = (unsigned)std::min<int64_t>(cdiv(n, 8), 148 * 8);
    if (in_type == FX_F32)
        k_extract<float><<<grid, 256, 0, st>>>(n, D, d_oid, (const float *)d_in, ld_in, sigma, seed, d_out, ld_out,
                                               d_flag);
    else
        k_extract<double><<<grid, 256, 0, st>>>(n, D, d_oid, (const double *)d_in, ld_in, sigma, seed, d_out,
                                                ld_out, d_flag);
    FX_LAUNCHED();
}

}  // namespace fx

extern "C" int fx_extract_features(int32_t device, int64_t n, int32_t dim, const int64_t *object_ids,
                                   const void *feats, int32_t feat_type, double sigma, uint64_t seed, double *out,
                                   int64_t *n_flagged) {
    using namespace fx;
    try {
        if (n < 0 || dim <= 0 || (feat_type != FX_F32 && feat_type != FX_F64) || !(sigma >= 0.0))
            throw Error{FX_E_USAGE, "fx_extract_features: bad arguments"};
        if (n_flagged) *n_flagged = 0;
        if (n == 0) return FX_OK;
        FX_CUDA(cudaSetDevice(device));
        cudaStream_t st = nullptr;
        FX_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        StreamGuard sg_(st);
        const size_t es = feat_type == FX_F32 ? 4 : 8;
        {
            DevBuf<int64_t> o;
            DevBuf<char> in;
            DevBuf<double> res;
            DevBuf<unsigned long long> fl;
            o.reserve(n);
            in.reserve((size_t)n * dim * es);
            res.reserve((size_t)n * dim);
            fl.reserve(1);
            FX_CUDA(cudaMemsetAsync(fl.p, 0, sizeof(unsigned long long), st));
            FX_CUDA(cudaMemcpyAsync(o.p, object_ids, sizeof(int64_t) * n, cudaMemcpyHostToDevice, st));
            FX_CUDA(cudaMemcpyAsync(in.p, feats, (size_t)n * dim * es, cudaMemcpyHostToDevice, st));
            launch_extract(device, n, dim, o.p, in.p, feat_type, dim, sigma, seed, res.p, dim, fl.p, st);
            FX_CUDA(cudaMemcpyAsync(out, res.p, sizeof(double) * n * dim, cudaMemcpyDeviceToHost, st));
            unsigned long long h = 0;
            FX_CUDA(cudaMemcpyAsync(&h, fl.p, sizeof(h), cudaMemcpyDeviceToHost, st));
            FX_CUDA(cudaStreamSynchronize(st));
            if (n_flagged) *n_flagged = (int64_t)h;
        }
        FX_CUDA(cudaStreamSynchronize(st));
        FX_CUDA(cudaStreamDestroy(st));
    } catch (const Error &e) {
        set_error(e.msg);
        return e.code;
    }
    return FX_OK;
}

extern "C" int fx_extract_features_device(int32_t device, int64_t n, int32_t dim, const int64_t *object_ids,
                                          const void *feats, int32_t feat_type, int64_t ld_in, double sigma,
                                          uint64_t seed, double *out, int64_t ld_out, uint64_t *d_flagged,
                                          void *cuda_stream) {
    using namespace fx;
    try {
        if (n < 0 || dim <= 0 || ld_in < dim || ld_out < dim || (feat_type != FX_F32 && feat_type != FX_F64) ||
            !(sigma >= 0.0))
            throw Error{FX_E_USAGE, "fx_extract_features_device: bad arguments"};
        if (n == 0) return FX_OK;
        FX_CUDA(cudaSetDevice(device));
        launch_extract(device, n, dim, object_ids, feats, feat_type, ld_in, sigma, seed, out, ld_out,
                       (unsigned long long *)d_flagged, (cudaStream_t)cuda_stream);
    } catch (const Error &e) {
        set_error(e.msg);
        return e.code;
    }
    return FX_OK;
}
