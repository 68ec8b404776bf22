// fx_internal.cuh -- shared device helpers and handle layouts for libfocus_b200.
//
// Exactness contract: the reference computes in
// float64 with numpy's pairwise summation; every "exact" device path below
// uses __dadd_rn/__dsub_rn/__dmul_rn/__ddiv_rn/__dsqrt_rn (never contracted
// into FMA) in numpy's summation order, so results are bit-identical.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "../../include/focus_b200.h"

namespace fx {

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------

void set_error(const std::string &msg);
struct Error {
    int code;
    std::string msg;
};

#define FX_CUDA(call)                                                                        \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess)                                                               \
            throw ::fx::Error{e_ == cudaErrorMemoryAllocation ? FX_E_OOM : FX_E_CUDA,        \
                              std::string(#call) + ": " + cudaGetErrorString(e_)};           \
    } while (0)

#define FX_LAUNCHED()                                                                        \
    do {                                                                                     \
        ::fx::count_launch();                                                                \
        cudaError_t e_ = cudaGetLastError();                                                 \
        if (e_ != cudaSuccess)                                                               \
            throw ::fx::Error{FX_E_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e_)}; \
    } while (0)

void count_launch();

// cudaFuncSetAttribute applies per device: launchers remember what they set
// per device ordinal (a process may drive several GPUs)
inline int dev_slot() {
    int d = 0;
    cudaGetDevice(&d);
    return d < 0 ? 0 : (d > 63 ? 63 : d);
}

// Programmatic dependent launch for the per-batch kernel chain (screen ->
// residual columns -> row pass -> resolve -> fold -> next batch's pack):
// the next kernel is launched while this one runs, its CTAs park in
// griddepcontrol.wait until this grid has finished and flushed, so the
// launch latency between dependent kernels is hidden.  Every kernel of the
// chain calls pdl_enter() first (a no-op when launched without the attribute).
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

bool pdl_enabled();  // FOCUS_B200_NOPDL=1 turns programmatic dependent launch off (diagnostics)
void pdl_suppress(bool s);  // this host thread launches without PDL while set
int live_engines(int dev, int delta);  // engines alive on a device (after adding delta)

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args &&...args) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = grid;
    lc.blockDim = block;
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = pdl_enabled() ? 1 : 0;
    FX_CUDA(cudaLaunchKernelEx(&lc, kern, std::forward<Args>(args)...));
}

// ---------------------------------------------------------------------------
// device buffers
// ---------------------------------------------------------------------------

// Stream-ordered allocation from the device's default memory pool
// (cudaMallocAsync / cudaFreeAsync): no device-wide synchronisation on free,
// cached blocks are reused.  Every C-ABI entry point sets the stream its
// handle works on (StreamGuard); DevBuf allocates and frees on it.
cudaStream_t &cur_stream();
void init_pool(int device);
// Small pinned host blocks from a process-wide slab (cudaMallocHost pins pages
// and can stall for a long time under host memory pressure; engines are
// created and destroyed per stream, so they borrow instead).
void *pinned_borrow(size_t bytes);
void pinned_return(void *p);

struct StreamGuard {
    cudaStream_t prev;
    explicit StreamGuard(cudaStream_t s) : prev(cur_stream()) { cur_stream() = s; }
    ~StreamGuard() { cur_stream() = prev; }
};

template <typename T>
struct DevBuf {
    T *p = nullptr;
    size_t n = 0;  // capacity in elements
    DevBuf() = default;
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFreeAsync(p, cur_stream());
        p = nullptr;
        n = 0;
    }
    // ensure capacity >= want (contents NOT preserved)
    void reserve(size_t want) {
        if (want <= n && p) return;
        release();
        size_t bytes = sizeof(T) * (want ? want : 1);
        FX_CUDA(cudaMallocAsync((void **)&p, bytes, cur_stream()));
        n = want ? want : 1;
    }
    // ensure capacity >= want, preserving the first `keep` elements
    void grow(size_t want, size_t keep, cudaStream_t st) {
        if (want <= n && p) return;
        size_t cap = n ? n : 16;
        while (cap < want) cap *= 2;
        T *q = nullptr;
        FX_CUDA(cudaMallocAsync((void **)&q, sizeof(T) * cap, st));
        if (p && keep) FX_CUDA(cudaMemcpyAsync(q, p, sizeof(T) * keep, cudaMemcpyDeviceToDevice, st));
        if (p) FX_CUDA(cudaFreeAsync(p, st));
        p = q;
        n = cap;
    }
};

// ---------------------------------------------------------------------------
// numpy pairwise summation plan (loops_utils.h.src pairwise_sum, PW_BLOCKSIZE
// 128): leaves of <=128 elements + binary combine tree.  Shared by the exact
// distance (np.linalg.norm axis=1, clustering.py:77,116) and np.mean
// (ingest.py:47).
// ---------------------------------------------------------------------------

constexpr int kMaxLeaves = 256;  // D <= 16384
constexpr int kMaxChains = kMaxLeaves * 9;

struct PwPlan {
    int n;           // row length
    int n_leaves;
    int n_chains;
    int n_ops;       // combine ops (node = left + right), post-order
    int leaf_start[kMaxLeaves];
    int leaf_len[kMaxLeaves];
    int leaf_chain0[kMaxLeaves];    // first chain index of the leaf
    // chain c: sums elements start + acc, start + acc + 8, ... (len>=8: 8 chains
    // over len - len%8 elements) or the whole leaf sequentially (len<8: 1 chain)
    int op_left[kMaxLeaves], op_right[kMaxLeaves];  // node ids: <n_leaves = leaf, else op
};

void build_pw_plan(int n, PwPlan *plan);

// ---------------------------------------------------------------------------
// device-side helpers
// ---------------------------------------------------------------------------

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

template <typename T>
__device__ __forceinline__ double to_d(T x) { return (double)x; }

// numpy pairwise_sum over a generated sequence term(i), i in [lo, lo+n),
// evaluated by ONE thread (short rows: pixel signatures).  Recursion mirrors
// loops_utils.h.src pairwise_sum exactly.
template <typename F>
__device__ double pw_block_seq(int lo, int n, const F &term) {
    if (n < 8) {
        double res = 0.0;
        for (int i = 0; i < n; i++) res = dadd(res, term(lo + i));
        return res;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; j++) r[j] = term(lo + j);
        int i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] = dadd(r[j], term(lo + i + j));
        double res = dadd(dadd(dadd(r[0], r[1]), dadd(r[2], r[3])), dadd(dadd(r[4], r[5]), dadd(r[6], r[7])));
        for (; i < n; i++) res = dadd(res, term(lo + i));
        return res;
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    double a = pw_block_seq(lo, n2, term);
    double b = pw_block_seq(lo + n2, n - n2, term);
    return dadd(a, b);
}
template <typename F>
__device__ double pw_sum_seq(int n, const F &term) {
    return dadd(0.0, pw_block_seq(0, n, term));
}

// Warp-cooperative numpy pairwise sum of term(i), i in [0, plan.n), using the
// plan; `scratch` holds >= plan.n_chains + plan.n_leaves + plan.n_ops doubles
// private to the warp.  Result valid in all lanes.
template <typename F>
__device__ double pw_sum_warp(const PwPlan &plan, F term, double *scratch) {
    const int lane = threadIdx.x & 31;
    double *chain = scratch;
    double *node = scratch + plan.n_chains;  // leaves then ops
    // chains
    for (int c = lane; c < plan.n_chains; c += 32) {
        // locate leaf: leaf_chain0 is increasing; small linear search from a guess
        int lo = 0, hi = plan.n_leaves - 1;
        while (lo < hi) {
            int mid = (lo + hi + 1) >> 1;
            if (plan.leaf_chain0[mid] <= c) lo = mid; else hi = mid - 1;
        }
        const int L = lo, s = plan.leaf_start[L], len = plan.leaf_len[L];
        double r;
        if (len < 8) {
            r = 0.0;
            for (int i = 0; i < len; i++) r = dadd(r, term(s + i));
        } else {
            const int a = c - plan.leaf_chain0[L];
            const int end = len - (len % 8);
            const int nt = (end - a + 7) / 8;  // terms a, a+8, ... < end (leaves hold <= 128 elements: nt <= 16)
            if (nt <= 16) {
                // every term's loads issued before the dependent adds (same add order)
                double v[16];
#pragma unroll
                for (int t = 0; t < 16; t++) v[t] = t < nt ? term(s + a + 8 * t) : 0.0;
                r = v[0];
#pragma unroll
                for (int t = 1; t < 16; t++)
                    if (t < nt) r = dadd(r, v[t]);
            } else {
                r = term(s + a);
                for (int i = 8 + a; i < end; i += 8) r = dadd(r, term(s + i));
            }
        }
        chain[c] = r;
    }
    __syncwarp();
    for (int L = lane; L < plan.n_leaves; L += 32) {
        const int c0 = plan.leaf_chain0[L], s = plan.leaf_start[L], len = plan.leaf_len[L];
        double res;
        if (len < 8) {
            res = chain[c0];
        } else {
            const double *r = chain + c0;
            res = dadd(dadd(dadd(r[0], r[1]), dadd(r[2], r[3])), dadd(dadd(r[4], r[5]), dadd(r[6], r[7])));
            for (int i = len - (len % 8); i < len; i++) res = dadd(res, term(s + i));
        }
        node[L] = res;
    }
    __syncwarp();
    if (lane == 0) {
        for (int o = 0; o < plan.n_ops; o++)
            node[plan.n_leaves + o] = dadd(node[plan.op_left[o]], node[plan.op_right[o]]);
    }
    __syncwarp();
    double out = plan.n_ops ? node[plan.n_leaves + plan.n_ops - 1] : (plan.n_leaves ? node[0] : 0.0);
    __syncwarp();
    return dadd(0.0, out);  // add.reduce starts from the identity 0.0
}

// ---------------------------------------------------------------------------
// numpy SeedSequence (pool 4) + PCG64 XSL-RR: first Generator.random() of
// default_rng([seed, oid, word]) (classifiers.py:132-133).
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint32_t ss_hashmix(uint32_t v, uint32_t &hc) {
    v ^= hc;
    hc *= 0x931e8875u;
    v *= hc;
    v ^= v >> 16;
    return v;
}
__device__ __forceinline__ uint32_t ss_mix(uint32_t x, uint32_t y) {
    uint32_t r = 0xca01f9ddu * x - 0x4973f715u * y;
    return r ^ (r >> 16);
}

struct U128 {
    uint64_t hi, lo;
};
__device__ __forceinline__ U128 mul128(U128 a, U128 b) {
    U128 r;
    r.lo = a.lo * b.lo;
    r.hi = __umul64hi(a.lo, b.lo) + a.hi * b.lo + a.lo * b.hi;
    return r;
}
__device__ __forceinline__ U128 add128(U128 a, U128 b) {
    U128 r;
    r.lo = a.lo + b.lo;
    r.hi = a.hi + b.hi + (r.lo < a.lo ? 1 : 0);
    return r;
}

// PCG64 state after SeedSequence([a, b, c]) seeding (numpy
// _pcg64.pyx / pcg64.h pcg64_set_seed): the state BEFORE the first
// next_uint64 step.  Draw p (0-based) uses state_{p+1} = mult * state_p + inc.
__device__ __forceinline__ void pcg64_seed(uint64_t a, uint64_t b, uint64_t c, U128 &state, U128 &inc) {
    uint32_t ent[6];
    int ne = 0;
    uint64_t ints[3] = {a, b, c};
#pragma unroll
    for (int i = 0; i < 3; i++) {
        uint64_t v = ints[i];
        if (v == 0) {
            ent[ne++] = 0;
        } else {
            ent[ne++] = (uint32_t)v;
            if (v >> 32) ent[ne++] = (uint32_t)(v >> 32);
        }
    }
    uint32_t pool[4];
    uint32_t hc = 0x43b0d7e5u;
#pragma unroll
    for (int i = 0; i < 4; i++) pool[i] = ss_hashmix(i < ne ? ent[i] : 0u, hc);
#pragma unroll
    for (int s = 0; s < 4; s++)
#pragma unroll
        for (int d = 0; d < 4; d++)
            if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], hc));
    for (int s = 4; s < ne; s++)
#pragma unroll
        for (int d = 0; d < 4; d++) pool[d] = ss_mix(pool[d], ss_hashmix(ent[s], hc));
    uint32_t hb = 0x8b51f9ddu, w[8];
#pragma unroll
    for (int i = 0; i < 8; i++) {
        uint32_t v = pool[i & 3];
        v ^= hb;
        hb *= 0x58f38dedu;
        v *= hb;
        v ^= v >> 16;
        w[i] = v;
    }
    uint64_t w0 = (uint64_t)w[0] | ((uint64_t)w[1] << 32), w1 = (uint64_t)w[2] | ((uint64_t)w[3] << 32);
    uint64_t w2 = (uint64_t)w[4] | ((uint64_t)w[5] << 32), w3 = (uint64_t)w[6] | ((uint64_t)w[7] << 32);
    const U128 mult{0x2360ed051fc65da4ull, 0x4385df649fccf645ull};
    inc = U128{(w2 << 1) | (w3 >> 63), (w3 << 1) | 1ull};
    state = U128{0, 0};
    state = add128(mul128(state, mult), inc);
    state = add128(state, U128{w0, w1});
    state = add128(mul128(state, mult), inc);
}

// PCG64 XSL-RR output of a stepped state
__device__ __forceinline__ uint64_t pcg64_out(U128 st) {
    const uint64_t x = st.hi ^ st.lo;
    const unsigned rot = (unsigned)(st.hi >> 58);
    return (x >> rot) | (x << ((64 - rot) & 63));
}

// 53-bit integer of the first random() draw (random() = u53 * 2^-53)
__device__ __forceinline__ uint64_t first_u53(uint64_t a, uint64_t b, uint64_t c) {
    U128 state, inc;
    pcg64_seed(a, b, c, state, inc);
    const U128 mult{0x2360ed051fc65da4ull, 0x4385df649fccf645ull};
    state = add128(mul128(state, mult), inc);  // next_uint64 steps first
    return pcg64_out(state) >> 11;
}

// ---------------------------------------------------------------------------
// small device utilities
// ---------------------------------------------------------------------------

template <typename T>
__device__ __forceinline__ T warp_min(T v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        T w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w < v ? w : v;
    }
    return v;
}
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Error model of the snapshot screen.  SIMT mode stores the
// FP32 direct-difference distance d with |d - d_ref| <= rel*d + absc*(|c|+|f|);
// TC mode stores the TF32 GEMM-expansion value v ~ d^2 with
// |v - d_ref^2| <= g2*|c|*|f| + kap*(|c|^2 + |f|^2).
struct ScreenModel {
    int tc;
    float rel, absc, g2, kap;
};

__device__ __forceinline__ void snap_bounds(const ScreenModel &m, float v, float cn, float fn, float &lb, float &ub) {
    if (m.tc) {
        const float E = m.g2 * cn * fn + m.kap * (cn * cn + fn * fn) + 1e-30f;
        lb = sqrtf(fmaxf(v - E, 0.f)) * (1.f - 4e-7f);
        ub = sqrtf(fmaxf(v + E, 0.f)) * (1.f + 4e-7f) + 1e-30f;
    } else {
        const float e = m.rel * v + m.absc * (cn + fn) + 1e-30f;
        lb = v - e;
        ub = v + e;
    }
}

// exclusive scan of int32 flags/counts into int64 offsets (device), returns total
int64_t scan_i32_to_i64(const int32_t *in, int64_t n, int64_t *out_excl, cudaStream_t st, int64_t *scratch_total);

}  // namespace fx
