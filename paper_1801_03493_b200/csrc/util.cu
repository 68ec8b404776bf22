// util.cu -- device prefix scans, the numpy pairwise-summation plan, error state.
#include <atomic>
#include <mutex>
#include <vector>

#include "fx_handles.cuh"

namespace fx {

static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};

static thread_local cudaStream_t g_cur_stream = nullptr;
cudaStream_t &cur_stream() { return g_cur_stream; }

void init_pool(int device) {
    static std::mutex mu;
    static bool done[64] = {false};
    std::lock_guard<std::mutex> lk(mu);
    if (device < 0 || device >= 64 || done[device]) return;
    cudaMemPool_t pool;
    FX_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = ~0ull;  // keep freed blocks cached in the pool
    FX_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    done[device] = true;
}

namespace {
constexpr size_t kPinBlock = 4096, kPinBlocks = 1024;
std::mutex g_pin_mu;
char *g_pin_slab = nullptr;
std::vector<int> g_pin_free;
}  // namespace

void *pinned_borrow(size_t bytes) {
    if (bytes > kPinBlock) throw Error{FX_E_INTERNAL, "pinned_borrow: block too large"};
    std::lock_guard<std::mutex> lk(g_pin_mu);
    if (!g_pin_slab) {
        FX_CUDA(cudaMallocHost((void **)&g_pin_slab, kPinBlock * kPinBlocks));
        for (int i = (int)kPinBlocks - 1; i >= 0; i--) g_pin_free.push_back(i);
    }
    if (g_pin_free.empty()) throw Error{FX_E_OOM, "pinned_borrow: slab exhausted"};
    const int i = g_pin_free.back();
    g_pin_free.pop_back();
    return g_pin_slab + (size_t)i * kPinBlock;
}

void pinned_return(void *p) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_pin_mu);
    g_pin_free.push_back((int)(((char *)p - g_pin_slab) / kPinBlock));
}

void set_error(const std::string &msg) { g_last_error = msg; }
const char *last_error() { return g_last_error.c_str(); }
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
int64_t launches() { return g_launches.load(); }

// ---------------------------------------------------------------------------
// numpy pairwise plan: leaves (<=128 elements) in order + post-order combines
// ---------------------------------------------------------------------------

static int plan_rec(PwPlan *p, int lo, int n) {
    if (n <= 128) {
        int id = p->n_leaves++;
        if (id >= kMaxLeaves) throw Error{FX_E_USAGE, "feature dimension too large for the pairwise plan"};
        p->leaf_start[id] = lo;
        p->leaf_len[id] = n;
        p->leaf_chain0[id] = p->n_chains;
        p->n_chains += n < 8 ? 1 : 8;
        return id;  // provisional leaf id (leaves are numbered in order)
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    int l = plan_rec(p, lo, n2);
    int r = plan_rec(p, lo + n2, n - n2);
    int op = p->n_ops++;
    p->op_left[op] = l;
    p->op_right[op] = r;
    return -(op + 1);  // ops encoded negative until leaves are counted
}

void build_pw_plan(int n, PwPlan *p) {
    memset(p, 0, sizeof(*p));
    p->n = n;
    if (n <= 0) {
        p->n_leaves = 0;
        return;
    }
    int root = plan_rec(p, 0, n);
    (void)root;
    // remap op operands: leaves keep ids, op k -> n_leaves + k
    for (int o = 0; o < p->n_ops; o++) {
        int l = p->op_left[o], r = p->op_right[o];
        p->op_left[o] = l >= 0 ? l : p->n_leaves + (-l - 1);
        p->op_right[o] = r >= 0 ? r : p->n_leaves + (-r - 1);
    }
}

// ---------------------------------------------------------------------------
// exclusive scans (3-phase: tile sums, single-block scan of tile sums, apply)
// ---------------------------------------------------------------------------

constexpr int SCAN_T = 1024, SCAN_ITEMS = 4, SCAN_TILE = SCAN_T * SCAN_ITEMS;

template <typename F>
__global__ void __launch_bounds__(SCAN_T) k_scan_tiles(int64_t n, F get, int64_t *__restrict__ tile_sum) {
    __shared__ int64_t ws[32];
    int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
    int64_t acc = 0;
    for (int j = 0; j < SCAN_ITEMS; j++) {
        int64_t i = base + threadIdx.x * SCAN_ITEMS + j;
        if (i < n) acc += get(i);
    }
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        int64_t v = ws[threadIdx.x];
        v = warp_sum(v);
        if (threadIdx.x == 0) tile_sum[blockIdx.x] = v;
    }
}

__global__ void __launch_bounds__(SCAN_T) k_scan_sums(int64_t nt, int64_t *__restrict__ tile_sum, int64_t *__restrict__ total) {
    __shared__ int64_t ws[32];
    __shared__ int64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t b0 = 0; b0 < nt; b0 += SCAN_T) {
        int64_t i = b0 + threadIdx.x;
        int64_t v = i < nt ? tile_sum[i] : 0;
        // inclusive warp scan
        int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        int64_t x = v;
        for (int o = 1; o < 32; o <<= 1) {
            int64_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) ws[w] = x;
        __syncthreads();
        if (w == 0) {
            int64_t s = ws[lane];
            for (int o = 1; o < 32; o <<= 1) {
                int64_t y = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += y;
            }
            ws[lane] = s;
        }
        __syncthreads();
        int64_t excl = x - v + (w ? ws[w - 1] : 0) + carry;
        if (i < nt) tile_sum[i] = excl;
        __syncthreads();
        if (threadIdx.x == SCAN_T - 1) carry = excl + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = carry;
}

template <typename F>
__global__ void __launch_bounds__(SCAN_T) k_scan_apply(int64_t n, F get, const int64_t *__restrict__ tile_sum,
                                                       int64_t *__restrict__ out) {
    __shared__ int64_t ws[32];
    int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
    int64_t v[SCAN_ITEMS];
    int64_t acc = 0;
    for (int j = 0; j < SCAN_ITEMS; j++) {
        int64_t i = base + threadIdx.x * SCAN_ITEMS + j;
        v[j] = i < n ? get(i) : 0;
        acc += v[j];
    }
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int64_t x = acc;
    for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) ws[w] = x;
    __syncthreads();
    if (w == 0) {
        int64_t s = ws[lane];
        for (int o = 1; o < 32; o <<= 1) {
            int64_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        ws[lane] = s;
    }
    __syncthreads();
    int64_t run = x - acc + (w ? ws[w - 1] : 0) + tile_sum[blockIdx.x];
    for (int j = 0; j < SCAN_ITEMS; j++) {
        int64_t i = base + threadIdx.x * SCAN_ITEMS + j;
        if (i < n) out[i] = run;
        run += v[j];
    }
}

struct GetI32 {
    const int32_t *p;
    __device__ int64_t operator()(int64_t i) const { return p[i]; }
};
struct GetU8 {
    const uint8_t *p;
    int invert;
    __device__ int64_t operator()(int64_t i) const { return invert ? (p[i] ? 0 : 1) : (p[i] ? 1 : 0); }
};

template <typename F>
static int64_t scan_generic(int64_t n, F get, int64_t *out_excl, cudaStream_t st, int64_t *d_total, bool sync) {
    if (n <= 0) {
        FX_CUDA(cudaMemsetAsync(d_total, 0, sizeof(int64_t), st));
        if (out_excl) FX_CUDA(cudaMemsetAsync(out_excl, 0, sizeof(int64_t), st));
        return 0;
    }
    const int64_t nt = cdiv(n, SCAN_TILE);
    DevBuf<int64_t> ts;
    ts.reserve(nt + 1);
    k_scan_tiles<F><<<(unsigned)nt, SCAN_T, 0, st>>>(n, get, ts.p);
    FX_LAUNCHED();
    k_scan_sums<<<1, SCAN_T, 0, st>>>(nt, ts.p, d_total);
    FX_LAUNCHED();
    k_scan_apply<F><<<(unsigned)nt, SCAN_T, 0, st>>>(n, get, ts.p, out_excl);
    FX_LAUNCHED();
    // out_excl[n] = total
    FX_CUDA(cudaMemcpyAsync(out_excl + n, d_total, sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
    int64_t h = 0;
    if (sync) {
        FX_CUDA(cudaMemcpyAsync(&h, d_total, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        FX_CUDA(cudaStreamSynchronize(st));
    }
    return h;
}

// out_excl must hold n+1 entries (out_excl[n] = total)
int64_t scan_i32_to_i64(const int32_t *in, int64_t n, int64_t *out_excl, cudaStream_t st, int64_t *d_total) {
    return scan_generic(n, GetI32{in}, out_excl, st, d_total, true);
}

void scan_u8_to_i64(const uint8_t *in, int64_t n, int invert, int64_t *out_excl, int64_t *d_total, cudaStream_t st) {
    scan_generic(n, GetU8{in, invert}, out_excl, st, d_total, false);
}

}  // namespace fx

namespace fx {
static thread_local bool t_pdl_suppressed = false;
bool pdl_enabled() {
    static const bool on = !(getenv("FOCUS_B200_NOPDL") && atoi(getenv("FOCUS_B200_NOPDL")));
    return on && !t_pdl_suppressed;
}
void pdl_suppress(bool s) { t_pdl_suppressed = s; }

// engines alive per device: several concurrent engines run without PDL and
// with the exact chain on their main stream (run_batches)
static std::atomic<int> g_live_engines[64];
int live_engines(int dev, int delta) { return g_live_engines[dev & 63].fetch_add(delta) + delta; }
}  // namespace fx
