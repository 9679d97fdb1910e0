// capi.cu -- the extern "C" boundary (include/minikv_b200.h).
//
// Validates arguments with the reference's error classes, keeps an exact host
// mirror of every unit's cache state (so planning never needs a device sync),
// owns device memory, and launches the K1-K4 kernels.  No exceptions cross the
// ABI; no CPU fallback exists -- on a non-sm_100 device every compute call
// fails with MKV_ERR_UNSUPPORTED.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "mkv_kernels.h"

using namespace mkv;

namespace {

thread_local std::string g_err;

int fail(int status, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return status;
}

int cuda_fail(cudaError_t e, const char* where) {
    return fail(MKV_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

#define CK(call)                                                    \
    do {                                                            \
        cudaError_t e_ = (call);                                    \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call);         \
    } while (0)

int g_device_ok = -1;  // cached per process (single device per process)

int require_device() {
    if (g_device_ok < 0) {
        int dev = 0;
        cudaDeviceProp prop;
        if (cudaGetDevice(&dev) != cudaSuccess || cudaGetDeviceProperties(&prop, dev) != cudaSuccess) {
            g_device_ok = 0;
        } else {
            g_device_ok = (prop.major == 10 && prop.minor == 0) ? 1 : 0;
        }
    }
    if (!g_device_ok) return fail(MKV_ERR_UNSUPPORTED, "no compute-capability 10.0 (B200, sm_100a) device");
    return MKV_OK;
}

int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

// ---------------------------------------------------------------------------
// cache object
// ---------------------------------------------------------------------------
// Pinned staging buffers of page plans, kept across caches: pinning host memory costs ~1-3 ms
// per buffer, which would otherwise land on every make_cache.  A freed buffer is parked here and
// handed to the next request it fits (smallest fit); buffers are never unpinned.
struct PinnedPool {
    std::mutex mu;
    std::multimap<size_t, void*> free_;  // capacity -> buffer
};
static PinnedPool& pinned_pool() {
    static PinnedPool* p = new PinnedPool;  // leaked on purpose: outlives static caches at exit
    return *p;
}
static cudaError_t pinned_get(size_t need, void** out, size_t* cap) {
    PinnedPool& pp = pinned_pool();
    {
        std::lock_guard<std::mutex> g(pp.mu);
        auto it = pp.free_.lower_bound(need);
        if (it != pp.free_.end()) {
            *cap = it->first;
            *out = it->second;
            pp.free_.erase(it);
            return cudaSuccess;
        }
    }
    *cap = need;
    return cudaMallocHost(out, need);
}
static void pinned_put(void* p, size_t cap) {
    if (!p) return;
    PinnedPool& pp = pinned_pool();
    std::lock_guard<std::mutex> g(pp.mu);
    pp.free_.emplace(cap, p);
}

struct Plan {
    std::vector<int32_t> sig;  // per unit (pages, prefill rows) the plan was built for
    int total = 0, warps = 0, grid = 0;  // padded pages, workers (balanced ranges), CTAs
    int32_t* d_pref = nullptr;    // [n_units + 1] local page prefix, then [warps] first unit per warp
    int32_t* d_wstart = nullptr;
    UnitRec* d_rec = nullptr;     // [n_units]
    float* d_part_ml = nullptr;   // this range's page partials (slot = warp + unit), private to the plan
    float* d_part_o = nullptr;
    // Double buffer for plans prepared ahead (fused flush): after a step whose finish kernels
    // flushed residual blocks, the next plan is computed on the host and uploaded on the copy
    // stream into the other buffer; the next call that needs it waits on `ready` and swaps.
    int32_t* d_buf[2] = {nullptr, nullptr};
    int cur = 0;
    bool pending = false;
    std::vector<int32_t> pending_sig;
    int p_total = 0, p_warps = 0, p_grid = 0;
    cudaEvent_t ready = nullptr;
    void* h_stage = nullptr;      // pinned staging of the pending upload
    size_t stage_bytes = 0;
};

struct mkv_cache {
    int n_units = 0, d = 0, n_r = 0, gs = 0, max_decode = 0;
    bool shadow = false;
    // host mirror
    std::vector<int64_t> page_base;
    std::vector<int32_t> cap_pages, n_pages, n_prefill, n_res, n_blocks;
    int64_t total_pages = 0;
    // device
    UnitMeta* d_meta = nullptr;
    uint8_t* d_pool = nullptr;
    float* d_shadow = nullptr;
    __half* d_res_k = nullptr;
    __half* d_res_v = nullptr;
    uint32_t* d_status = nullptr;
    int* d_unit_cnt = nullptr;    // split finish: per-unit arrival counters (zero between calls)
    int* d_scratch_cnt = nullptr; // mkv_decode_pages_only: counts nobody reads (the counting kernel, timed alone)
    float* d_res_ml = nullptr;    // split finish: residual partial per unit
    float* d_res_o = nullptr;
    uint64_t* d_trace = nullptr;  // diagnostics only (MKV_DECODE_TRACE)
    int32_t* d_kept = nullptr;    // prefill selection scratch (grow-only: no allocation per call)
    size_t kept_cap = 0;
    uint64_t trace_seq = 0;
    int part_slots = 0;  // upper bound of page-partial slots per plan (each plan owns its buffers)
    std::unordered_map<uint64_t, Plan> plans;  // key: (unit_begin, n_units)

    cudaStream_t copy_stream = nullptr;  // async plan uploads (fused flush)
    cudaEvent_t ev_compute = nullptr;
    ~mkv_cache() {
        for (auto& kv : plans) {
            cudaFree(kv.second.d_buf[0]);
            cudaFree(kv.second.d_buf[1]);
            cudaFree(kv.second.d_part_ml);
            cudaFree(kv.second.d_part_o);
            if (kv.second.ready) cudaEventDestroy(kv.second.ready);
            pinned_put(kv.second.h_stage, kv.second.stage_bytes);
        }
        if (copy_stream) cudaStreamDestroy(copy_stream);
        if (ev_compute) cudaEventDestroy(ev_compute);
        cudaFree(d_meta); cudaFree(d_pool); cudaFree(d_shadow); cudaFree(d_res_k); cudaFree(d_res_v);
        cudaFree(d_status);
        cudaFree(d_unit_cnt); cudaFree(d_scratch_cnt); cudaFree(d_res_ml); cudaFree(d_res_o);
        cudaFree(d_trace);
        cudaFree(d_kept);
    }

    UnitMeta meta_of(int u) const {
        UnitMeta m;
        m.page_base = page_base[u];
        m.n_pages = n_pages[u];
        m.n_prefill = n_prefill[u];
        m.n_built = 0;  // (an upload restarts the block's page build: the flush builds every group)
        m.n_res = n_res[u];
        m.cap_pages = cap_pages[u];
        return m;
    }
    cudaError_t upload_meta(int ub, int n, cudaStream_t s) {
        std::vector<UnitMeta> h(n);
        for (int i = 0; i < n; ++i) h[i] = meta_of(ub + i);
        // pageable source: the copy is staged before return, so the host vector may die.
        return cudaMemcpyAsync(d_meta + ub, h.data(), sizeof(UnitMeta) * n, cudaMemcpyHostToDevice, s);
    }
};

extern "C" {

const char* mkv_last_error(void) { return g_err.c_str(); }
int mkv_abi_version(void) { return MKV_ABI_VERSION; }

int mkv_device_check(int device) {
    cudaDeviceProp prop;
    cudaError_t e = cudaGetDeviceProperties(&prop, device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceProperties");
    if (!(prop.major == 10 && prop.minor == 0))
        return fail(MKV_ERR_UNSUPPORTED, "device %d is sm_%d%d, kernels are built for sm_100a", device,
                    prop.major, prop.minor);
    return MKV_OK;
}

// ---------------------------------------------------------------------------
// host allocation helpers (selection.cpp:48-83, exact double arithmetic)
// ---------------------------------------------------------------------------
int mkv_allocate_uniform(size_t total_hh, size_t layers, int64_t* out) {
    if (layers < 1) return fail(MKV_ERR_INVALID_ARGUMENT, "allocate_uniform: layers must be >= 1");
    for (size_t i = 0; i < layers; ++i) out[i] = static_cast<int64_t>(total_hh / layers);
    for (size_t i = 0; i < total_hh % layers; ++i) ++out[i];
    return MKV_OK;
}

int mkv_allocate_pyramid(size_t mean_x, size_t layers, size_t depth, int bottom_heavy, int64_t* out) {
    if (layers < 1) return fail(MKV_ERR_INVALID_ARGUMENT, "allocate_pyramid: layers must be >= 1");
    if (depth < 1) return fail(MKV_ERR_INVALID_ARGUMENT, "allocate_pyramid: depth must be >= 1");
    const double x = static_cast<double>(mean_x);
    const double small_end = x / static_cast<double>(depth);
    const double large_end = 2.0 * x - small_end;
    const double first = bottom_heavy ? large_end : small_end;
    const double last = bottom_heavy ? small_end : large_end;
    for (size_t i = 0; i < layers; ++i) {
        const double t = (layers == 1) ? 0.0 : static_cast<double>(i) / static_cast<double>(layers - 1);
        volatile double span = (last - first) * t;  // no contraction into an FMA
        const double v = first + span;
        out[i] = static_cast<int64_t>(std::llround(std::max(v, 0.0)));
    }
    return MKV_OK;
}

int mkv_allocate_variance(const float* var, size_t layers, size_t total_hh, int inverse, int64_t* out,
                          int* uniform_fallback) {
    if (layers < 1) return fail(MKV_ERR_INVALID_ARGUMENT, "allocate_variance: no layers");
    if (!var || !out || !uniform_fallback) return fail(MKV_ERR_INVALID_ARGUMENT, "allocate_variance: null argument");
    constexpr double kEps = 1e-6;
    std::vector<double> shares(layers);
    double sum = 0.0;
    bool all_zero = true;
    for (size_t i = 0; i < layers; ++i) {
        if (var[i] < 0) return fail(MKV_ERR_INVALID_ARGUMENT, "allocate_variance: negative variance");
        if (var[i] > 0) all_zero = false;
        shares[i] = inverse ? 1.0 / (static_cast<double>(var[i]) + kEps) : static_cast<double>(var[i]);
        sum += shares[i];
    }
    *uniform_fallback = 0;
    if (all_zero && !inverse) {  // degenerate Prop: uniform allocation, flagged
        *uniform_fallback = 1;
        return mkv_allocate_uniform(total_hh, layers, out);
    }
    // largest-remainder rounding; remainder ties go to the lower layer
    std::vector<std::pair<double, size_t>> fracs(layers);
    size_t assigned = 0;
    for (size_t i = 0; i < layers; ++i) {
        const double target = static_cast<double>(total_hh) * shares[i] / sum;
        out[i] = static_cast<int64_t>(std::floor(target));
        assigned += static_cast<size_t>(out[i]);
        fracs[i] = {target - std::floor(target), i};
    }
    std::stable_sort(fracs.begin(), fracs.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
    for (size_t r = 0; assigned < total_hh; ++r, ++assigned) ++out[fracs[r % layers].second];
    return MKV_OK;
}

int mkv_score_variance(const float* a_cumul, int64_t a_stride, int n_units, int length, float* out, void* stream) {
    if (n_units < 0 || length < 0) return fail(MKV_ERR_INVALID_ARGUMENT, "layer_score_variance: bad shape");
    if (n_units == 0) return MKV_OK;
    if (length == 0) return fail(MKV_ERR_INVALID_ARGUMENT, "layer_score_variance: empty input");
    if (!a_cumul || !out || a_stride < length) return fail(MKV_ERR_INVALID_ARGUMENT, "layer_score_variance: bad tensor");
    if (int r = require_device()) return r;
    CK(launch_score_variance(a_cumul, a_stride, n_units, length, out, static_cast<cudaStream_t>(stream)));
    return MKV_OK;
}

// ---------------------------------------------------------------------------
// H2O baseline (harness.cpp:83-150)
// ---------------------------------------------------------------------------
int mkv_h2o_dynamic_baseline(const mkv_h2o_args* a, void* stream) {
    if (!a) return fail(MKV_ERR_INVALID_ARGUMENT, "h2o_dynamic_baseline: null args");
    if (a->hh_budget < 0 || a->rw_budget < 0 || a->hh_budget + a->rw_budget < 1)
        return fail(MKV_ERR_INVALID_ARGUMENT, "h2o_dynamic_baseline: budget must be >= 1");
    if (a->l_prompt < 0 || a->steps < 0 || a->d < 1) return fail(MKV_ERR_INVALID_ARGUMENT, "h2o_dynamic_baseline: bad shape");
    if (a->d > 8192) return fail(MKV_ERR_UNSUPPORTED, "h2o_dynamic_baseline: d %d > 8192 (query staged in shared memory)", a->d);
    const int64_t total = (int64_t)a->l_prompt + a->steps;
    if (total > INT32_MAX / 2 || a->hh_budget + a->rw_budget > INT32_MAX)
        return fail(MKV_ERR_INVALID_ARGUMENT, "h2o_dynamic_baseline: too long");
    const int64_t need = std::min<int64_t>(total, a->hh_budget + a->rw_budget);
    if (a->kept_stride < need || !a->kept || !a->kept_count)
        return fail(MKV_ERR_INVALID_ARGUMENT, "h2o_dynamic_baseline: kept buffer stride %lld < %lld",
                    (long long)a->kept_stride, (long long)need);
    if ((a->l_prompt > 0 && (!a->prompt_k || !a->prompt_scores || a->ld_k < a->d)) || (a->steps > 0 && (!a->qs || !a->ks)))
        return fail(MKV_ERR_INVALID_ARGUMENT, "h2o_dynamic_baseline: null tensor");
    if (int r = require_device()) return r;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t n = (size_t)std::max<int64_t>(total, 1);
    void* ws = nullptr;
    CK(cudaMallocAsync(&ws, n * (sizeof(double) + sizeof(int) + sizeof(float)), s));
    H2OParams p;
    p.prompt_k = a->prompt_k; p.ld_k = a->ld_k; p.prompt_scores = a->prompt_scores;
    p.qs = a->qs; p.ks = a->ks; p.l_prompt = a->l_prompt; p.d = a->d; p.steps = a->steps;
    p.hh_budget = (int)a->hh_budget; p.rw_budget = (int)std::min<int64_t>(a->rw_budget, INT32_MAX);
    p.scale = a->scale; p.kept = a->kept; p.kept_stride = a->kept_stride; p.kept_count = a->kept_count;
    p.ws_score = static_cast<double*>(ws);
    p.ws_pos = reinterpret_cast<int*>(p.ws_score + n);
    p.ws_attn = reinterpret_cast<float*>(p.ws_pos + n);
    const cudaError_t e = launch_h2o(p, s);
    cudaFreeAsync(ws, s);
    CK(e);
    return MKV_OK;
}

// ---------------------------------------------------------------------------
// K1 prefill attention
// ---------------------------------------------------------------------------
int mkv_prefill_attn(const mkv_prefill_args* a, void* stream) {
    if (!a) return fail(MKV_ERR_INVALID_ARGUMENT, "attention: null args");
    if (a->len_q <= 0 || a->len_k <= 0) return fail(MKV_ERR_INVALID_ARGUMENT, "attention: zero-length sequence");
    if (a->causal && a->len_q > a->len_k)
        return fail(MKV_ERR_INVALID_ARGUMENT, "attention: causal requires l_query <= l_key");
    if (a->head_dim != 128) return fail(MKV_ERR_UNSUPPORTED, "attention: head_dim %d (device kernel: 128)", a->head_dim);
    if (a->batch <= 0 || a->n_q_heads <= 0 || a->n_kv_heads <= 0 || a->n_q_heads % a->n_kv_heads)
        return fail(MKV_ERR_INVALID_ARGUMENT, "attention: bad head counts (Hq %d, Hkv %d)", a->n_q_heads, a->n_kv_heads);
    if (!a->q || !a->k || !a->v || !a->out || !a->lse || !a->a_cumul)
        return fail(MKV_ERR_INVALID_ARGUMENT, "attention: null tensor");
    if (!aligned16(a->q) || !aligned16(a->k) || !aligned16(a->v) || !aligned16(a->out) ||
        (a->q_st % 8) || (a->k_st % 8) || (a->v_st % 8) || (a->o_st % 8) || (a->q_sh % 8) ||
        (a->k_sh % 8) || (a->v_sh % 8) || (a->o_sh % 8) || (a->q_sb % 8) || (a->k_sb % 8) ||
        (a->v_sb % 8) || (a->o_sb % 8))
        return fail(MKV_ERR_INVALID_ARGUMENT, "attention: rows must be 16-byte aligned");
    if (int r = require_device()) return r;
    PrefillAttnParams p;
    p.q = static_cast<const __half*>(a->q); p.q_sb = a->q_sb; p.q_sh = a->q_sh; p.q_st = a->q_st;
    p.k = static_cast<const __half*>(a->k); p.k_sb = a->k_sb; p.k_sh = a->k_sh; p.k_st = a->k_st;
    p.v = static_cast<const __half*>(a->v); p.v_sb = a->v_sb; p.v_sh = a->v_sh; p.v_st = a->v_st;
    p.out = static_cast<__half*>(a->out); p.o_sb = a->o_sb; p.o_sh = a->o_sh; p.o_st = a->o_st;
    p.lse = a->lse; p.a_cumul = a->a_cumul;
    p.batch = a->batch; p.hq = a->n_q_heads; p.hkv = a->n_kv_heads; p.lq = a->len_q; p.lk = a->len_k;
    p.scale = a->scale; p.causal = a->causal;
    CK(launch_prefill_attn(p, static_cast<cudaStream_t>(stream)));
    return MKV_OK;
}

// ---------------------------------------------------------------------------
// K2 selection
// ---------------------------------------------------------------------------
static int do_select(const float* a_cumul, int64_t a_stride, int n_units, int length, const int32_t* hh_host,
                     int rw, int32_t* kept, int64_t kept_stride, int32_t* n_kept, cudaStream_t s) {
    // one budget for every unit (the common case) travels as a kernel argument: no
    // host->device copy (a pageable copy would serialise the host with the stream)
    bool uniform = true;
    for (int i = 1; i < n_units; ++i) uniform &= hh_host[i] == hh_host[0];
    int32_t* d_hh = nullptr;
    if (!uniform) {
        CK(cudaMallocAsync(&d_hh, sizeof(int32_t) * n_units, s));
        CK(cudaMemcpyAsync(d_hh, hh_host, sizeof(int32_t) * n_units, cudaMemcpyHostToDevice, s));
    }
    SelectParams p{a_cumul, a_stride, n_units, length, d_hh, uniform ? hh_host[0] : 0, rw, kept, kept_stride, n_kept};
    cudaError_t e = launch_select(p, s);
    if (d_hh) cudaFreeAsync(d_hh, s);
    if (e != cudaSuccess) return cuda_fail(e, "select kernel");
    return MKV_OK;
}

int mkv_select(const mkv_select_args* a, void* stream) {
    if (!a) return fail(MKV_ERR_INVALID_ARGUMENT, "select: null args");
    if (a->n_units < 0 || a->length < 0 || a->rw_count < 0 || !a->hh_count)
        return fail(MKV_ERR_INVALID_ARGUMENT, "select: negative budget");
    for (int u = 0; u < a->n_units; ++u)
        if (a->hh_count[u] < 0) return fail(MKV_ERR_INVALID_ARGUMENT, "select_tokens: negative budget");
    if (a->n_units == 0) return MKV_OK;
    if (!a->a_cumul || !a->kept) return fail(MKV_ERR_INVALID_ARGUMENT, "select: null tensor");
    // every unit writes min(hh[u] + rw, L) indices at kept + u * kept_stride
    int64_t need = 0;
    for (int u = 0; u < a->n_units; ++u)
        need = std::max<int64_t>(need, std::min<int64_t>((int64_t)a->hh_count[u] + a->rw_count, a->length));
    if (a->kept_stride < std::max<int64_t>(need, 1))
        return fail(MKV_ERR_INVALID_ARGUMENT, "select: kept_stride %lld < max kept %lld", (long long)a->kept_stride,
                    (long long)need);
    if (int r = require_device()) return r;
    return do_select(a->a_cumul, a->a_stride, a->n_units, a->length, a->hh_count, a->rw_count, a->kept,
                     a->kept_stride, a->n_kept, static_cast<cudaStream_t>(stream));
}

// ---------------------------------------------------------------------------
// cache lifecycle
// ---------------------------------------------------------------------------
static int plan_reserve(mkv_cache* c, int ub, int n);

int mkv_cache_create(const mkv_cache_config* cfg, mkv_cache** out) {
    if (!cfg || !out) return fail(MKV_ERR_INVALID_ARGUMENT, "make_cache: null argument");
    if (cfg->head_dim < 1) return fail(MKV_ERR_INVALID_ARGUMENT, "make_cache: d must be >= 1");
    if (cfg->group_size < 1 || cfg->n_r <= 0 || cfg->n_r % cfg->group_size != 0)
        return fail(MKV_ERR_INVALID_ARGUMENT, "make_cache: n_r must be a positive multiple of group_size");
    if (cfg->head_dim != kHeadDim) return fail(MKV_ERR_UNSUPPORTED, "make_cache: head_dim %d (device cache: 128)", cfg->head_dim);
    if (cfg->group_size != kGroup) return fail(MKV_ERR_UNSUPPORTED, "make_cache: group_size %d (device cache: 16)", cfg->group_size);
    if (cfg->n_r > 128) return fail(MKV_ERR_UNSUPPORTED, "make_cache: n_r %d > 128", cfg->n_r);
    if (cfg->n_units <= 0 || !cfg->prefill_capacity || cfg->max_decode_tokens < 0)
        return fail(MKV_ERR_INVALID_ARGUMENT, "make_cache: bad unit configuration");
    if (int r = require_device()) return r;
    auto* c = new mkv_cache;
    c->n_units = cfg->n_units;
    c->d = cfg->head_dim;
    c->n_r = cfg->n_r;
    c->gs = cfg->group_size;
    c->max_decode = cfg->max_decode_tokens;
    c->shadow = cfg->keep_fp32_params != 0;
    const int n = c->n_units;
    c->page_base.resize(n);
    c->cap_pages.resize(n);
    c->n_pages.assign(n, 0);
    c->n_prefill.assign(n, 0);
    c->n_res.assign(n, 0);
    c->n_blocks.assign(n, 0);
    const int flush_pages = ((cfg->max_decode_tokens + c->n_r - 1) / c->n_r) * (c->n_r / kGroup);
    int64_t acc = 0;
    for (int u = 0; u < n; ++u) {
        if (cfg->prefill_capacity[u] < 0) {
            delete c;
            return fail(MKV_ERR_INVALID_ARGUMENT, "make_cache: negative capacity");
        }
        c->page_base[u] = acc;
        c->cap_pages[u] = (cfg->prefill_capacity[u] + kGroup - 1) / kGroup + flush_pages;
        acc += c->cap_pages[u];
    }
    c->total_pages = acc;
    c->part_slots = num_sms() * kMaxPagesWarps + n;
    auto al = [&](void** p, size_t bytes) -> cudaError_t { return cudaMalloc(p, std::max<size_t>(bytes, 16)); };
    cudaError_t e = cudaSuccess;
    if (e == cudaSuccess) e = al((void**)&c->d_meta, sizeof(UnitMeta) * n);
    if (e == cudaSuccess) e = al((void**)&c->d_pool, (size_t)acc * kPageBytes);
    if (e == cudaSuccess && c->shadow) e = al((void**)&c->d_shadow, (size_t)acc * kShadowBytes);
    if (e == cudaSuccess) e = al((void**)&c->d_res_k, (size_t)n * c->n_r * c->d * sizeof(__half));
    if (e == cudaSuccess) e = al((void**)&c->d_res_v, (size_t)n * c->n_r * c->d * sizeof(__half));
    if (e == cudaSuccess) e = al((void**)&c->d_status, sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMemset(c->d_status, 0, sizeof(uint32_t));
    if (e == cudaSuccess) e = al((void**)&c->d_unit_cnt, sizeof(int) * n);
    if (e == cudaSuccess) e = cudaMemset(c->d_unit_cnt, 0, sizeof(int) * std::max(n, 1));
    if (e == cudaSuccess) e = al((void**)&c->d_scratch_cnt, sizeof(int) * n);
    if (e == cudaSuccess) e = cudaMemset(c->d_scratch_cnt, 0, sizeof(int) * std::max(n, 1));
    if (e == cudaSuccess) e = al((void**)&c->d_res_ml, sizeof(float) * 2 * kMaxG * n);
    if (e == cudaSuccess) e = al((void**)&c->d_res_o, sizeof(float) * kMaxG * c->d * n);
    if (e == cudaSuccess) e = cudaMemset(c->d_pool, 0, (size_t)acc * kPageBytes);
    if (e == cudaSuccess) e = c->upload_meta(0, n, 0);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        delete c;
        return cuda_fail(e, "make_cache: device allocation");
    }
    // the page plan of a call over every unit (the usual decode call) is allocated with the pool:
    // its device buffers, partial slots and pinned staging buffer otherwise cost the first decode
    // step after a prefill ~3 ms of host time (cudaMalloc / cudaMallocHost)
    static const bool reserve = [] {
        const char* e = getenv("MKV_PLAN_RESERVE");
        return !(e && e[0] == '0');
    }();
    if (reserve)
        if (int r = plan_reserve(c, 0, n)) {
            delete c;
            return r;
        }
    *out = c;
    return MKV_OK;
}

int mkv_cache_destroy(mkv_cache* c) {
    if (c) {
        cudaDeviceSynchronize();
        delete c;
    }
    return MKV_OK;
}

int mkv_cache_bytes(const mkv_cache* c, uint64_t* page_bytes, uint64_t* residual_bytes, uint64_t* total) {
    if (!c) return fail(MKV_ERR_INVALID_ARGUMENT, "cache: null handle");
    const uint64_t pb = (uint64_t)c->total_pages * kPageBytes;
    const uint64_t rb = (uint64_t)c->n_units * c->n_r * c->d * 2 * 2;
    if (page_bytes) *page_bytes = pb;
    if (residual_bytes) *residual_bytes = rb;
    if (total) *total = pb + rb + (c->shadow ? (uint64_t)c->total_pages * kShadowBytes : 0) +
                        (uint64_t)c->plans.size() * c->part_slots * kMaxG * (kHeadDim + 2) * 4;
    return MKV_OK;
}

int mkv_cache_unit_info(const mkv_cache* c, int u, int64_t* tq, int64_t* tr, int64_t* np, int64_t* nb) {
    if (!c) return fail(MKV_ERR_INVALID_ARGUMENT, "cache: null handle");
    if (u < 0 || u >= c->n_units) return fail(MKV_ERR_OUT_OF_RANGE, "cache: unit %d out of range", u);
    if (tq) *tq = c->n_prefill[u] + (int64_t)(c->n_blocks[u] - (c->n_prefill[u] > 0 ? 1 : 0)) * c->n_r;
    if (tr) *tr = c->n_res[u];
    if (np) *np = c->n_pages[u];
    if (nb) *nb = c->n_blocks[u];
    return MKV_OK;
}

static int check_range(const mkv_cache* c, int ub, int n) {
    if (!c) return fail(MKV_ERR_INVALID_ARGUMENT, "cache: null handle");
    if (ub < 0 || n < 0 || ub + n > c->n_units)
        return fail(MKV_ERR_OUT_OF_RANGE, "cache: units [%d, %d) outside [0, %d)", ub, ub + n, c->n_units);
    return MKV_OK;
}

// ---------------------------------------------------------------------------
// K3 prefill quantize + pack
// ---------------------------------------------------------------------------
static int prefill_pages_impl(mkv_cache* c, int ub, int n, const void* k, int64_t k_su, int64_t k_st,
                              const void* v, int64_t v_su, int64_t v_st, const int32_t* kept,
                              int64_t kept_stride, const int32_t* n_kept, cudaStream_t s) {
    int max_pages = 0;
    for (int i = 0; i < n; ++i) {
        const int u = ub + i;
        if (n_kept[i] <= 0) return fail(MKV_ERR_INVALID_ARGUMENT, "append_block: empty block (unit %d)", u);
        const int pages = (n_kept[i] + kGroup - 1) / kGroup;
        if (pages > c->cap_pages[u])
            return fail(MKV_ERR_OUT_OF_RANGE, "prefill: unit %d keeps %d tokens > capacity", u, n_kept[i]);
        max_pages = std::max(max_pages, pages);
    }
    for (int i = 0; i < n; ++i) {  // make_cache + store_block (cache_engine.cpp:70-74)
        const int u = ub + i;
        c->n_prefill[u] = n_kept[i];
        c->n_pages[u] = (n_kept[i] + kGroup - 1) / kGroup;
        c->n_res[u] = 0;
        c->n_blocks[u] = 1;
    }
    CK(c->upload_meta(ub, n, s));
    PrefillPagesParams p;
    p.k = static_cast<const __half*>(k); p.k_su = k_su; p.k_st = k_st;
    p.v = static_cast<const __half*>(v); p.v_su = v_su; p.v_st = v_st;
    p.kept = kept; p.kept_stride = kept_stride;
    p.meta = c->d_meta; p.unit_begin = ub; p.n_units = n; p.max_pages = max_pages;
    p.pool = c->d_pool; p.shadow = c->d_shadow; p.status = c->d_status;
    CK(launch_prefill_pages(p, s));
    return MKV_OK;
}

int mkv_cache_prefill(mkv_cache* c, const mkv_cache_prefill_args* a, void* stream) {
    if (!a) return fail(MKV_ERR_INVALID_ARGUMENT, "prefill: null args");
    if (int r = check_range(c, a->unit_begin, a->n_units)) return r;
    if (a->n_units == 0) return MKV_OK;
    if (!a->k || !a->v || !a->kept || !a->n_kept_host) return fail(MKV_ERR_INVALID_ARGUMENT, "prefill: null tensor");
    if (!aligned16(a->k) || !aligned16(a->v) || (a->k_st % 8) || (a->v_st % 8) || (a->k_su % 8) || (a->v_su % 8))
        return fail(MKV_ERR_INVALID_ARGUMENT, "prefill: K/V rows must be 16-byte aligned");
    if (int r = require_device()) return r;
    return prefill_pages_impl(c, a->unit_begin, a->n_units, a->k, a->k_su, a->k_st, a->v, a->v_su, a->v_st,
                              a->kept, a->kept_stride, a->n_kept_host, static_cast<cudaStream_t>(stream));
}

int mkv_cache_prefill_select(mkv_cache* c, const mkv_prefill_select_args* a, void* stream) {
    if (!a) return fail(MKV_ERR_INVALID_ARGUMENT, "prefill: null args");
    if (int r = check_range(c, a->unit_begin, a->n_units)) return r;
    if (a->n_units == 0) return MKV_OK;
    if (!a->a_cumul || !a->k || !a->v || !a->hh_count) return fail(MKV_ERR_INVALID_ARGUMENT, "prefill: null tensor");
    if (a->length < 0 || a->rw_count < 0) return fail(MKV_ERR_INVALID_ARGUMENT, "prefill: k/v/a_cumul length mismatch");
    std::vector<int32_t> n_kept(a->n_units);
    for (int i = 0; i < a->n_units; ++i) {
        if (a->hh_count[i] < 0) return fail(MKV_ERR_INVALID_ARGUMENT, "prefill: negative budget");
        if ((int64_t)a->hh_count[i] + a->rw_count == 0) return fail(MKV_ERR_RUNTIME, "prefill: zero kept tokens");
        n_kept[i] = (int32_t)std::min<int64_t>((int64_t)a->hh_count[i] + a->rw_count, a->length);
    }
    if (!aligned16(a->k) || !aligned16(a->v) || (a->k_st % 8) || (a->v_st % 8) || (a->k_su % 8) || (a->v_su % 8))
        return fail(MKV_ERR_INVALID_ARGUMENT, "prefill: K/V rows must be 16-byte aligned");
    if (int r = require_device()) return r;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t ks = std::max(a->length, 1);
    const size_t need = (size_t)ks * a->n_units;
    if (need > c->kept_cap) {  // grow-only scratch (cudaFree synchronizes: earlier users are done)
        cudaFree(c->d_kept);
        c->d_kept = nullptr;
        c->kept_cap = 0;
        CK(cudaMalloc(&c->d_kept, sizeof(int32_t) * need));
        c->kept_cap = need;
    }
    int32_t* kept = c->d_kept;
    int r = do_select(a->a_cumul, a->a_stride, a->n_units, a->length, a->hh_count, a->rw_count, kept, ks,
                      nullptr, s);
    if (r == MKV_OK)
        r = prefill_pages_impl(c, a->unit_begin, a->n_units, a->k, a->k_su, a->k_st, a->v, a->v_su, a->v_st, kept,
                               ks, n_kept.data(), s);
    return r;
}

// ---------------------------------------------------------------------------
// K4 decode
// ---------------------------------------------------------------------------
// The plan depends on every unit's page count and prefill rows (its partial last page);
// it is reused while that signature is unchanged (exact compare: a hash of many units'
// counts can collide).
static void range_signature(const mkv_cache* c, int ub, int n, std::vector<int32_t>& sig) {
    sig.resize(2 * (size_t)n);
    for (int i = 0; i < n; ++i) {
        sig[2 * i] = c->n_pages[ub + i];
        sig[2 * i + 1] = c->n_prefill[ub + i];
    }
}

// The host arithmetic of a plan for the current mirror counts of units [ub, ub + n): every
// unit's pages padded to whole batches, worker ranges whole batches (every worker gets the
// same number of batches: a batch costs the same however full it is).  buf = [pref (n + 1)]
// [wstart (max workers)] (staged layout: ints), then the unit records.
struct HostPlan {
    std::vector<int32_t> buf;
    std::vector<UnitRec> rec;
    int total = 0, warps = 0, grid = 0;
};
static size_t plan_ints(const mkv_cache* c) { return ((c->n_units + 1 + (size_t)num_sms() * kMaxPagesWarps + 3) / 4) * 4; }
// CTAs of the page pass (one per SM at most): MKV_PAGE_CTAS overrides (A/B of leaving SMs to
// the co-scheduled finish kernels)
static int page_ctas() {
    static const int n = [] {
        const char* e = getenv("MKV_PAGE_CTAS");
        const int v = e ? atoi(e) : 0;
        return (v > 0 && v <= num_sms()) ? v : num_sms();
    }();
    return n;
}
static void host_plan(const mkv_cache* c, int ub, int n, HostPlan& hp) {
    const PagesConfig pc = pages_config();
    const int wpc = pc.warps, bm = pc.batch - 1;
    const int max_warps = page_ctas() * wpc;
    hp.buf.assign(plan_ints(c), 0);
    int32_t* pref = hp.buf.data();
    for (int i = 0; i < n; ++i) pref[i + 1] = pref[i] + ((c->n_pages[ub + i] + bm) & ~bm);
    hp.total = pref[n];
    // balanced worker ranges (range_begin): every worker >= 2 batches (>= 8 pages for the
    // mma.sync pass), at most one worker per resident warp slot
    const int T = hp.total / pc.batch;
    const int min_batches = std::max(1, 8 / pc.batch);
    hp.warps = T > 0 ? std::max(1, std::min(max_warps, T / min_batches)) : 0;
    int32_t* wstart = pref + n + 1;
    for (int w = 0, i = 0; w < hp.warps; ++w) {  // first unit with pages that contains the range's first page
        const int p = pc.batch * range_begin(w, T, hp.warps);
        while (i < n - 1 && pref[i + 1] <= p) ++i;
        wstart[w] = i;
    }
    hp.rec.assign(n, UnitRec{});
    for (int i = 0; i < n; ++i) {
        const int u = ub + i;
        hp.rec[i].base = c->page_base[u] - pref[i];
        hp.rec[i].pbeg = pref[i];
        hp.rec[i].pend = pref[i + 1];
        hp.rec[i].rend = pref[i] + c->n_pages[u];
        hp.rec[i].n_prefill = c->n_prefill[u];
    }
    hp.grid = (hp.warps + wpc - 1) / wpc;
}
static void plan_point(const mkv_cache* c, Plan& pl, int n) {
    pl.d_pref = pl.d_buf[pl.cur];
    pl.d_rec = reinterpret_cast<UnitRec*>(pl.d_pref + plan_ints(c));
    pl.d_wstart = pl.d_pref + n + 1;
}
static int plan_alloc(mkv_cache* c, Plan& pl, int n) {
    if (pl.d_buf[0]) return MKV_OK;
    const size_t bytes = sizeof(int32_t) * plan_ints(c) + sizeof(UnitRec) * c->n_units;
    CK(cudaMalloc(&pl.d_buf[0], bytes));
    CK(cudaMalloc(&pl.d_buf[1], bytes));
    const size_t slots = (size_t)num_sms() * kMaxPagesWarps + n;  // slot = worker + local unit
    CK(cudaMalloc(&pl.d_part_ml, sizeof(float) * 2 * kMaxG * slots));
    CK(cudaMalloc(&pl.d_part_o, sizeof(float) * kMaxG * kHeadDim * slots));
    pl.cur = 0;
    plan_point(c, pl, n);
    return MKV_OK;
}

// A plan's host image ([ints plan_ints][UnitRec n], the layout of one d_buf) in the plan's pinned
// staging buffer, once the previous upload from it has completed (pl.ready): uploads are then
// plain DMA in stream order, never a host-blocking pageable copy.
static int stage_plan(mkv_cache* c, Plan& pl, const HostPlan& hp, int n, size_t* bytes) {
    if (!pl.ready) CK(cudaEventCreateWithFlags(&pl.ready, cudaEventDisableTiming));
    CK(cudaEventSynchronize(pl.ready));
    const size_t ib = sizeof(int32_t) * plan_ints(c), rb = sizeof(UnitRec) * n;
    if (pl.stage_bytes < ib + rb) {
        pinned_put(pl.h_stage, pl.stage_bytes);
        pl.h_stage = nullptr;
        pl.stage_bytes = 0;
        CK(pinned_get(ib + rb, &pl.h_stage, &pl.stage_bytes));
    }
    memcpy(pl.h_stage, hp.buf.data(), ib);
    memcpy(static_cast<uint8_t*>(pl.h_stage) + ib, hp.rec.data(), rb);
    *bytes = ib + rb;
    return MKV_OK;
}

// Allocates the plan of calls over units [ub, ub + n) ahead of its first use (device buffers,
// partial slots, upload event, pinned staging buffer); its contents are built by the first call.
static int plan_reserve(mkv_cache* c, int ub, int n) {
    const uint64_t key = ((uint64_t)(uint32_t)ub << 32) | (uint32_t)n;
    Plan& pl = c->plans[key];
    if (int r = plan_alloc(c, pl, n)) return r;
    if (!pl.ready) CK(cudaEventCreateWithFlags(&pl.ready, cudaEventDisableTiming));
    const size_t need = sizeof(int32_t) * plan_ints(c) + sizeof(UnitRec) * n;
    if (pl.stage_bytes < need) {
        pinned_put(pl.h_stage, pl.stage_bytes);
        pl.h_stage = nullptr;
        pl.stage_bytes = 0;
        CK(pinned_get(need, &pl.h_stage, &pl.stage_bytes));
    }
    return MKV_OK;
}

// jobs != nullptr: a changed plan is not uploaded but queued for plan_build_kernel (the
// caller launches it once the device meta holds the new page counts).  *swapped: the plan was
// prepared ahead and uploaded on the copy stream (the stream now waits for it; the caller
// launches its first reader with a full dependency).
static int get_plan(mkv_cache* c, int ub, int n, cudaStream_t s, Plan** out, PlanBuildJobs* jobs = nullptr,
                    bool* swapped = nullptr) {
    const uint64_t key = ((uint64_t)(uint32_t)ub << 32) | (uint32_t)n;
    Plan& pl = c->plans[key];
    thread_local std::vector<int32_t> sig;
    range_signature(c, ub, n, sig);
    if (swapped) *swapped = false;
    if (pl.d_pref && pl.sig == sig) {
        *out = &pl;
        return MKV_OK;
    }
    if (pl.pending && pl.pending_sig == sig) {  // prepared ahead: wait for its upload, swap
        CK(cudaStreamWaitEvent(s, pl.ready, 0));
        pl.cur ^= 1;
        plan_point(c, pl, n);
        pl.sig = sig;
        pl.total = pl.p_total; pl.warps = pl.p_warps; pl.grid = pl.p_grid;
        pl.pending = false;
        if (swapped) *swapped = true;
        *out = &pl;
        return MKV_OK;
    }
    pl.pending = false;
    HostPlan hp;
    host_plan(c, ub, n, hp);
    if (int r = plan_alloc(c, pl, n)) return r;
    if (jobs && jobs->n_jobs < kMaxPlanJobs && n > 0) {
        PlanBuildJob& jb = jobs->job[jobs->n_jobs++];
        jb.unit_begin = ub; jb.n = n; jb.warps = hp.warps; jb.batch = pages_config().batch;
        jb.pref = pl.d_pref; jb.wstart = pl.d_wstart; jb.rec = pl.d_rec;
    } else {
        size_t bytes = 0;
        if (int r = stage_plan(c, pl, hp, n, &bytes)) return r;
        CK(cudaMemcpyAsync(pl.d_pref, pl.h_stage, bytes, cudaMemcpyHostToDevice, s));
        CK(cudaEventRecord(pl.ready, s));
    }
    pl.sig = sig;
    pl.total = hp.total;
    pl.warps = hp.warps;
    pl.grid = hp.grid;
    *out = &pl;
    return MKV_OK;
}

// After a fused-flush step (the mirror already holds the new page counts): compute the plan
// the next call will need and upload it into the plan's other buffer on the copy stream, after
// everything queued on `s` so far (the other buffer's last readers included).
static int prepare_next_plan(mkv_cache* c, int ub, int n, cudaStream_t s) {
    const uint64_t key = ((uint64_t)(uint32_t)ub << 32) | (uint32_t)n;
    Plan& pl = c->plans[key];
    if (int r = plan_alloc(c, pl, n)) return r;
    if (!c->copy_stream) {
        CK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&c->ev_compute, cudaEventDisableTiming));
    }
    HostPlan hp;
    host_plan(c, ub, n, hp);
    size_t bytes = 0;
    if (int r = stage_plan(c, pl, hp, n, &bytes)) return r;
    CK(cudaEventRecord(c->ev_compute, s));
    CK(cudaStreamWaitEvent(c->copy_stream, c->ev_compute, 0));
    CK(cudaMemcpyAsync(pl.d_buf[pl.cur ^ 1], pl.h_stage, bytes, cudaMemcpyHostToDevice, c->copy_stream));
    CK(cudaEventRecord(pl.ready, c->copy_stream));
    range_signature(c, ub, n, pl.pending_sig);
    pl.pending = true;
    pl.p_total = hp.total; pl.p_warps = hp.warps; pl.p_grid = hp.grid;
    return MKV_OK;
}

// MKV_FLUSH=fused: a residual block is flushed by the finish kernel of the step that fills it
// (no append_kernel / plan_build_kernel launch; the next plan is uploaded off the critical
// path).  Measured slower than the default: the flush then runs per layer
// on 128 CTAs of 4 warps on the step's critical path, instead of one append launch for every
// layer's units across the whole GPU.
static bool fused_flush_enabled() {
    static const bool on = [] {
        const char* e = getenv("MKV_FLUSH");
        return e && e[0] == 'f';
    }();
    return on;
}

// Diagnostics (MKV_DECODE_TRACE): two alternating slots (consecutive decode calls), each
// [page-kernel warps x 4 stamps][finish CTAs x 4 stamps] of globaltimer values.
// page-kernel region: mma.sync 4 stamps per warp (<= kMaxPagesWarps per SM); tcgen05 kTcTraceWords
// per worker (2 per SM)
static size_t trace_page_words() {
    return (size_t)num_sms() * std::max<size_t>(4 * kMaxPagesWarps, 2 * kTcTraceWords);
}
static size_t trace_slot_words() { return trace_page_words() + 4 * (size_t)kTraceFinishCtas; }
static uint64_t* trace_slot(mkv_cache* c) {
    static const bool tracing = getenv("MKV_DECODE_TRACE") != nullptr;
    if (!tracing) return nullptr;
    if (!c->d_trace) {
        if (cudaMalloc(&c->d_trace, sizeof(uint64_t) * 2 * trace_slot_words()) != cudaSuccess) return nullptr;
        cudaMemset(c->d_trace, 0, sizeof(uint64_t) * 2 * trace_slot_words());
    }
    return c->d_trace + (c->trace_seq & 1) * trace_slot_words();
}

static void fill_pages_params(mkv_cache* c, const Plan* pl, const mkv_decode_args* a, PagesParams& pp) {
    pp.pool = c->d_pool; pp.meta = c->d_meta; pp.unit_begin = a->unit_begin; pp.n_units = a->n_units;
    pp.group = a->group; pp.q = static_cast<const __half*>(a->q);
    pp.pref = pl->d_pref; pp.wstart = pl->d_wstart; pp.rec = pl->d_rec; pp.total_pages = pl->total;
    pp.n_warps = pl->warps;
    pp.part_ml = pl->d_part_ml; pp.part_o = pl->d_part_o;
    pp.scale_log2 = a->scale * 1.4426950408889634f;
    pp.trace = trace_slot(c);
    pp.early = 0;
    pp.unit_cnt = nullptr;
}

// The finish step in one kernel (finish_kernel: a CTA per unit attends the unit's residual
// beside the page pass, waits for the page grid, merges) or two (launch_resid_merge: a
// persistent residual kernel + a merge kernel on per-unit arrival counters).  One finish CTA
// fits beside each page CTA, so with more units than SMs most finish CTAs -- residual attention
// included -- would only start after the page pass; the split form then keeps the residual work
// inside the page pass and leaves only the merges after it (headline step 0.622 -> 0.610 ms).
// With at most one unit per SM the one-kernel form is faster (one grid hop less per call: the
// dependent per-layer form, 0.84 vs 0.90 ms per 32-layer step).  MKV_MERGE=finish|split forces
// a form.  The tcgen05 page-kernel A/B variant does not count arrivals: always one kernel.
static bool split_finish(int n_units) {
    static const int mode = [] {
        const char* e = getenv("MKV_MERGE");
        if (pages_config().tc || (e && e[0] == 'f')) return 0;
        return (e && e[0] == 's') ? 1 : 2;
    }();
    return mode == 1 || (mode == 2 && n_units > num_sms());
}

// early: a later layer of one mkv_decode_step_layers call -- its q was written before the
// call, so the page kernel may read it while the previous layer's finish kernel still runs
// argument / capacity checks of one decode call (no state change)
static int decode_validate(mkv_cache* c, const mkv_decode_args* a, bool attend) {
    const int ub = a->unit_begin, n = a->n_units;
    if (int r = check_range(c, ub, n)) return r;
    if (n == 0) return MKV_OK;
    const bool append = a->k_new != nullptr;
    if (append && !a->v_new) return fail(MKV_ERR_INVALID_ARGUMENT, "decode_append: null v");
    if (attend) {
        if (a->group < 1 || a->group > kMaxG) return fail(MKV_ERR_UNSUPPORTED, "decode: group %d outside 1..8", a->group);
        if (!a->q || !a->out) return fail(MKV_ERR_INVALID_ARGUMENT, "decode: null q/out");
        if (!aligned16(a->q) || !aligned16(a->out)) return fail(MKV_ERR_INVALID_ARGUMENT, "decode: q/out must be 16-byte aligned");
    }
    if (append && (!aligned16(a->k_new) || !aligned16(a->v_new)))
        return fail(MKV_ERR_INVALID_ARGUMENT, "decode_append: k/v must be 16-byte aligned");
    for (int i = 0; i < n; ++i) {
        const int u = ub + i;
        const int64_t total = (int64_t)c->n_pages[u] + c->n_res[u];
        if (attend && total == 0) return fail(MKV_ERR_RUNTIME, "decode_step: empty cache (unit %d)", u);
        if (append && c->n_res[u] + 1 == c->n_r && c->n_pages[u] + c->n_r / kGroup > c->cap_pages[u])
            return fail(MKV_ERR_OUT_OF_RANGE, "decode: unit %d exceeds max_decode_tokens", u);
    }
    return MKV_OK;
}

// after_plan_build: the plan this call's page kernel reads was just written by plan_build_kernel
// (fused flush step, first layer): launch that page kernel with a full dependency, since it
// reads its plan before griddepcontrol.wait.
static int decode_impl(mkv_cache* c, const mkv_decode_args* a, bool attend, cudaStream_t s, bool early = false,
                       bool after_plan_build = false) {
    const int ub = a->unit_begin, n = a->n_units;
    if (int r = check_range(c, ub, n)) return r;
    if (n == 0) return MKV_OK;
    const bool append = a->k_new != nullptr;
    if (append && !a->v_new) return fail(MKV_ERR_INVALID_ARGUMENT, "decode_append: null v");
    if (attend) {
        if (a->group < 1 || a->group > kMaxG) return fail(MKV_ERR_UNSUPPORTED, "decode: group %d outside 1..8", a->group);
        if (!a->q || !a->out) return fail(MKV_ERR_INVALID_ARGUMENT, "decode: null q/out");
        if (!aligned16(a->q) || !aligned16(a->out)) return fail(MKV_ERR_INVALID_ARGUMENT, "decode: q/out must be 16-byte aligned");
    }
    if (append && (!aligned16(a->k_new) || !aligned16(a->v_new)))
        return fail(MKV_ERR_INVALID_ARGUMENT, "decode_append: k/v must be 16-byte aligned");
    // validate everything before mutating the mirror
    for (int i = 0; i < n; ++i) {
        const int u = ub + i;
        const int64_t total = (int64_t)c->n_pages[u] + c->n_res[u];
        if (attend && total == 0) return fail(MKV_ERR_RUNTIME, "decode_step: empty cache (unit %d)", u);
        if (append && c->n_res[u] + 1 == c->n_r && c->n_pages[u] + c->n_r / kGroup > c->cap_pages[u])
            return fail(MKV_ERR_OUT_OF_RANGE, "decode: unit %d exceeds max_decode_tokens", u);
    }
    if (int r = require_device()) return r;
    // Fused flush (default): a unit whose residual this append fills is flushed by this step's
    // finish kernel (quantize the block into pages, attend it dequantized); this step's page pass
    // covers the pages that existed before, so its plan is taken before the mirror moves on.
    const bool fused = attend && append && fused_flush_enabled();
    Plan* pl = nullptr;
    bool swapped = false;
    if (fused)
        if (int r = get_plan(c, ub, n, s, &pl, nullptr, &swapped)) return r;
    bool any_flush = false;
    if (append) {
        for (int i = 0; i < n; ++i) {
            const int u = ub + i;
            if (++c->n_res[u] == c->n_r) {
                c->n_res[u] = 0;
                c->n_pages[u] += c->n_r / kGroup;
                c->n_blocks[u] += 1;
                any_flush = true;
            }
        }
    }
    ResidualParams rp;
    rp.meta = c->d_meta; rp.unit_begin = ub; rp.n_units = n; rp.group = a->group; rp.n_r = c->n_r;
    rp.q = static_cast<const __half*>(a->q);
    rp.k_new = static_cast<const __half*>(a->k_new);
    rp.v_new = static_cast<const __half*>(a->v_new);
    rp.res_k = c->d_res_k; rp.res_v = c->d_res_v; rp.pool = c->d_pool; rp.shadow = c->d_shadow;
    rp.out = static_cast<__half*>(a->out);
    rp.scale_log2 = a->scale * 1.4426950408889634f;
    rp.status = c->d_status;
    rp.trace = nullptr;
    rp.fused_flush = fused && any_flush ? 1 : 0;
    rp.unit_cnt = nullptr; rp.res_ml = c->d_res_ml; rp.res_o = c->d_res_o;
    const bool split = attend && split_finish(n);
    // unfused flush steps (or append-only calls): append (+ quantize the full block) before the
    // page pass
    if (!fused && append && (any_flush || !attend)) {
        CK(launch_append(rp, s));
        rp.k_new = nullptr;
        rp.v_new = nullptr;
    }
    if (!attend) return MKV_OK;
    if (!fused)
        if (int r = get_plan(c, ub, n, s, &pl, nullptr, &swapped)) return r;
    if (pl->total > 0) {
        PagesParams pp;
        fill_pages_params(c, pl, a, pp);
        // split finish: no early page passes -- the merge kernel does not wait for the page /
        // residual grids, so a page kernel's start wait on the previous merge is what orders
        // every later kernel after the previous layer's partials were consumed
        pp.early = early && !split && (fused || !any_flush) ? 1 : 0;
        if (split) pp.unit_cnt = c->d_unit_cnt;
        // full dependency when the plan was just written by a kernel or swapped in behind an
        // event wait (the page kernel reads it before its griddepcontrol.wait)
        CK(launch_pages(pp, pl->grid, s, !(after_plan_build || swapped)));
    }
    rp.part_ml = pl->d_part_ml; rp.part_o = pl->d_part_o;
    rp.trace = trace_slot(c);
    if (rp.trace) rp.trace += trace_page_words();
    const WorkerRanges wr{std::max(pl->warps, 1), std::max(pl->total / pages_config().batch, 1), pages_config().batch};
    if (split) {
        rp.unit_cnt = c->d_unit_cnt;
        if (cudaError_t e = launch_resid_merge(rp, pl->d_pref, wr, pl->total > 0, std::min(n, num_sms()), s)) {
            // the page kernel may have counted: leave no stale arrivals for a later merge
            cudaMemsetAsync(c->d_unit_cnt + ub, 0, sizeof(int) * n, s);
            return cuda_fail(e, "decode: residual / merge kernels");
        }
    } else {
        CK(launch_finish(rp, pl->d_pref, wr, pl->total > 0, s));
    }
    ++c->trace_seq;
    // the next call's plan (new page counts), prepared and uploaded off the critical path
    if (fused && any_flush)
        if (int r = prepare_next_plan(c, ub, n, s)) return r;
    return MKV_OK;
}

uint64_t mkv_debug_launch_count(void) { return launch_count(); }

int mkv_debug_decode_trace(const mkv_cache* c, uint64_t* out, int max_words) {
    if (!c || !out) return fail(MKV_ERR_INVALID_ARGUMENT, "trace: null");
    if (!c->d_trace) return fail(MKV_ERR_RUNTIME, "trace: run with MKV_DECODE_TRACE set");
    CK(cudaDeviceSynchronize());
    const int n = (int)std::min<size_t>(max_words, 2 * trace_slot_words());
    CK(cudaMemcpy(out, c->d_trace, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost));
    return n;
}

int mkv_decode_step(mkv_cache* c, const mkv_decode_args* a, void* stream) {
    if (!a) return fail(MKV_ERR_INVALID_ARGUMENT, "decode_step: null args");
    return decode_impl(c, a, true, static_cast<cudaStream_t>(stream));
}

// The unit-resident steps kernel (one CTA per unit for all steps, decode.cu steps_kernel) serves
// a decode_steps call when its units fit one CTA each and are short: at most one unit per SM and
// at most kStepsMaxPages pages per unit by the last step.  MKV_STEPS=off keeps the per-step
// kernels (page pass + finish per step), MKV_STEPS=on ignores the size limits.
constexpr int kStepsMaxPages = 1024;
static int steps_mode() {
    static const int m = [] {
        const char* e = getenv("MKV_STEPS");
        if (!e) return 1;
        return e[1] == 'f' ? 0 : (e[1] == 'n' ? 2 : 1);
    }();
    return m;
}
// validates every step up front (the per-step path checks each step as it goes) and, if the
// steps kernel serves the call, launches it and moves the host mirror through the same appends
static int decode_steps_resident(mkv_cache* c, const mkv_decode_steps_args* a, cudaStream_t s, bool* done) {
    *done = false;
    const int mode = steps_mode();
    const int ub = a->unit_begin, n = a->n_units;
    if (mode == 0 || n <= 0 || a->n_steps == 0 || n > num_sms() || check_range(c, ub, n) != MKV_OK) return MKV_OK;
    if (a->group < 1 || a->group > kMaxG || !a->q || !a->out) return MKV_OK;  // the per-step path reports it
    const bool append = a->k_new != nullptr;
    if (!aligned16(a->q) || !aligned16(a->out) || a->q_step % 8 || a->out_step % 8 ||
        (append && (!aligned16(a->k_new) || !aligned16(a->v_new) || a->kv_step % 8)))
        return MKV_OK;
    const int npg = c->n_r / kGroup;
    for (int i = 0; i < n; ++i) {
        const int u = ub + i;
        if ((int64_t)c->n_pages[u] + c->n_res[u] == 0 && !append) return MKV_OK;
        const int64_t flushes = append ? (c->n_res[u] + (int64_t)a->n_steps) / c->n_r : 0;
        const int64_t pages = c->n_pages[u] + flushes * npg;
        if (pages > c->cap_pages[u]) return MKV_OK;  // the per-step path fails at the right step
        if (mode == 1 && pages > kStepsMaxPages) return MKV_OK;
    }
    if (int r = require_device()) return r;
    StepsParams sp;
    sp.meta = c->d_meta; sp.unit_begin = ub; sp.n_units = n; sp.group = a->group; sp.n_r = c->n_r;
    sp.n_steps = a->n_steps;
    sp.q = static_cast<const __half*>(a->q); sp.q_step = a->q_step;
    sp.k_new = static_cast<const __half*>(a->k_new); sp.v_new = static_cast<const __half*>(a->v_new);
    sp.kv_step = a->kv_step;
    sp.out = static_cast<__half*>(a->out); sp.out_step = a->out_step;
    sp.res_k = c->d_res_k; sp.res_v = c->d_res_v; sp.pool = c->d_pool; sp.shadow = c->d_shadow;
    sp.scale_log2 = a->scale * 1.4426950408889634f;
    sp.status = c->d_status;
    CK(launch_steps(sp, s));
    if (append)
        for (int i = 0; i < n; ++i) {
            const int u = ub + i;
            const int64_t tot = (int64_t)c->n_res[u] + a->n_steps;
            c->n_pages[u] += (int)(tot / c->n_r) * npg;
            c->n_blocks[u] += (int)(tot / c->n_r);
            c->n_res[u] = (int)(tot % c->n_r);
        }
    *done = true;
    return MKV_OK;
}

int mkv_decode_steps(mkv_cache* c, const mkv_decode_steps_args* a, void* stream) {
    if (!a) return fail(MKV_ERR_INVALID_ARGUMENT, "decode_steps: null args");
    if (a->n_steps < 0) return fail(MKV_ERR_INVALID_ARGUMENT, "decode_steps: negative step count");
    if ((a->k_new == nullptr) != (a->v_new == nullptr)) return fail(MKV_ERR_INVALID_ARGUMENT, "decode_append: null v");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    {
        bool done = false;
        if (int r = decode_steps_resident(c, a, s, &done)) return r;
        if (done) return MKV_OK;
    }
    auto at = [](const void* base, int64_t elems) -> const void* {
        return base ? static_cast<const __half*>(base) + elems : nullptr;
    };
    for (int st = 0; st < a->n_steps; ++st) {
        mkv_decode_args d;
        d.unit_begin = a->unit_begin;
        d.n_units = a->n_units;
        d.group = a->group;
        d.q = at(a->q, st * a->q_step);
        d.k_new = at(a->k_new, st * a->kv_step);
        d.v_new = at(a->v_new, st * a->kv_step);
        d.out = const_cast<void*>(at(a->out, st * a->out_step));
        d.scale = a->scale;
        if (int r = decode_impl(c, &d, true, s)) return r;
    }
    return MKV_OK;
}

int mkv_decode_pages_only(mkv_cache* c, const mkv_decode_args* a, void* stream) {
    if (!a) return fail(MKV_ERR_INVALID_ARGUMENT, "decode: null args");
    if (int r = check_range(c, a->unit_begin, a->n_units)) return r;
    if (a->group < 1 || a->group > kMaxG || !a->q || !a->out) return fail(MKV_ERR_INVALID_ARGUMENT, "decode: bad args");
    if (int r = require_device()) return r;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Plan* pl = nullptr;
    bool swapped = false;
    if (int r = get_plan(c, a->unit_begin, a->n_units, s, &pl, nullptr, &swapped)) return r;
    if (pl->total == 0) return MKV_OK;
    PagesParams pp;
    fill_pages_params(c, pl, a, pp);
    // the page kernel a decode call of this size runs: the counting variant when its finish step
    // is split (counts go to a scratch array: no merge follows)
    if (split_finish(a->n_units)) pp.unit_cnt = c->d_scratch_cnt;
    CK(launch_pages(pp, pl->grid, s, !swapped));
    return MKV_OK;
}

// Layer l+1 continues layer l: adjacent unit ranges, the same group and scale, and q / out (and
// the appended k / v, if any) laid out back to back, as in one [layers][units] array.  Such
// layers are one batch of independent units -- one page pass and one finish pass cover them.
static bool continues(const mkv_decode_args& p, const mkv_decode_args& l) {
    auto at = [](const void* base, int64_t bytes) { return static_cast<const uint8_t*>(base) + bytes; };
    const int64_t n = p.n_units, G = p.group;
    if (l.unit_begin != p.unit_begin + p.n_units || l.group != p.group || l.scale != p.scale) return false;
    if (!p.q || !p.out || l.q != at(p.q, n * G * kHeadDim * 2) || l.out != at(p.out, n * G * kHeadDim * 2)) return false;
    if ((p.k_new == nullptr) != (l.k_new == nullptr) || (p.v_new == nullptr) != (l.v_new == nullptr)) return false;
    if (p.k_new && (l.k_new != at(p.k_new, n * kHeadDim * 2) || l.v_new != at(p.v_new, n * kHeadDim * 2))) return false;
    return true;
}

static int decode_layers(mkv_cache* c, int n_layers, const mkv_decode_args* a, cudaStream_t s);

int mkv_decode_step_layers(mkv_cache* c, int n_layers, const mkv_decode_args* a, void* stream) {
    if (!a || n_layers < 0) return fail(MKV_ERR_INVALID_ARGUMENT, "decode_step: bad layer list");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // coalesce runs of continuing layers (MKV_LAYERS_SPLIT=1 keeps one pass per layer: A/B)
    static const bool split = getenv("MKV_LAYERS_SPLIT") != nullptr;
    if (split || n_layers < 2) return decode_layers(c, n_layers, a, s);
    std::vector<mkv_decode_args> runs;
    runs.reserve(n_layers);
    for (int l = 0; l < n_layers; ++l) {
        if (!runs.empty() && a[l].n_units > 0 && runs.back().n_units > 0 && continues(runs.back(), a[l]))
            runs.back().n_units += a[l].n_units;
        else
            runs.push_back(a[l]);
    }
    return decode_layers(c, (int)runs.size(), runs.data(), s);
}

static int decode_layers(mkv_cache* c, int n_layers, const mkv_decode_args* a, cudaStream_t s) {
    // A layer's page kernel may skip its early griddepcontrol.wait (P.early) only if its unit
    // range is disjoint from every earlier layer's range in this call: the early kernel reads
    // meta/plan and triggers its dependents before the previous finish kernel (which appends
    // to, and merges into, the units it owns) has completed.
    auto disjoint = [&](int l, int m) {
        return a[l].unit_begin + a[l].n_units <= a[m].unit_begin || a[m].unit_begin + a[m].n_units <= a[l].unit_begin;
    };
    std::vector<char> early(n_layers, 0);
    bool all_disjoint = true;
    for (int l = 0; l < n_layers; ++l) {
        bool ok = l > 0;
        for (int m = 0; m < l && ok; ++m) ok = disjoint(l, m);
        early[l] = ok ? 1 : 0;
        if (l > 0 && !ok) all_disjoint = false;
    }
    bool all_append = n_layers > 1 && n_layers <= kMaxAppendSegs, flush = false;
    for (int l = 0; l < n_layers; ++l) all_append = all_append && a[l].k_new != nullptr && a[l].n_units > 0;
    // A flush step with every layer appending: validate everything, update the mirror, then append
    // + flush every layer's units in ONE launch and build the changed plans on the device, so the
    // per-layer kernels that follow carry no append launches or copies between them.  The fused
    // append needs pairwise-disjoint ranges (one launch appends every layer's units).
    if (all_disjoint && all_append && !fused_flush_enabled()) {
        for (int l = 0; l < n_layers && !flush; ++l)
            for (int i = 0; i < a[l].n_units && !flush; ++i) {
                const int u = a[l].unit_begin + i;
                if (u >= 0 && u < c->n_units && c->n_res[u] + 1 == c->n_r) flush = true;
            }
    }
    if (all_disjoint && all_append && flush && !fused_flush_enabled()) {
        for (int l = 0; l < n_layers; ++l)
            if (int r = decode_validate(c, a + l, true)) return r;
        if (int r = require_device()) return r;
        // the mirror of every unit of the call, restored (and the affected plans invalidated)
        // if anything below fails before the device work is queued
        struct Saved { int u, n_res, n_pages, n_blocks; };
        std::vector<Saved> saved;
        for (int l = 0; l < n_layers; ++l)
            for (int i = 0; i < a[l].n_units; ++i) {
                const int u = a[l].unit_begin + i;
                saved.push_back({u, c->n_res[u], c->n_pages[u], c->n_blocks[u]});
            }
        auto rollback = [&](int r) {
            for (const Saved& sv : saved) {
                c->n_res[sv.u] = sv.n_res; c->n_pages[sv.u] = sv.n_pages; c->n_blocks[sv.u] = sv.n_blocks;
            }
            for (int l = 0; l < n_layers; ++l) {
                auto it = c->plans.find(((uint64_t)(uint32_t)a[l].unit_begin << 32) | (uint32_t)a[l].n_units);
                if (it != c->plans.end()) it->second.sig.clear();
            }
            return r;
        };
        AppendSegs segs{};
        segs.n_seg = n_layers;
        for (int l = 0; l < n_layers; ++l) {
            for (int i = 0; i < a[l].n_units; ++i) {
                const int u = a[l].unit_begin + i;
                if (++c->n_res[u] == c->n_r) {
                    c->n_res[u] = 0;
                    c->n_pages[u] += c->n_r / kGroup;
                    c->n_blocks[u] += 1;
                }
            }
            segs.block_begin[l + 1] = segs.block_begin[l] + a[l].n_units;
            segs.unit_begin[l] = a[l].unit_begin;
            segs.k_new[l] = static_cast<const __half*>(a[l].k_new);
            segs.v_new[l] = static_cast<const __half*>(a[l].v_new);
        }
        // changed plans are built on the device from the meta the append kernel updates
        PlanBuildJobs jobs{};
        for (int l = 0; l < n_layers; ++l) {
            Plan* pl = nullptr;
            if (int r = get_plan(c, a[l].unit_begin, a[l].n_units, s, &pl, &jobs)) return rollback(r);
        }
        ResidualParams rp{};
        rp.meta = c->d_meta; rp.n_r = c->n_r; rp.res_k = c->d_res_k; rp.res_v = c->d_res_v;
        rp.pool = c->d_pool; rp.shadow = c->d_shadow; rp.status = c->d_status;
        if (cudaError_t e = launch_append_segments(rp, segs, s)) return rollback(cuda_fail(e, "append kernel"));
        if (cudaError_t e = launch_plan_build(c->d_meta, jobs, s)) return rollback(cuda_fail(e, "plan build kernel"));
        for (int l = 0; l < n_layers; ++l) {
            mkv_decode_args al = a[l];
            al.k_new = nullptr;  // appended above
            al.v_new = nullptr;
            // layer 0's page kernel reads a plan plan_build_kernel just wrote: no PDL for it
            if (int r = decode_impl(c, &al, true, s, early[l] != 0, l == 0 && jobs.n_jobs > 0)) return r;
        }
        return MKV_OK;
    }
    for (int l = 0; l < n_layers; ++l)
        if (int r = decode_impl(c, a + l, true, s, early[l] != 0)) return r;
    return MKV_OK;
}

int mkv_cache_append(mkv_cache* c, int ub, int n, const void* k_new, const void* v_new, void* stream) {
    if (!k_new || !v_new) return fail(MKV_ERR_INVALID_ARGUMENT, "decode_append: null token");
    mkv_decode_args a{};
    a.unit_begin = ub; a.n_units = n; a.group = 1; a.k_new = k_new; a.v_new = v_new;
    return decode_impl(c, &a, false, static_cast<cudaStream_t>(stream));
}

// ---------------------------------------------------------------------------
// export to the reference QuantizedTensor format (quantizer.hpp:30-42)
// ---------------------------------------------------------------------------
static void block_list(const mkv_cache* c, int u, std::vector<int>& rows) {
    rows.clear();
    if (c->n_blocks[u] == 0) return;
    // a prefill block (n_prefill > 0 rows; prefill never keeps zero) then n_r-row flush blocks
    const int pre = c->n_prefill[u] > 0 ? 1 : 0;
    if (pre) rows.push_back(c->n_prefill[u]);
    for (int b = pre; b < c->n_blocks[u]; ++b) rows.push_back(c->n_r);
}

int mkv_cache_export_sizes(const mkv_cache* c, int u, int which, int64_t* n_words, int64_t* n_params,
                           int64_t* n_blocks) {
    if (int r = check_range(c, u, 1)) return r;
    std::vector<int> rows;
    block_list(c, u, rows);
    int64_t codes = 0, params = 0;
    for (int R : rows) {
        codes += (int64_t)R * c->d;
        params += which == 0 ? (int64_t)c->d * ((R + c->gs - 1) / c->gs) : (int64_t)R * (c->d / c->gs);
    }
    if (n_words) *n_words = (codes + 15) / 16;
    if (n_params) *n_params = params;
    if (n_blocks) *n_blocks = (int64_t)rows.size();
    return MKV_OK;
}

int mkv_cache_export_reference(const mkv_cache* c, int u, int which, uint32_t* words, float* params,
                               int64_t* block_rows) {
    if (int r = check_range(c, u, 1)) return r;
    if (which != 0 && which != 1) return fail(MKV_ERR_INVALID_ARGUMENT, "export: which must be 0 or 1");
    CK(cudaDeviceSynchronize());
    const int np = c->n_pages[u];
    std::vector<uint8_t> pages((size_t)np * kPageBytes);
    std::vector<float> shadow;
    if (np) CK(cudaMemcpy(pages.data(), c->d_pool + (size_t)c->page_base[u] * kPageBytes, pages.size(), cudaMemcpyDeviceToHost));
    if (c->shadow && np) {
        shadow.resize((size_t)np * kShadowBytes / 4);
        CK(cudaMemcpy(shadow.data(), c->d_shadow + (size_t)c->page_base[u] * (kShadowBytes / 4),
                      shadow.size() * 4, cudaMemcpyDeviceToHost));
    }
    std::vector<int> rows;
    block_list(c, u, rows);
    auto half_to_float = [](uint16_t h) { __half_raw r; r.x = h; return __half2float(__half(r)); };
    auto code_of = [&](int pg, int t, int ch) -> uint32_t {
        const uint8_t* page = pages.data() + (size_t)pg * kPageBytes;
        const CodePos cp = which == 0 ? k_code_pos(t, ch) : v_code_pos(t, ch);
        const uint32_t* w = reinterpret_cast<const uint32_t*>(page + (which == 0 ? kKC : kVC));
        return (w[cp.word] >> cp.shift) & 3u;
    };
    auto param_of = [&](int pg, int t, int ch, float* sc, float* zp) {
        const uint8_t* page = pages.data() + (size_t)pg * kPageBytes;
        if (!shadow.empty()) {
            const float* sh = shadow.data() + (size_t)pg * (kShadowBytes / 4);
            if (which == 0) { *sc = sh[2 * ch]; *zp = sh[2 * ch + 1]; }
            else { const int g = ch / 16; *sc = sh[256 + 2 * (t * 8 + g)]; *zp = sh[256 + 2 * (t * 8 + g) + 1]; }
            return;
        }
        const uint16_t* hs;
        if (which == 0) {
            hs = reinterpret_cast<const uint16_t*>(page + kKS);
            *sc = half_to_float(hs[k_param_idx(ch)]);
            *zp = half_to_float(reinterpret_cast<const uint16_t*>(page + kKZ)[k_param_idx(ch)]);
        } else {
            const int g = ch / 16;
            *sc = half_to_float(reinterpret_cast<const uint16_t*>(page + kVS)[vs_param_idx(t, g)]);
            *zp = half_to_float(reinterpret_cast<const uint16_t*>(page + kVZ)[vz_param_idx(t, g)]);
        }
    };
    int64_t code_idx = 0, group_idx = 0;
    int64_t nw = 0;
    mkv_cache_export_sizes(c, u, which, &nw, nullptr, nullptr);
    if (words) std::fill(words, words + nw, 0u);
    auto push = [&](uint32_t code) {
        if (words) words[code_idx / 16] |= code << (2 * (code_idx % 16));
        ++code_idx;
    };
    int page0 = 0;
    const int d = c->d;
    for (size_t b = 0; b < rows.size(); ++b) {
        const int R = rows[b];
        if (which == 0) {  // PerChannel: for channel, for token group
            for (int ch = 0; ch < d; ++ch) {
                for (int g0 = 0; g0 < R; g0 += 16) {
                    const int glen = std::min(16, R - g0), pg = page0 + g0 / 16;
                    float sc, zp;
                    param_of(pg, 0, ch, &sc, &zp);
                    if (params) { params[2 * group_idx] = sc; params[2 * group_idx + 1] = zp; }
                    ++group_idx;
                    for (int t = 0; t < glen; ++t) push(code_of(pg, t, ch));
                }
            }
        } else {  // PerToken: for token, for channel group
            for (int r = 0; r < R; ++r) {
                const int pg = page0 + r / 16, t = r % 16;
                for (int g0 = 0; g0 < d; g0 += 16) {
                    float sc, zp;
                    param_of(pg, t, g0, &sc, &zp);
                    if (params) { params[2 * group_idx] = sc; params[2 * group_idx + 1] = zp; }
                    ++group_idx;
                    for (int ch = g0; ch < g0 + 16; ++ch) push(code_of(pg, t, ch));
                }
            }
        }
        if (block_rows) block_rows[b] = R;
        page0 += (R + 15) / 16;
    }
    return MKV_OK;
}

int mkv_cache_export_residual(const mkv_cache* c, int u, uint16_t* rk, uint16_t* rv) {
    if (int r = check_range(c, u, 1)) return r;
    CK(cudaDeviceSynchronize());
    const size_t bytes = (size_t)c->n_res[u] * c->d * sizeof(__half);
    if (bytes) {
        CK(cudaMemcpy(rk, c->d_res_k + (size_t)u * c->n_r * c->d, bytes, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(rv, c->d_res_v + (size_t)u * c->n_r * c->d, bytes, cudaMemcpyDeviceToHost));
    }
    return MKV_OK;
}

int mkv_cache_check(mkv_cache* c) {
    if (!c) return fail(MKV_ERR_INVALID_ARGUMENT, "cache: null handle");
    CK(cudaDeviceSynchronize());
    uint32_t st = 0;
    CK(cudaMemcpy(&st, c->d_status, sizeof(st), cudaMemcpyDeviceToHost));
    if (st) {
        CK(cudaMemset(c->d_status, 0, sizeof(uint32_t)));
        if (st & kStatusNonFinite) return fail(MKV_ERR_DOMAIN, "quantize_group: non-finite input");
        if (st & kStatusMergeTimeout) return fail(MKV_ERR_RUNTIME, "decode: a merge timed out waiting for its partials");
    }
    return MKV_OK;
}

// ---------------------------------------------------------------------------
// MKVC snapshots (snapshot.cpp:71-198)
// ---------------------------------------------------------------------------
namespace {
void put_u32(std::vector<uint8_t>& b, uint32_t v) {
    for (int i = 0; i < 4; ++i) b.push_back(static_cast<uint8_t>((v >> (8 * i)) & 0xFF));
}
void put_u64(std::vector<uint8_t>& b, uint64_t v) {
    for (int i = 0; i < 8; ++i) b.push_back(static_cast<uint8_t>((v >> (8 * i)) & 0xFF));
}
void put_f32(std::vector<uint8_t>& b, float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    put_u32(b, u);
}
struct Reader {
    const std::vector<uint8_t>& b;
    size_t pos = 0;
    bool ok = true;
    uint64_t get(int bytes) {
        if (pos + bytes > b.size()) {
            ok = false;
            return 0;
        }
        uint64_t v = 0;
        for (int i = 0; i < bytes; ++i) v |= static_cast<uint64_t>(b[pos + i]) << (8 * i);
        pos += bytes;
        return v;
    }
    uint32_t u32() { return static_cast<uint32_t>(get(4)); }
    uint64_t u64() { return get(8); }
    float f32() {
        const uint32_t u = u32();
        float f;
        memcpy(&f, &u, 4);
        return f;
    }
};
struct SnapTensor {
    uint32_t axis = 0;
    uint64_t rows = 0;
    std::vector<uint64_t> blocks;
    std::vector<uint32_t> words;
    std::vector<float> params;  // (scale, zero) pairs
};
bool read_tensor(Reader& r, SnapTensor& t, uint64_t d) {
    t.axis = r.u32();
    t.rows = r.u64();
    const uint64_t nb = r.u64();
    if (!r.ok || nb > r.b.size()) return false;
    t.blocks.resize(nb);
    uint64_t codes = 0;
    for (auto& x : t.blocks) {
        x = r.u64();
        codes += x * d;
    }
    const uint64_t nw = r.u64();
    if (!r.ok || nw > r.b.size()) return false;
    t.words.resize(nw);
    for (auto& w : t.words) w = r.u32();
    const uint64_t np = r.u64();
    if (!r.ok || np > r.b.size()) return false;
    t.params.resize(2 * np);
    for (auto& p : t.params) p = r.f32();
    return r.ok && nw == (codes + 15) / 16;  // snapshot.cpp:126-131
}
}  // namespace

int mkv_cache_save_mkvc(const mkv_cache* c, int u, const char* path) {
    if (int r = check_range(c, u, 1)) return r;
    if (!path) return fail(MKV_ERR_INVALID_ARGUMENT, "snapshot: null path");
    int64_t tq = 0;
    mkv_cache_unit_info(c, u, &tq, nullptr, nullptr, nullptr);
    std::vector<uint8_t> b;
    b.insert(b.end(), {'M', 'K', 'V', 'C'});
    put_u32(b, 1);
    put_u64(b, c->d);
    put_u64(b, c->n_r);
    put_u64(b, c->gs);
    put_u64(b, 0);  // QuantMode::TwoBit
    put_u64(b, (uint64_t)tq);
    for (int which = 0; which < 2; ++which) {
        int64_t nw = 0, np = 0, nb = 0;
        if (int r = mkv_cache_export_sizes(c, u, which, &nw, &np, &nb)) return r;
        std::vector<uint32_t> words(std::max<int64_t>(nw, 1));
        std::vector<float> params(std::max<int64_t>(2 * np, 2));
        std::vector<int64_t> br(std::max<int64_t>(nb, 1));
        if (int r = mkv_cache_export_reference(c, u, which, words.data(), params.data(), br.data())) return r;
        put_u32(b, which == 0 ? 0u : 1u);  // PerChannel keys, PerToken values
        put_u64(b, (uint64_t)tq);
        put_u64(b, (uint64_t)nb);
        for (int64_t i = 0; i < nb; ++i) put_u64(b, (uint64_t)br[i]);
        put_u64(b, (uint64_t)nw);
        for (int64_t i = 0; i < nw; ++i) put_u32(b, words[i]);
        put_u64(b, (uint64_t)np);
        for (int64_t i = 0; i < 2 * np; ++i) put_f32(b, params[i]);
    }
    put_u64(b, 0);  // identity-mode key / value stores: empty in 2-bit mode
    put_u64(b, 0);
    const int rows = c->n_res[u];
    std::vector<uint16_t> rk((size_t)std::max(rows, 1) * c->d), rv(rk.size());
    if (int r = mkv_cache_export_residual(c, u, rk.data(), rv.data())) return r;
    auto half_to_float = [](uint16_t h) { __half_raw x; x.x = h; return __half2float(__half(x)); };
    for (const auto* m : {&rk, &rv}) {
        put_u64(b, (uint64_t)rows);
        for (size_t i = 0; i < (size_t)rows * c->d; ++i) put_f32(b, half_to_float((*m)[i]));
    }
    FILE* f = fopen(path, "wb");
    if (!f) return fail(MKV_ERR_RUNTIME, "snapshot: cannot open %s", path);
    const size_t w = fwrite(b.data(), 1, b.size(), f);
    const int cl = fclose(f);
    if (w != b.size() || cl != 0) return fail(MKV_ERR_RUNTIME, "snapshot: write failed");
    return MKV_OK;
}

int mkv_cache_load_mkvc(mkv_cache* c, int u, const char* path) {
    if (int r = check_range(c, u, 1)) return r;
    if (!path) return fail(MKV_ERR_INVALID_ARGUMENT, "snapshot: null path");
    if (int r = require_device()) return r;
    std::vector<uint8_t> buf;
    {
        FILE* f = fopen(path, "rb");
        if (!f) return fail(MKV_ERR_RUNTIME, "snapshot: cannot open %s", path);
        uint8_t tmp[1 << 16];
        size_t n;
        while ((n = fread(tmp, 1, sizeof(tmp), f)) > 0) buf.insert(buf.end(), tmp, tmp + n);
        fclose(f);
    }
    if (buf.size() < 4 || memcmp(buf.data(), "MKVC", 4) != 0) return fail(MKV_ERR_RUNTIME, "snapshot: bad magic");
    Reader r{buf};
    r.pos = 4;
    const uint32_t version = r.u32();
    if (!r.ok) return fail(MKV_ERR_RUNTIME, "snapshot: truncated file");
    if (version != 1) return fail(MKV_ERR_RUNTIME, "snapshot: unsupported version");
    const uint64_t d = r.u64(), n_r = r.u64(), gs = r.u64(), mode = r.u64(), tq = r.u64();
    if (!r.ok) return fail(MKV_ERR_RUNTIME, "snapshot: truncated file");
    if (mode != 0) return fail(MKV_ERR_UNSUPPORTED, "snapshot: identity-mode caches have no device form");
    if (d != (uint64_t)c->d || n_r != (uint64_t)c->n_r || gs != (uint64_t)c->gs)
        return fail(MKV_ERR_INVALID_ARGUMENT, "snapshot: d/n_r/group_size %llu/%llu/%llu differ from the cache",
                    (unsigned long long)d, (unsigned long long)n_r, (unsigned long long)gs);
    SnapTensor tk, tv;
    if (!read_tensor(r, tk, d) || !read_tensor(r, tv, d)) {
        if (!r.ok) return fail(MKV_ERR_RUNTIME, "snapshot: truncated file");
        return fail(MKV_ERR_RUNTIME, "snapshot: packed word count inconsistent");
    }
    const uint64_t fk = r.u64();
    if (fk) return fail(MKV_ERR_UNSUPPORTED, "snapshot: identity stores in a 2-bit snapshot");
    const uint64_t fv = r.u64();
    if (fv) return fail(MKV_ERR_UNSUPPORTED, "snapshot: identity stores in a 2-bit snapshot");
    const uint64_t rrows = r.u64();
    if (!r.ok || rrows > n_r) return fail(MKV_ERR_RUNTIME, "snapshot: truncated file");
    std::vector<float> res_k(rrows * d), res_v;
    for (auto& x : res_k) x = r.f32();
    const uint64_t rrows_v = r.u64();
    if (!r.ok || rrows_v > n_r) return fail(MKV_ERR_RUNTIME, "snapshot: truncated file");
    res_v.resize(rrows_v * d);
    for (auto& x : res_v) x = r.f32();
    if (!r.ok) return fail(MKV_ERR_RUNTIME, "snapshot: truncated file");
    if (rrows != rrows_v || rrows >= n_r) return fail(MKV_ERR_RUNTIME, "snapshot: residual buffer state invalid");
    // device form: an optional first block of any size (the prefill block), then n_r-row blocks
    if (tk.blocks != tv.blocks || tk.axis != 0 || tv.axis != 1)
        return fail(MKV_ERR_UNSUPPORTED, "snapshot: key/value block structure not produced by the cache engine");
    uint64_t rows_total = 0;
    for (size_t b = 0; b < tk.blocks.size(); ++b) {
        if (tk.blocks[b] == 0 || (b > 0 && tk.blocks[b] != n_r))
            return fail(MKV_ERR_UNSUPPORTED, "snapshot: block %zu of %llu rows (device blocks: prefill, then n_r)", b,
                        (unsigned long long)tk.blocks[b]);
        rows_total += tk.blocks[b];
    }
    if (rows_total != tq || tk.rows != tq) return fail(MKV_ERR_RUNTIME, "snapshot: token counts inconsistent");
    const int nb = (int)tk.blocks.size();
    const int n_prefill = nb ? (int)tk.blocks[0] : 0;
    const int n_pages = nb ? (n_prefill + kGroup - 1) / kGroup + (nb - 1) * (c->n_r / kGroup) : 0;
    if (n_pages > c->cap_pages[u]) return fail(MKV_ERR_OUT_OF_RANGE, "snapshot: %d pages exceed the unit's capacity", n_pages);
    // rebuild the pages in the device layout (inverse of mkv_cache_export_reference)
    std::vector<uint8_t> pages((size_t)std::max(n_pages, 1) * kPageBytes, 0);
    std::vector<float> shadow(c->shadow ? (size_t)std::max(n_pages, 1) * kShadowBytes / 4 : 0, 0.0f);
    auto code_at = [](const std::vector<uint32_t>& w, uint64_t i) { return (w[i / 16] >> (2 * (i % 16))) & 3u; };
    auto half_bits = [](float f) { __half h = __float2half_rn(f); return *reinterpret_cast<uint16_t*>(&h); };
    uint64_t kc0 = 0, kg0 = 0, vc0 = 0, vg0 = 0;
    int page0 = 0;
    for (int b = 0; b < nb; ++b) {
        const int R = (int)tk.blocks[b], gpr = (R + kGroup - 1) / kGroup;
        for (int g = 0; g < gpr; ++g) {
            uint8_t* pg = pages.data() + (size_t)(page0 + g) * kPageBytes;
            uint32_t* kwords = reinterpret_cast<uint32_t*>(pg + kKC);
            uint32_t* vwords = reinterpret_cast<uint32_t*>(pg + kVC);
            uint16_t* ks = reinterpret_cast<uint16_t*>(pg + kKS);
            uint16_t* kz = reinterpret_cast<uint16_t*>(pg + kKZ);
            uint16_t* vs = reinterpret_cast<uint16_t*>(pg + kVS);
            uint16_t* vz = reinterpret_cast<uint16_t*>(pg + kVZ);
            float* sh = c->shadow ? shadow.data() + (size_t)(page0 + g) * (kShadowBytes / 4) : nullptr;
            const int valid = std::min(kGroup, R - kGroup * g);
            for (int ch = 0; ch < c->d; ++ch) {  // keys: PerChannel groups (channel-major within the block)
                const uint64_t gi = kg0 + (uint64_t)ch * gpr + g;
                const float sc = tk.params[2 * gi], zp = tk.params[2 * gi + 1];
                ks[k_param_idx(ch)] = half_bits(sc);
                kz[k_param_idx(ch)] = half_bits(zp);
                if (sh) { sh[2 * ch] = sc; sh[2 * ch + 1] = zp; }
                for (int t = 0; t < valid; ++t) {
                    const CodePos cp = k_code_pos(t, ch);
                    kwords[cp.word] |= code_at(tk.words, kc0 + (uint64_t)ch * R + kGroup * g + t) << cp.shift;
                }
            }
            for (int t = 0; t < valid; ++t) {  // values: PerToken groups (token-major)
                const uint64_t row = (uint64_t)kGroup * g + t;
                for (int vg = 0; vg < c->d / kGroup; ++vg) {
                    const uint64_t gi = vg0 + row * (c->d / kGroup) + vg;
                    const float sc = tv.params[2 * gi], zp = tv.params[2 * gi + 1];
                    vs[vs_param_idx(t, vg)] = half_bits(sc);
                    vz[vz_param_idx(t, vg)] = half_bits(zp);
                    if (sh) { sh[256 + 2 * (t * 8 + vg)] = sc; sh[256 + 2 * (t * 8 + vg) + 1] = zp; }
                    for (int cc = 0; cc < kGroup; ++cc) {
                        const int ch = kGroup * vg + cc;
                        const CodePos cp = v_code_pos(t, ch);
                        vwords[cp.word] |= code_at(tv.words, vc0 + row * c->d + ch) << cp.shift;
                    }
                }
            }
        }
        kc0 += (uint64_t)R * c->d;
        kg0 += (uint64_t)c->d * gpr;
        vc0 += (uint64_t)R * c->d;
        vg0 += (uint64_t)R * (c->d / kGroup);
        page0 += gpr;
    }
    if (kg0 * 2 != tk.params.size() || vg0 * 2 != tv.params.size())
        return fail(MKV_ERR_RUNTIME, "snapshot: parameter count inconsistent");
    CK(cudaDeviceSynchronize());
    if (n_pages) {
        CK(cudaMemcpy(c->d_pool + (size_t)c->page_base[u] * kPageBytes, pages.data(), (size_t)n_pages * kPageBytes,
                      cudaMemcpyHostToDevice));
        if (c->shadow)
            CK(cudaMemcpy(c->d_shadow + (size_t)c->page_base[u] * (kShadowBytes / 4), shadow.data(),
                          (size_t)n_pages * kShadowBytes, cudaMemcpyHostToDevice));
    }
    if (rrows) {
        std::vector<__half> hk(rrows * d), hv(rrows * d);
        for (size_t i = 0; i < hk.size(); ++i) {
            hk[i] = __float2half_rn(res_k[i]);
            hv[i] = __float2half_rn(res_v[i]);
        }
        CK(cudaMemcpy(c->d_res_k + (size_t)u * c->n_r * c->d, hk.data(), hk.size() * 2, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(c->d_res_v + (size_t)u * c->n_r * c->d, hv.data(), hv.size() * 2, cudaMemcpyHostToDevice));
    }
    c->n_prefill[u] = n_prefill;
    c->n_pages[u] = n_pages;
    c->n_blocks[u] = nb;
    c->n_res[u] = (int)rrows;
    CK(c->upload_meta(u, 1, 0));
    CK(cudaDeviceSynchronize());
    return MKV_OK;
}

// ---------------------------------------------------------------------------
// synthetic inputs
// ---------------------------------------------------------------------------
int mkv_synth_fp16(void* out, int64_t n, uint64_t seed, uint64_t stream_id, void* stream) {
    if (!out || n < 0) return fail(MKV_ERR_INVALID_ARGUMENT, "synth: bad args");
    if (int r = require_device()) return r;
    CK(launch_synth_fp16(static_cast<__half*>(out), 1, n, n, seed, stream_id, 0, static_cast<cudaStream_t>(stream)));
    return MKV_OK;
}

int mkv_synth_fp16_rows(void* out, int64_t n_rows, int64_t row_len, int64_t ld, uint64_t seed, uint64_t base,
                        uint64_t step, void* stream) {
    if (!out || n_rows < 0 || row_len < 0 || ld < row_len) return fail(MKV_ERR_INVALID_ARGUMENT, "synth: bad args");
    if (int r = require_device()) return r;
    CK(launch_synth_fp16(static_cast<__half*>(out), n_rows, row_len, ld, seed, base, step,
                         static_cast<cudaStream_t>(stream)));
    return MKV_OK;
}

int mkv_synth_uniform_f32(float* out, int64_t n_rows, int64_t row_len, int64_t ld, uint64_t seed, uint64_t base,
                          uint64_t step, void* stream) {
    if (!out || n_rows < 0 || row_len < 0 || ld < row_len) return fail(MKV_ERR_INVALID_ARGUMENT, "synth: bad args");
    if (int r = require_device()) return r;
    CK(launch_synth_uniform(out, n_rows, row_len, ld, seed, base, step, static_cast<cudaStream_t>(stream)));
    return MKV_OK;
}

// ---------------------------------------------------------------------------
// reference-format fp32 entries (refmt.cu)
// ---------------------------------------------------------------------------
int mkv_attention_f32(const mkv_attention_f32_args* a, void* stream) {
    if (!a) return fail(MKV_ERR_INVALID_ARGUMENT, "attention: null args");
    if (a->len_q <= 0 || a->len_k <= 0) return fail(MKV_ERR_INVALID_ARGUMENT, "attention: zero-length sequence");
    if (a->d <= 0 || a->dv <= 0) return fail(MKV_ERR_INVALID_ARGUMENT, "attention: q/k head dimension mismatch");
    if (a->causal && a->len_q > a->len_k)
        return fail(MKV_ERR_INVALID_ARGUMENT, "attention: causal requires l_query <= l_key");
    if (a->dv > attn_f32_max_dv()) return fail(MKV_ERR_UNSUPPORTED, "attention: value width %d > %d", a->dv, attn_f32_max_dv());
    if (!a->q || !a->k || !a->v || !a->out || !a->lse) return fail(MKV_ERR_INVALID_ARGUMENT, "attention: null tensor");
    if (int r = require_device()) return r;
    AttnF32Params p{a->q, a->k, a->v, a->ld_q, a->ld_k, a->ld_v, a->ld_o, a->out, a->lse, a->a_cumul,
                    a->len_q, a->len_k, a->d, a->dv, a->scale, a->causal};
    CK(launch_attn_f32(p, static_cast<cudaStream_t>(stream)));
    return MKV_OK;
}

int mkv_decode_attention_f32(const float* q, const float* keys, int64_t ld_k, const float* values, int64_t ld_v,
                             int n, int d, int dv, float scale, float* out, float* attn, void* stream) {
    if (n <= 0) return fail(MKV_ERR_INVALID_ARGUMENT, "decode_attention: empty key set");
    if (d <= 0 || dv <= 0) return fail(MKV_ERR_INVALID_ARGUMENT, "decode_attention: query dimension mismatch");
    if (!q || !keys || !values || !out || !attn) return fail(MKV_ERR_INVALID_ARGUMENT, "decode_attention: null tensor");
    if (int r = require_device()) return r;
    DecodeF32Params p{q, keys, values, ld_k, ld_v, n, d, dv, scale, out, attn};
    CK(launch_decode_attn_f32(p, static_cast<cudaStream_t>(stream)));
    return MKV_OK;
}

int mkv_quantize_block_f32(const float* src, int64_t ld, const int32_t* row_idx, int rows, int cols, int gs, int axis,
                           int64_t code_offset, uint32_t first_word, uint32_t* words_out, float* params_out,
                           void* stream) {
    if (rows <= 0 || cols <= 0) return fail(MKV_ERR_INVALID_ARGUMENT, "append_block: empty block");
    if (gs < 1) return fail(MKV_ERR_INVALID_ARGUMENT, "quantize_matrix: group_size must be >= 1");
    if (axis != 0 && axis != 1) return fail(MKV_ERR_INVALID_ARGUMENT, "quantize: axis must be 0 or 1");
    if (!src || !words_out || !params_out || code_offset < 0)
        return fail(MKV_ERR_INVALID_ARGUMENT, "quantize: null tensor");
    if (int r = require_device()) return r;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t n = (int64_t)rows * cols;
    uint8_t* codes = nullptr;
    uint32_t* status = nullptr;
    CK(cudaMallocAsync(&codes, n + 16, s));
    CK(cudaMallocAsync(&status, sizeof(uint32_t), s));
    cudaError_t e = cudaMemsetAsync(status, 0, sizeof(uint32_t), s);
    QuantBlockParams p{src, ld, row_idx, rows, cols, gs, axis, codes, params_out, status};
    if (e == cudaSuccess) e = launch_quantize_block(p, s);
    if (e == cudaSuccess) e = launch_pack_codes(codes, n, code_offset, first_word, words_out, status, s);
    uint32_t st = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&st, status, sizeof(uint32_t), cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(codes, s);
    cudaFreeAsync(status, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "quantize_block");
    if (st & 1u) return fail(MKV_ERR_DOMAIN, "quantize_group: non-finite input");
    if (st & 2u) return fail(MKV_ERR_DOMAIN, "pack_codes: code out of range");
    return MKV_OK;
}

int mkv_dequantize_f32(const uint32_t* words, const float* params, const int64_t* block_rows, int n_blocks, int cols,
                       int gs, int axis, float* out, int64_t ld_out, void* stream) {
    if (n_blocks < 0 || cols <= 0 || gs < 1 || (axis != 0 && axis != 1))
        return fail(MKV_ERR_INVALID_ARGUMENT, "dequantize_matrix: bad layout");
    if (n_blocks == 0) return MKV_OK;
    if (!words || !params || !block_rows || !out) return fail(MKV_ERR_INVALID_ARGUMENT, "dequantize_matrix: null tensor");
    if (int r = require_device()) return r;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    std::vector<DequantBlock> blk(n_blocks);
    int64_t code = 0, group = 0, row = 0;
    for (int b = 0; b < n_blocks; ++b) {
        const int64_t R = block_rows[b];
        if (R <= 0) return fail(MKV_ERR_INVALID_ARGUMENT, "dequantize_matrix: empty block");
        blk[b] = DequantBlock{code, group, row, (int)R, 0};
        code += R * cols;
        group += axis == 0 ? (int64_t)cols * ((R + gs - 1) / gs) : R * ((cols + gs - 1) / gs);
        row += R;
    }
    DequantBlock* d_blk = nullptr;
    CK(cudaMallocAsync(&d_blk, sizeof(DequantBlock) * n_blocks, s));
    cudaError_t e = cudaMemcpyAsync(d_blk, blk.data(), sizeof(DequantBlock) * n_blocks, cudaMemcpyHostToDevice, s);
    DequantParams p{words, params, d_blk, n_blocks, code, cols, gs, axis, out, ld_out};
    if (e == cudaSuccess) e = launch_dequantize(p, s);
    cudaFreeAsync(d_blk, s);
    // the host table must outlive the async copy
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "dequantize");
    return MKV_OK;
}

}  // extern "C"
