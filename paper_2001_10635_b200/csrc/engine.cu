// engine.cu -- host side of the C ABI (include/pirk_c.h).
//
// Restates the reference's method drivers (reach.cpp:65-323) around device
// kernels: validation (system_model.cpp:10-32, interval.cpp:10-23), step
// planning (rk4.cpp:8-17, reach.cpp:28-39), the step loop with last-step
// shortening (rk4.cpp:98-112), recording, and the error contract (messages
// and priorities of reach.cpp:107-117, 181-192, 306-312).  All arithmetic on
// the state runs in the device kernels; the host only plans, launches,
// transfers and formats.  There is no CPU fallback: an unsupported model or
// a missing device is an error.
#include <cuda.h>  // driver types for the entry points taken via cudaGetDriverEntryPoint
#include <cuda_runtime.h>
#include <nvrtc.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#define PIRK_TU_EXACT 1
#include "../../include/pirk_c.h"
#include "common.cuh"
#include "kernels.h"
#include "user_rt.cuh"

using namespace pirk;

// A user-defined model's evaluators (pirk_program_create): source, and per
// arithmetic mode the NVRTC-compiled sm_100a image loaded as a
// context-independent library (user_models.cuh).
struct UserBuild {
    bool tried = false, ok = false;
    std::string log;
    std::vector<char> cubin;
    cudaLibrary_t lib = nullptr;
    cudaKernel_t k_small = nullptr, k_stage = nullptr, k_mc = nullptr, k_tile = nullptr;
    unsigned long long tile_devices = 0;  // devices the tile kernel's smem opt-in is set on
};

struct pirk_program {
    std::string source;
    uint64_t dim = 0, input_dim = 0;
    uint32_t flags = 0;
    uint64_t stencil = 0;  // pirk_program_set_stencil: radius of a 1-D stencil model (0 = unknown)
    std::mutex mu;
    UserBuild build[2];  // [pirk_mode]
    ~pirk_program() {
        for (UserBuild& b : build)
            if (b.lib) cudaLibraryUnload(b.lib);
    }
};

// A block of device memory kept for reuse by the next run of the same size.
struct CachedBlock {
    void* p;
    size_t bytes;
};

// One shard lane of a multi-device context (pirk_create_multi): a device, its
// compute and copy streams and its own state-buffer cache.  Lane 0 is the
// context's primary device/stream (pirk_ctx::device / ::stream).
struct PirkLane {
    int device = 0;
    cudaStream_t stream = nullptr;   // compute (owned)
    cudaStream_t xstream = nullptr;  // halo sends (owned)
    std::vector<CachedBlock> cache;
};

struct pirk_ctx {
    int device = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    cudaStream_t own_xstream = nullptr;  // lane 0's copy stream
    int mode = PIRK_MODE_EXACT;
    std::string err;
    uint64_t launches = 0;
    unsigned long long* d_flags = nullptr;  // scratch device flags [16]
    unsigned long long* h_flags = nullptr;  // pinned mirror
    // state buffers of the last finished run, kept for the next run of the same
    // size: freeing 4 x 32 GB costs up to ~0.5 s of unmapping per call
    std::vector<CachedBlock> cache;
    std::vector<PirkLane> peers;  // lanes 1 .. W-1 (empty for a one-device context)
    bool peer_stores = true;      // every adjacent pair of lanes can address the other's memory
    // streaming observer (pirk_set_record_callback): called per recorded slot
    pirk_record_fn record_fn = nullptr;
    void* record_user = nullptr;
    // catalog vector fields as generated NVRTC sources (Monte Carlo with
    // n > kSmallMax, user_models.cuh), keyed by source
    std::map<std::string, std::unique_ptr<pirk_program>> catalog_programs;
    // every ABI call on a context holds this: calls from several threads on one
    // context serialise instead of racing on err / h_flags / the caches
    std::recursive_mutex mu;
    int lanes() const { return 1 + static_cast<int>(peers.size()); }
    void flush_cache() {
        for (const CachedBlock& b : cache) cudaFree(b.p);
        cache.clear();
    }
    // every lane's cache (device allocations retry after this on OOM)
    void flush_all() {
        flush_cache();
        for (PirkLane& l : peers) {
            for (const CachedBlock& b : l.cache) cudaFree(b.p);
            l.cache.clear();
        }
    }
};

namespace {

using Clock = std::chrono::steady_clock;
double since(Clock::time_point t) { return std::chrono::duration<double>(Clock::now() - t).count(); }

pirk_status fail(pirk_ctx* ctx, pirk_status st, const std::string& msg) {
    if (ctx) ctx->err = msg;
    return st;
}

pirk_status cuda_fail(pirk_ctx* ctx, cudaError_t e, const char* what) {
    const pirk_status st = (e == cudaErrorMemoryAllocation) ? PIRK_ENOMEM : PIRK_ECUDA;
    if (e == cudaErrorMemoryAllocation) cudaGetLastError();  // clear the sticky-free error
    return fail(ctx, st, std::string(what) + ": " + cudaGetErrorString(e));
}

#define LOCK(ctx) std::lock_guard<std::recursive_mutex> lock_guard_((ctx)->mu)

#define CK(ctx, expr)                                                  \
    do {                                                               \
        cudaError_t e_ = (expr);                                       \
        if (e_ != cudaSuccess) return cuda_fail((ctx), e_, #expr);     \
    } while (0)

// std::to_string(double) == "%f" (the reference formats t and radii this way)
std::string fstr(double v) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "%f", v);
    return buf;
}

struct Plan {
    uint64_t full = 0, total = 0;
    bool rem = false;
};

// rk4.cpp:8-17
bool plan_steps(double t0, double t1, double h, Plan& p) {
    if (!(h > 0.0) || !(t0 < t1)) return false;
    const double span = t1 - t0;
    p.full = static_cast<uint64_t>(std::floor(span / h + 1e-9));
    const double remainder = span - static_cast<double>(p.full) * h;
    p.rem = remainder > 1e-9 * h;
    p.total = p.full + (p.rem ? 1 : 0);
    return true;
}

// reach.cpp:28-39
void record_schedule(double t0, double t1, double h, uint64_t stride, const Plan& plan,
                     std::vector<uint64_t>& steps, std::vector<double>& times) {
    steps.clear();
    times.clear();
    if (stride > 0) {
        steps.push_back(0);
        times.push_back(t0);
        for (uint64_t k = stride; k < plan.total; k += stride) {
            steps.push_back(k);
            times.push_back(t0 + static_cast<double>(k) * h);
        }
    }
    steps.push_back(plan.total);
    times.push_back(t1);
}

// rk4.cpp:99-100, 38-39
StepConsts host_step(double t0, double t1, double h, uint64_t k, uint64_t total) {
    StepConsts c;
    c.t = t0 + static_cast<double>(k) * h;
    c.hk = (k + 1 == total) ? t1 - c.t : h;
    c.h2 = 0.5 * c.hk;
    c.h6 = c.hk / 6.0;
    return c;
}

bool is_chain(const pirk_model* m) { return m->kind == PIRK_TRAFFIC || m->kind == PIRK_CHAIN; }
bool is_heat(const pirk_model* m) { return m->kind == PIRK_HEAT3D; }

#ifndef PIRK_CHAIN_FUSE_DEFAULT
// RK4 steps per chain launch in full-domain runs.  Measured (ms per step,
// S = 2 / 3 / 4): fast traffic n=1e6 0.0096 / 0.0111 / 0.0102, n=1e7 0.068 /
// 0.066 / 0.069; fast chain n=1e7 0.087 / 0.082 / 0.086; exact chain 0.144 /
// 0.153 / 0.167.
#define PIRK_CHAIN_FUSE_DEFAULT 2
#endif

// Descriptor consistency (the reference's make_* constructors enforce these,
// models.cpp:47-53, 92-97, and fix dim/input_dim per model).
bool check_model(pirk_ctx* ctx, const pirk_model* m, pirk_status& st) {
    auto bad = [&](const std::string& s) {
        st = fail(ctx, PIRK_EINVAL, "model descriptor: " + s);
        return false;
    };
    if (!m) return bad("null model");
    if (m->dim == 0) {
        st = fail(ctx, PIRK_EINVAL, "problem: model has no dynamics");
        return false;
    }
    switch (m->kind) {
        case PIRK_ZERO:
            if (m->input_dim != 0) return bad("zero model has no inputs");
            break;
        case PIRK_SCALAR_DECAY:
            if (m->dim != 1 || m->input_dim != 1) return bad("scalar-decay is 1-D with 1 input");
            break;
        case PIRK_SCALAR_LINEAR:
            if (m->dim != 1 || m->input_dim != 0) return bad("scalar-linear is 1-D without inputs");
            break;
        case PIRK_TRAFFIC:
            if (m->dim < 3) return bad("traffic model needs at least 3 segments");
            if (m->input_dim != 1) return bad("traffic has one input");
            break;
        case PIRK_HEAT3D:
            if (m->grid < 2 || m->grid * m->grid * m->grid != m->dim)
                return bad("heat3d needs grid >= 2 and dim == grid^3");
            if (m->input_dim != 0) return bad("heat3d has no inputs");
            break;
        case PIRK_CHAIN:
            if (m->input_dim != 1) return bad("chain has one input");
            break;
        case PIRK_LAUB_LOOMIS:
            if (m->dim != 7 || m->input_dim != 0) return bad("laub-loomis is 7-D without inputs");
            break;
        case PIRK_ARCH_QUAD:
            if (m->dim != 12 || m->input_dim != 0) return bad("arch-quadrotor is 12-D without inputs");
            break;
        case PIRK_VDP:
            if (m->dim != 2 || m->input_dim != 0) return bad("vdp is 2-D without inputs");
            break;
        case PIRK_USER:
            if (!m->program) return bad("user model without a program");
            if (m->program->dim != m->dim || m->program->input_dim != m->input_dim)
                return bad("user model dim / input_dim differ from its program's");
            break;
        default:
            return bad("unknown model kind " + std::to_string(m->kind));
    }
    if (m->decomp < PIRK_DECOMP_NONE || m->decomp > PIRK_DECOMP_JACOBIAN)
        return bad("unknown decomposition");
    return true;
}

// Dense growth matrices (models.cpp:457-460, 488-500, 557-611), computed with
// the host libm exactly as the reference constructs them.
bool growth_matrix(const pirk_model* m, double* C) {
    const uint64_t n = m->dim;
    std::memset(C, 0, sizeof(double) * 144);
    if (m->kind == PIRK_VDP) {
        const double mu = m->params[0], op_x = m->params[1], op_y = m->params[2];
        C[0 * 2 + 1] = 1.0;
        C[1 * 2 + 0] = 2.0 * mu * op_x * op_y + 1.0;
        C[1 * 2 + 1] = mu;
        return true;
    }
    if (m->kind == PIRK_LAUB_LOOMIS) {
        const double xm = 5.0;
        const double rows[7][7] = {
            {-0.9, 0, 1.4, 0, 0, 0, 0},     {0, -1.5, 0, 0, 2.5, 0, 0},
            {0, 0.8 * xm, 0, 0, 0, 0, 0.6}, {0, 0, 1.3 * xm, 0, 0, 0, 0},
            {0.7, 0, 0, xm, 0, 0, 0},       {0.3, 0, 0, 0, 0, -3.1, 0},
            {0, 1.5 * xm, 0, 0, 0, 1.8, 0},
        };
        for (uint64_t i = 0; i < 7; ++i)
            for (uint64_t j = 0; j < 7; ++j) C[i * n + j] = rows[i][j];
        return true;
    }
    if (m->kind == PIRK_ARCH_QUAD) {
        const double mass = m->params[0], gravity = m->params[1];
        const double jx = m->params[2], jy = m->params[3], jz = m->params[4];
        const double kx = (jy - jz) / jx, ky = (jz - jx) / jy, kz = (jx - jy) / jz;
        const double vb = 5.0, ab = 0.5, rb = 2.0;
        const double tanb = std::tan(ab);
        const double secb = 1.0 / std::cos(ab);
        const double sec2b = secb * secb;
        const double akx = std::fabs(kx), aky = std::fabs(ky), akz = std::fabs(kz);
        auto c = [&](int r, int col) -> double& { return C[r * 12 + col]; };
        for (int row = 0; row < 3; ++row) {
            c(row, 3) = c(row, 4) = c(row, 5) = 1.0;
            c(row, 6) = c(row, 7) = 6.0 * vb;
            if (row < 2) c(row, 8) = 6.0 * vb;
        }
        c(3, 4) = rb; c(3, 5) = rb; c(3, 7) = gravity; c(3, 10) = vb; c(3, 11) = vb;
        c(4, 3) = rb; c(4, 5) = rb; c(4, 6) = gravity; c(4, 7) = gravity; c(4, 9) = vb; c(4, 11) = vb;
        c(5, 2) = 10.0 / mass; c(5, 3) = rb; c(5, 4) = rb; c(5, 5) = -3.0 / mass;
        c(5, 6) = gravity; c(5, 7) = gravity; c(5, 9) = vb; c(5, 10) = vb;
        c(6, 6) = 2.0 * tanb * rb; c(6, 7) = 2.0 * sec2b * rb; c(6, 9) = 1.0;
        c(6, 10) = tanb; c(6, 11) = tanb;
        c(7, 6) = 2.0 * rb; c(7, 10) = 1.0; c(7, 11) = 1.0;
        c(8, 6) = 2.0 * secb * rb; c(8, 7) = 2.0 * secb * tanb * rb; c(8, 10) = secb; c(8, 11) = secb;
        c(9, 6) = 1.0 / jx; c(9, 9) = -1.0 / jx; c(9, 10) = akx * rb; c(9, 11) = akx * rb;
        c(10, 7) = 1.0 / jy; c(10, 9) = aky * rb; c(10, 10) = -1.0 / jy; c(10, 11) = aky * rb;
        c(11, 9) = akz * rb; c(11, 10) = akz * rb;
        return true;
    }
    return false;
}

bool has_growth(const pirk_model* m) {
    if (m->kind == PIRK_USER) return m->program && (m->program->flags & PIRK_HAS_GROWTH);
    return m->kind == PIRK_ZERO || m->kind == PIRK_SCALAR_DECAY || m->kind == PIRK_SCALAR_LINEAR ||
           m->kind == PIRK_TRAFFIC || m->kind == PIRK_HEAT3D || m->kind == PIRK_LAUB_LOOMIS ||
           m->kind == PIRK_ARCH_QUAD || m->kind == PIRK_VDP;
}

SmallModel small_model(const pirk_model* m) {
    SmallModel s{};
    s.kind = m->kind;
    s.decomp = m->decomp;
    s.n = static_cast<int>(m->dim);
    s.ni = static_cast<int>(m->input_dim);
    s.grid = m->grid;
    for (int i = 0; i < 8; ++i) s.P[i] = m->params[i];
    s.has_C = growth_matrix(m, s.C) ? 1 : 0;
    if (m->kind == PIRK_ARCH_QUAD) {  // uniform divisions hoisted out of every RHS evaluation
        const double mass = m->params[0], jx = m->params[2], jy = m->params[3], jz = m->params[4];
        s.Q[0] = (jy - jz) / jx;
        s.Q[1] = (jz - jx) / jy;
        s.Q[2] = (jx - jy) / jz;
        s.Q[3] = 1.0 / jx;
        s.Q[4] = 1.0 / jy;
        s.Q[5] = 1.0 / mass;
    }
    return s;
}

ChainModel chain_model(const pirk_model* m, int method, double p0, double p1) {
    ChainModel c{};
    c.kind = m->kind;
    c.method = method;
    c.n = m->dim;
    for (int i = 0; i < 8; ++i) c.P[i] = m->params[i];
    c.p0 = p0;
    c.p1 = p1;
    if (m->kind == PIRK_TRAFFIC) {  // models.cpp:55, 79-81
        const double v = m->params[0], w = m->params[1], beta = m->params[5];
        c.inv_t = 1.0 / m->params[4];
        c.a_prev = beta * v * c.inv_t;
        c.a_next = (w / beta) * c.inv_t;
        c.a_in = beta * c.inv_t;
        c.wb = w / beta;
    }
    return c;
}

HeatModel heat_model(const pirk_model* m, int method) {
    HeatModel h{};  // models.cpp:99-101
    h.method = method;
    h.g = m->grid;
    const double delta = 1.0 / static_cast<double>(m->grid - 1);
    h.kk = m->params[0] / (delta * delta);
    h.robin = 2.0 * delta * m->params[1];
    return h;
}

bool small_ok(const pirk_model* m) { return m->dim <= static_cast<uint64_t>(kSmallMax); }

bool has_decomposition(const pirk_model* m) {
    if (m->kind == PIRK_USER) return m->program && (m->program->flags & PIRK_HAS_DECOMPOSITION);
    return m->decomp != PIRK_DECOMP_NONE;
}

// Problem validation (system_model.cpp:10-32) except the per-component box
// checks of large models, which run on the device after upload.
bool check_problem(pirk_ctx* ctx, const pirk_model* m, const pirk_problem* p, bool host_box,
                   pirk_status& st) {
    if (!check_model(ctx, m, st)) return false;
    if (!p || !p->init_lower || !p->init_upper) {
        st = fail(ctx, PIRK_EINVAL, "problem: initial box missing");
        return false;
    }
    if (host_box) {
        for (uint64_t i = 0; i < m->dim; ++i) {
            if (!std::isfinite(p->init_lower[i]) || !std::isfinite(p->init_upper[i])) {
                st = fail(ctx, PIRK_EINVAL, "interval: non-finite bound at component " + std::to_string(i));
                return false;
            }
            if (p->init_lower[i] > p->init_upper[i]) {
                st = fail(ctx, PIRK_EINVAL, "interval: lower > upper at component " + std::to_string(i));
                return false;
            }
        }
    }
    if (m->input_dim == 0) {
        if (p->input_lower || p->input_upper) {
            st = fail(ctx, PIRK_EINVAL, "problem: model has no inputs but an input box was given");
            return false;
        }
    } else {
        if (!p->input_lower || !p->input_upper) {
            st = fail(ctx, PIRK_EINVAL, "problem: model has " + std::to_string(m->input_dim) +
                                            " inputs but no input box was given");
            return false;
        }
        for (uint64_t j = 0; j < m->input_dim; ++j) {
            if (!std::isfinite(p->input_lower[j]) || !std::isfinite(p->input_upper[j])) {
                st = fail(ctx, PIRK_EINVAL, "interval: non-finite bound at component " + std::to_string(j));
                return false;
            }
            if (p->input_lower[j] > p->input_upper[j]) {
                st = fail(ctx, PIRK_EINVAL, "interval: lower > upper at component " + std::to_string(j));
                return false;
            }
        }
    }
    if (!(p->t0 < p->t1)) {
        st = fail(ctx, PIRK_EINVAL, "problem: t0 must be earlier than t1");
        return false;
    }
    if (!(p->h > 0.0)) {
        st = fail(ctx, PIRK_EINVAL, "problem: step size h must be positive");
        return false;
    }
    return true;
}

// cudaMalloc that, on out-of-memory, releases every cached state block of the
// context and tries once more (the cache must never cause an OOM).
cudaError_t dev_malloc(pirk_ctx* ctx, void** p, size_t bytes) {
    cudaError_t e = cudaMalloc(p, bytes);
    if (e == cudaErrorMemoryAllocation && ctx) {
        cudaGetLastError();
        ctx->flush_all();
        e = cudaMalloc(p, bytes);
    }
    return e;
}

template <typename T>
struct DevBuf {
    T* p = nullptr;
    std::vector<CachedBlock>* cache = nullptr;  // set: a state buffer that returns to this cache
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (!p) return;
        if (cache && cache->size() < 8) {
            cache->push_back({p, bytes});
        } else {
            cudaFree(p);
        }
        p = nullptr;
    }
    cudaError_t alloc(pirk_ctx* ctx, size_t count) {
        bytes = count * sizeof(T) + 16;
        return dev_malloc(ctx, reinterpret_cast<void**>(&p), bytes);
    }
    // take a cached block of exactly this size from `c`, else drop `c` (it was
    // sized for another problem) and allocate
    cudaError_t alloc_state(pirk_ctx* ctx, std::vector<CachedBlock>& c, size_t count) {
        bytes = count * sizeof(T) + 16;
        cache = &c;
        for (size_t i = 0; i < c.size(); ++i) {
            if (c[i].bytes == bytes) {
                p = static_cast<T*>(c[i].p);
                c.erase(c.begin() + static_cast<long>(i));
                return cudaSuccess;
            }
        }
        for (const CachedBlock& b : c) cudaFree(b.p);
        c.clear();
        return dev_malloc(ctx, reinterpret_cast<void**>(&p), bytes);
    }
    cudaError_t alloc_state(pirk_ctx* ctx, size_t count) { return alloc_state(ctx, ctx->cache, count); }
};

bool exact_mode(const pirk_ctx* ctx) { return ctx->mode == PIRK_MODE_EXACT; }

// PIRK_STATE_CACHE=0: free the state buffers after every run
bool state_cache_on() {
    static const bool on = [] {
        const char* v = std::getenv("PIRK_STATE_CACHE");
        return !(v && std::strcmp(v, "0") == 0);
    }();
    return on;
}

cudaError_t step_launch(pirk_ctx* ctx, cudaStream_t stream, const pirk_model* m, const ChainModel& cm,
                        const HeatModel& hm, const WindowArgs& w, const StepConsts& sc,
                        uint64_t k, unsigned long long* fail_ptr) {
    ctx->launches++;
    const bool ex = exact_mode(ctx);
    if (is_chain(m))
        return ex ? launch_chain_step<true>(cm, w, sc, k, fail_ptr, stream)
                  : launch_chain_step<false>(cm, w, sc, k, fail_ptr, stream);
    return ex ? launch_heat_step<true>(hm, w, sc, k, fail_ptr, stream)
              : launch_heat_step<false>(hm, w, sc, k, fail_ptr, stream);
}

std::string integ_msg(uint64_t step, uint64_t comp, double t) {
    return "integration produced a non-finite value at step " + std::to_string(step) +
           ", component " + std::to_string(comp) + ", t = " + fstr(t);
}

void fill_report(pirk_report* r, uint64_t n, uint64_t m, uint64_t steps, uint64_t peak,
                 uint64_t dev_bytes, bool exact, double setup, double integ, double red,
                 uint64_t launches) {
    if (!r) return;
    r->n = n;
    r->m = m;
    r->steps = steps;
    r->peak_state_bytes = peak;
    r->device_state_bytes = dev_bytes;
    r->workers = 1;
    r->exact = exact ? 1 : 0;
    r->setup_s = setup;
    r->integration_s = integ;
    r->reduction_s = red;
    r->kernel_launches = launches;
}

}  // namespace

// ============================================================= engine object

struct pirk_engine {
    pirk_ctx* ctx = nullptr;
    pirk_model model{};
    int method = 0;
    Plan plan;
    double t0 = 0, t1 = 0, h = 0;
    uint64_t n = 0, units = 0, unit = 1;
    DevBuf<double> a0, a1, b0, b1;
    int cur = 0;               // 0: state in (a0,a1); 1: in (b0,b1)
    bool cache_state = false;  // one-shot runs: state buffers go back to ctx->cache
    uint64_t done = 0;
    DevBuf<unsigned long long> d_fail;  // [2]
    ChainModel cm{};
    HeatModel hm{};
    double* s0() { return cur ? b0.p : a0.p; }
    double* s1() { return cur ? b1.p : a1.p; }
    double* o0() { return cur ? a0.p : b0.p; }
    double* o1() { return cur ? a1.p : b1.p; }
};

namespace {

pirk_status engine_init(pirk_ctx* ctx, const pirk_model* m, int method, const pirk_problem* p,
                        pirk_engine* e) {
    e->ctx = ctx;
    e->model = *m;
    e->method = method;
    e->t0 = p->t0;
    e->t1 = p->t1;
    e->h = p->h;
    plan_steps(p->t0, p->t1, p->h, e->plan);
    if (e->plan.total >= (1ull << 23))
        return fail(ctx, PIRK_EINVAL, "step count exceeds the device failure-key range (2^23)");
    e->n = m->dim;
    e->unit = is_heat(m) ? m->grid * m->grid : 1;
    e->units = e->n / e->unit;
    if (2 * e->n >= (1ull << kFailCompBits))
        return fail(ctx, PIRK_EINVAL, "dimension exceeds the device failure-key range");
    double p0 = 0.0, p1 = 0.0;
    if (m->input_dim > 0) {
        if (method == PIRK_METHOD_MM) {
            p0 = p->input_lower[0];
            p1 = p->input_upper[0];
        } else {  // interval.cpp:25-37 center / half-width
            p0 = 0.5 * (p->input_upper[0] + p->input_lower[0]);
            p1 = 0.5 * (p->input_upper[0] - p->input_lower[0]);
        }
    }
    e->cm = chain_model(m, method, p0, p1);
    e->hm = heat_model(m, method);
    const size_t n = e->n;
    if (e->cache_state && state_cache_on()) {
        CK(ctx, e->a0.alloc_state(ctx, n));
        CK(ctx, e->a1.alloc_state(ctx, n));
        CK(ctx, e->b0.alloc_state(ctx, n));
        CK(ctx, e->b1.alloc_state(ctx, n));
    } else {
        CK(ctx, e->a0.alloc(ctx, n));
        CK(ctx, e->a1.alloc(ctx, n));
        CK(ctx, e->b0.alloc(ctx, n));
        CK(ctx, e->b1.alloc(ctx, n));
    }
    CK(ctx, e->d_fail.alloc(ctx, 2));
    CK(ctx, cudaMemsetAsync(e->d_fail.p, 0xff, 2 * sizeof(unsigned long long), ctx->stream));
    CK(ctx, cudaMemcpyAsync(e->a0.p, p->init_lower, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    CK(ctx, cudaMemcpyAsync(e->a1.p, p->init_upper, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    // IntervalVector validation of the uploaded box, on the device
    CK(ctx, cudaMemsetAsync(ctx->d_flags, 0xff, sizeof(unsigned long long), ctx->stream));
    CK(ctx, launch_box_check(e->a0.p, e->a1.p, n, ctx->d_flags, ctx->stream));
    ctx->launches++;
    CK(ctx, cudaMemcpyAsync(ctx->h_flags, ctx->d_flags, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
    CK(ctx, cudaStreamSynchronize(ctx->stream));
    if (ctx->h_flags[0] != kNoFail) {
        const uint64_t i = ctx->h_flags[0];
        const bool nonfinite = !std::isfinite(p->init_lower[i]) || !std::isfinite(p->init_upper[i]);
        return fail(ctx, PIRK_EINVAL, std::string(nonfinite ? "interval: non-finite bound at component "
                                                            : "interval: lower > upper at component ") +
                                          std::to_string(i));
    }
    if (method == PIRK_METHOD_GB) {
        CK(ctx, launch_center_radius(e->a0.p, e->a1.p, n, ctx->stream));
        ctx->launches++;
    }
    e->cur = 0;
    e->done = 0;
    return PIRK_OK;
}

// Full-domain chain runs advance two RK4 steps per launch (chain_warp_kernel
// with S = 2: twice the halo, half the HBM round trips).  PIRK_CHAIN_FUSE=0 or
// PIRK_CHAIN_KERNEL=smem keep one step per launch.
int chain_fuse_steps() {  // PIRK_CHAIN_FUSE=0|1 (off), 2..4
    static const int v = [] {
        const char* f = std::getenv("PIRK_CHAIN_FUSE");
        const char* k = std::getenv("PIRK_CHAIN_KERNEL");
        if (k && std::strcmp(k, "smem") == 0) return 1;
        if (!f) return PIRK_CHAIN_FUSE_DEFAULT;
        const int n = std::atoi(f);
        return n < 1 ? 1 : (n > 4 ? 4 : n);
    }();
    return v;
}

pirk_status engine_advance(pirk_engine* e, uint64_t nsteps) {
    pirk_ctx* ctx = e->ctx;
    uint64_t left = nsteps;
    // measured (n = 1e7, ms per step, 1 vs 2 steps per launch): fast traffic
    // 0.092 -> 0.067, fast chain 0.099 -> 0.087, exact chain 0.153 -> 0.144;
    // exact traffic 0.158 -> 0.165 (register pressure), so it stays at one
    const int S = (is_chain(&e->model) && (!exact_mode(ctx) || e->model.kind == PIRK_CHAIN)) ? chain_fuse_steps() : 1;
    while (S >= 2 && left >= 2 && e->done + 2 <= e->plan.total) {
        const uint64_t k = e->done;
        int s_now = S;
        while (s_now > left || e->done + s_now > e->plan.total) --s_now;
        if (s_now < 2) break;
        StepConstsN scs;
        for (int q = 0; q < s_now; ++q) scs.s[q] = host_step(e->t0, e->t1, e->h, k + q, e->plan.total);
        WindowArgs w{e->s0(), e->s1(), e->o0(), e->o1(), 0, e->units, 0, e->units};
        ctx->launches++;
        CK(ctx, exact_mode(ctx) ? launch_chain_steps<true>(e->cm, w, scs, s_now, k, e->d_fail.p, ctx->stream)
                                : launch_chain_steps<false>(e->cm, w, scs, s_now, k, e->d_fail.p, ctx->stream));
        e->cur ^= 1;
        e->done += s_now;
        left -= s_now;
    }
    for (uint64_t i = 0; i < left && e->done < e->plan.total; ++i) {
        const uint64_t k = e->done;
        const StepConsts sc = host_step(e->t0, e->t1, e->h, k, e->plan.total);
        WindowArgs w{e->s0(), e->s1(), e->o0(), e->o1(), 0, e->units, 0, e->units};
        CK(ctx, step_launch(ctx, ctx->stream, &e->model, e->cm, e->hm, w, sc, k, e->d_fail.p));
        e->cur ^= 1;
        e->done++;
    }
    return PIRK_OK;
}

// RAII for the pipelined path's extra stream and events
struct StreamGuard {
    cudaStream_t s = nullptr;
    ~StreamGuard() { if (s) cudaStreamDestroy(s); }
};
struct EventGuard {
    EventGuard() = default;
    EventGuard(const EventGuard&) = delete;
    EventGuard& operator=(const EventGuard&) = delete;
    cudaEvent_t e = nullptr;
    ~EventGuard() { if (e) cudaEventDestroy(e); }
};

// The launcher's kernel choice can be overridden (PIRK_HEAT_BLOCK); one-field
// launches need the strip kernel.
// every step of the plan can run the fast strip kernel (its S form needs
// z = hk*kk in range; a tiny remainder step does not qualify)
bool heat_plan_strip_ok(const pirk_model* m, const pirk_problem* p, const Plan& pl) {
    const HeatModel hm = heat_model(m, PIRK_METHOD_MM);
    if (pl.total == 0) return true;
    if (pl.total > 1 && !heat_strip_step_ok(hm, host_step(p->t0, p->t1, p->h, 0, pl.total).hk)) return false;
    return heat_strip_step_ok(hm, host_step(p->t0, p->t1, p->h, pl.total - 1, pl.total).hk);
}

bool heat_single_field_ok() {
    const char* v = std::getenv("PIRK_HEAT_BLOCK");
    return !v || std::strcmp(v, "strip") == 0;
}

// Fronts of the skewed ("wavefront") schedule of one field in the
// field-pipelined driver.  Round r advances step k (state k -> k+1) over the
// z-planes [front(r-1) - 4k, front(r) - 4k), clamped to [0, U); the last front
// F = U + 4(K-1) completes every step.  Field 0 starts with a front of S0
// planes and doubles it while it stays within U/2, then completes: integration
// starts once the first S0+4 planes are on the device (not the whole 33 GB
// field) and the completing round still runs wide strips.  Field 1 completes
// in J tail rounds of S planes, so its final box leaves the device S planes at
// a time while the rest integrates.  Narrow strips cost wave quantisation and
// pipeline fill per launch, so S trades that against the exposed first upload
// and last download.  PIRK_SKEW=0: one round (full-field launches);
// PIRK_SKEW_S / _S0 / _J override S, S0, J (A/B).
std::vector<uint64_t> skew_fronts(int field, uint64_t U, uint64_t K) {
    const uint64_t F = U + 4 * (K - 1);
    auto env = [](const char* name) -> long long {
        const char* v = std::getenv(name);
        return v ? std::atoll(v) : 0ll;
    };
    static const bool off = [] {
        const char* v = std::getenv("PIRK_SKEW");
        return v && std::strcmp(v, "0") == 0;
    }();
    static const long long s_env = env("PIRK_SKEW_S"), s0_env = env("PIRK_SKEW_S0"), j_env = env("PIRK_SKEW_J");
    if (off) return {F};
    const uint64_t S = s_env > 0 ? static_cast<uint64_t>(s_env) : std::max<uint64_t>(64, (U / 8 + 3) & ~3ull);
    const uint64_t S0 = s0_env > 0 ? static_cast<uint64_t>(s0_env) : S;
    const uint64_t J = j_env > 0 ? static_cast<uint64_t>(j_env) : 3;
    std::vector<uint64_t> fr;
    if (field == 0) {
        for (uint64_t P = S0; P < F && (fr.empty() || P <= U / 2); P *= 2) fr.push_back(P);
    } else {
        for (uint64_t j = J; j >= 1; --j)
            if (F > j * S && F - j * S > (fr.empty() ? 0 : fr.back())) fr.push_back(F - j * S);
    }
    fr.push_back(F);
    return fr;
}

// heat3d CTMM recording only the final box (tube_stride 0).  The embedding's
// halves are independent (cooperative decomposition, models.cpp:20-27, and the
// heat field reads no input), so each field is integrated on its own, and the
// PCIe transfers hide behind the integration:
//   h2d:     lo (in slabs) | hi, box check
//   compute:   steps lo (skewed rounds)  | steps hi (skewed tail) | order check
//   d2h:           final planes of lo as rounds finish  | of hi ...
// Within a field the rounds of skew_fronts() let integration start on the
// first planes of the lower field while the rest uploads, and let the upper
// field's final planes download while its last planes integrate.  Every
// plane's state k+1 is computed by the same kernel from the same state-k
// planes as in a full-field launch (step k of round r reads state k on
// [lo - 4, hi + 4): computed by step k-1 of this round, and not yet
// overwritten by step k+1, whose front lags by 4 planes), so results and
// failure keys (field-1 keys carry +n as in the two-field launch) are those of
// run_large.
pirk_status run_heat_mm_pipelined(pirk_ctx* ctx, const pirk_model* m, const pirk_problem* p,
                                  pirk_tube* tube, pirk_report* rep) {
    const auto t_setup = Clock::now();
    static const bool trace = std::getenv("PIRK_TRACE") != nullptr;
    auto mark = [&](const char* what) {
        if (trace) std::fprintf(stderr, "[pirk] %-24s %8.3f s\n", what, since(t_setup));
    };
    const uint64_t launches0 = ctx->launches;
    pirk_engine e;
    e.ctx = ctx;
    e.model = *m;
    e.method = PIRK_METHOD_MM;
    e.t0 = p->t0;
    e.t1 = p->t1;
    e.h = p->h;
    plan_steps(p->t0, p->t1, p->h, e.plan);
    if (e.plan.total >= (1ull << 23))
        return fail(ctx, PIRK_EINVAL, "step count exceeds the device failure-key range (2^23)");
    e.n = m->dim;
    e.unit = m->grid * m->grid;
    e.units = e.n / e.unit;
    if (2 * e.n >= (1ull << kFailCompBits))
        return fail(ctx, PIRK_EINVAL, "dimension exceeds the device failure-key range");
    e.hm = heat_model(m, PIRK_METHOD_MM);
    const size_t n = e.n;
    const uint64_t U = e.units, K = e.plan.total, unit = e.unit;
    const bool cache = state_cache_on();
    CK(ctx, cache ? e.a0.alloc_state(ctx, n) : e.a0.alloc(ctx, n));
    CK(ctx, cache ? e.a1.alloc_state(ctx, n) : e.a1.alloc(ctx, n));
    CK(ctx, cache ? e.b0.alloc_state(ctx, n) : e.b0.alloc(ctx, n));
    CK(ctx, cache ? e.b1.alloc_state(ctx, n) : e.b1.alloc(ctx, n));
    CK(ctx, e.d_fail.alloc(ctx, 2));
    DevBuf<unsigned long long> flag;  // [0] box check, [1] order check
    CK(ctx, flag.alloc(ctx, 2));
    StreamGuard xs, ds;  // host->device, device->host
    CK(ctx, cudaStreamCreateWithFlags(&xs.s, cudaStreamNonBlocking));
    CK(ctx, cudaStreamCreateWithFlags(&ds.s, cudaStreamNonBlocking));
    const std::vector<uint64_t> fronts[2] = {skew_fronts(0, U, K), skew_fronts(1, U, K)};
    std::vector<EventGuard> ev_up(fronts[0].size() + 1), ev_done(fronts[0].size() + fronts[1].size());
    EventGuard ev_x;
    for (EventGuard& g : ev_up) CK(ctx, cudaEventCreateWithFlags(&g.e, cudaEventDisableTiming));
    for (EventGuard& g : ev_done) CK(ctx, cudaEventCreateWithFlags(&g.e, cudaEventDisableTiming));
    CK(ctx, cudaEventCreateWithFlags(&ev_x.e, cudaEventDisableTiming));
    cudaStream_t cs = ctx->stream;
    CK(ctx, cudaMemsetAsync(e.d_fail.p, 0xff, 2 * sizeof(unsigned long long), cs));
    CK(ctx, cudaMemsetAsync(flag.p, 0xff, 2 * sizeof(unsigned long long), cs));
    mark("allocated");
    CK(ctx, cudaEventRecord(ev_x.e, cs));
    CK(ctx, cudaStreamWaitEvent(xs.s, ev_x.e, 0));
    CK(ctx, cudaStreamWaitEvent(ds.s, ev_x.e, 0));
    // lower field in slabs: round r of field 0 needs planes [0, front_r + 4)
    uint64_t up = 0;
    for (size_t r = 0; r < fronts[0].size(); ++r) {
        const uint64_t end = std::min<uint64_t>(U, fronts[0][r] + 4);
        if (end > up) {
            CK(ctx, cudaMemcpyAsync(e.a0.p + up * unit, p->init_lower + up * unit, (end - up) * unit * sizeof(double),
                                    cudaMemcpyHostToDevice, xs.s));
            up = end;
        }
        CK(ctx, cudaEventRecord(ev_up[r].e, xs.s));
    }
    CK(ctx, cudaMemcpyAsync(e.a1.p, p->init_upper, n * sizeof(double), cudaMemcpyHostToDevice, xs.s));
    CK(ctx, launch_box_check(e.a0.p, e.a1.p, n, flag.p, xs.s));  // interval.cpp:14-22
    ctx->launches++;
    CK(ctx, cudaEventRecord(ev_up.back().e, xs.s));
    mark("uploads enqueued");
    const double setup_s = since(t_setup);

    const auto t_int = Clock::now();
    double* fin[2] = {nullptr, nullptr};
    size_t ne = 0;
    auto clampU = [&](uint64_t P, uint64_t k) -> uint64_t {
        const uint64_t d = 4 * k;
        return P <= d ? 0 : std::min<uint64_t>(U, P - d);
    };
    for (int f = 0; f < 2; ++f) {
        double* buf[2] = {f == 0 ? e.a0.p : e.a1.p, f == 0 ? e.b0.p : e.b1.p};
        fin[f] = buf[K % 2];
        double* host = f == 0 ? tube->lower : tube->upper;
        uint64_t prev = 0;
        for (size_t r = 0; r < fronts[f].size(); ++r) {
            const uint64_t P = fronts[f][r];
            if (f == 0) CK(ctx, cudaStreamWaitEvent(cs, ev_up[r].e, 0));
            else if (r == 0) CK(ctx, cudaStreamWaitEvent(cs, ev_up.back().e, 0));
            for (uint64_t k = 0; k < K; ++k) {
                const uint64_t lo = clampU(prev, k), hi = clampU(P, k);
                if (lo >= hi) continue;
                const StepConsts sc = host_step(e.t0, e.t1, e.h, k, K);
                double* in = buf[k % 2];
                double* out = buf[(k + 1) % 2] + lo * unit;
                WindowArgs w{in, in, out, out, 0, U, lo, hi};
                ctx->launches++;
                CK(ctx, exact_mode(ctx) ? launch_heat_step<true>(e.hm, w, sc, k, e.d_fail.p, cs, f)
                                        : launch_heat_step<false>(e.hm, w, sc, k, e.d_fail.p, cs, f));
            }
            // planes whose last step ran in this round leave the device now
            const uint64_t flo = clampU(prev, K - 1), fhi = clampU(P, K - 1);
            if (flo < fhi) {
                CK(ctx, cudaEventRecord(ev_done[ne].e, cs));
                CK(ctx, cudaStreamWaitEvent(ds.s, ev_done[ne].e, 0));
                ++ne;
                CK(ctx, cudaMemcpyAsync(host + flo * unit, fin[f] + flo * unit, (fhi - flo) * unit * sizeof(double),
                                        cudaMemcpyDeviceToHost, ds.s));
            }
            prev = P;
        }
    }
    CK(ctx, launch_order_check(fin[0], fin[1], n, flag.p + 1, cs));  // reach.cpp:181-186
    ctx->launches++;
    unsigned long long hf[4];
    CK(ctx, cudaMemcpyAsync(hf, e.d_fail.p, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, cs));
    CK(ctx, cudaMemcpyAsync(hf + 2, flag.p, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, cs));
    mark("all enqueued");
    CK(ctx, cudaStreamSynchronize(cs));
    mark("compute stream done");
    CK(ctx, cudaStreamSynchronize(xs.s));
    CK(ctx, cudaStreamSynchronize(ds.s));
    mark("copy streams done");
    const double integ_s = since(t_int);

    if (hf[2] != kNoFail) {  // the box is validated before anything else (interval.cpp:14-22)
        const uint64_t i = hf[2];
        const bool nonfinite = !std::isfinite(p->init_lower[i]) || !std::isfinite(p->init_upper[i]);
        return fail(ctx, PIRK_EINVAL, std::string(nonfinite ? "interval: non-finite bound at component "
                                                            : "interval: lower > upper at component ") +
                                          std::to_string(i));
    }
    tube->n_slots = 1;
    if (tube->times) tube->times[0] = p->t1;
    if (hf[0] != kNoFail) {
        const uint64_t fs = hf[0] >> kFailCompBits, fc = hf[0] & ((1ull << kFailCompBits) - 1);
        return fail(ctx, PIRK_EINTEGRATION, "mixed-monotonicity embedding integration: " +
                                                integ_msg(fs, fc, p->t0 + static_cast<double>(fs) * p->h));
    }
    if (hf[3] != kNoFail)
        return fail(ctx, PIRK_EORDER, "mixed-monotonicity: embedding order violated at step " +
                                          std::to_string(e.plan.total) + ", t = " + fstr(p->t1) +
                                          ", component " + std::to_string(hf[3]));
    if (ctx->record_fn) ctx->record_fn(ctx->record_user, 0, e.plan.total, p->t1, tube->lower, tube->upper, n);
    fill_report(rep, n, 0, e.plan.total, 7 * 2 * n * sizeof(double), 4 * n * sizeof(double), exact_mode(ctx),
                setup_s, integ_s, 0.0, ctx->launches - launches0);
    return PIRK_OK;
}

// Streams recorded slots to the context's record callback (the StepObserver of
// rk4.hpp:63-64, invoked at rk4.cpp:106-111): slot s's box is copied into one
// page-locked staging buffer (lower | upper) on the lanes' streams, and the
// callback for slot s runs on the host while the device integrates towards
// slot s+1 -- the driver enqueues those steps before delivering s.  Order per
// slot: steps(s+1) enqueued, deliver(s) (waits for copy(s), calls back), then
// copy(s+1) may reuse the buffer.
struct SlotStreamer {
    pirk_ctx* ctx = nullptr;
    uint64_t n = 0;
    double* buf = nullptr;  // pinned, 2n
    std::vector<cudaEvent_t> ev;
    int64_t pending = -1;
    uint64_t pend_step = 0;
    double pend_t = 0.0;
    bool on() const { return buf != nullptr; }
    cudaError_t init(pirk_ctx* c, uint64_t n_, int lanes) {
        ctx = c;
        n = n_;
        if (!c->record_fn) return cudaSuccess;
        cudaError_t e = cudaMallocHost(reinterpret_cast<void**>(&buf), 2 * n * sizeof(double));
        if (e != cudaSuccess) {
            buf = nullptr;
            return e;
        }
        ev.assign(static_cast<size_t>(lanes), nullptr);
        for (cudaEvent_t& x : ev)
            if ((e = cudaEventCreateWithFlags(&x, cudaEventDisableTiming)) != cudaSuccess) return e;
        return cudaSuccess;
    }
    // the slot's copies are enqueued on lane r's stream: mark them
    cudaError_t mark(int r, cudaStream_t st) { return cudaEventRecord(ev[static_cast<size_t>(r)], st); }
    cudaError_t deliver() {
        if (pending < 0) return cudaSuccess;
        for (cudaEvent_t x : ev) {
            const cudaError_t e = cudaEventSynchronize(x);
            if (e != cudaSuccess) return e;
        }
        ctx->record_fn(ctx->record_user, static_cast<uint64_t>(pending), pend_step, pend_t, buf, buf + n, n);
        pending = -1;
        return cudaSuccess;
    }
    void set_pending(uint64_t s, uint64_t step, double t) {
        pending = static_cast<int64_t>(s);
        pend_step = step;
        pend_t = t;
    }
    ~SlotStreamer() {
        for (cudaEvent_t x : ev)
            if (x) cudaEventDestroy(x);
        if (buf) cudaFreeHost(buf);
    }
};

// Host-side tubes (small systems, Monte Carlo): every slot to the callback
// after the run, from host memory.
void stream_host_tube(pirk_ctx* ctx, const std::vector<uint64_t>& slot_steps, const std::vector<double>& slot_times,
                      const double* lower, const double* upper, uint64_t n) {
    if (!ctx->record_fn || !lower || !upper) return;
    for (uint64_t s = 0; s < slot_steps.size(); ++s)
        ctx->record_fn(ctx->record_user, s, slot_steps[s], slot_times[s], lower + s * n, upper + s * n, n);
}

// The error contract of a finished large-model run, in the reference's order
// of detection (reach.cpp:107-117, 121-134, 181-192), and the report.  f0/f1:
// the minimum failure keys of the two fields; flags/vals: per recorded slot
// the minimum violating component (order / negative radius) and its radius.
pirk_status large_errors(pirk_ctx* ctx, int method, const pirk_problem* p, uint64_t total,
                         const std::vector<uint64_t>& slot_steps, const std::vector<double>& slot_times,
                         unsigned long long f0, unsigned long long f1,
                         const std::vector<unsigned long long>& flags, const std::vector<double>& vals,
                         uint64_t n, uint64_t dev_bytes, double setup_s, double integ_s,
                         uint64_t launches, int workers, pirk_report* rep) {
    const uint64_t S = slot_steps.size();
    auto decode = [](unsigned long long key, uint64_t& step, uint64_t& comp) {
        step = key >> kFailCompBits;
        comp = key & ((1ull << kFailCompBits) - 1);
    };
    if (method == PIRK_METHOD_MM) {
        uint64_t fs = 0, fc = 0;
        if (f0 != kNoFail) decode(f0, fs, fc);
        for (uint64_t s = 0; s < S; ++s) {
            // an integration failure in step k is raised before slot k+1 is observed
            if (f0 != kNoFail && fs < slot_steps[s])
                return fail(ctx, PIRK_EINTEGRATION, "mixed-monotonicity embedding integration: " +
                                                        integ_msg(fs, fc, p->t0 + static_cast<double>(fs) * p->h));
            if (flags[s] != kNoFail)
                return fail(ctx, PIRK_EORDER, "mixed-monotonicity: embedding order violated at step " +
                                                  std::to_string(slot_steps[s]) + ", t = " + fstr(slot_times[s]) +
                                                  ", component " + std::to_string(flags[s]));
        }
        if (f0 != kNoFail)
            return fail(ctx, PIRK_EINTEGRATION, "mixed-monotonicity embedding integration: " +
                                                    integ_msg(fs, fc, p->t0 + static_cast<double>(fs) * p->h));
        fill_report(rep, n, 0, total, 7 * 2 * n * sizeof(double), dev_bytes, exact_mode(ctx), setup_s,
                    integ_s, 0.0, launches);
    } else {
        // center integration runs to completion before the radius integration
        // (reach.cpp:103-117), and the clamp pass follows both (reach.cpp:121-134)
        uint64_t fs = 0, fc = 0;
        if (f0 != kNoFail) {
            decode(f0, fs, fc);
            return fail(ctx, PIRK_EINTEGRATION, "growth-bound center integration: " +
                                                    integ_msg(fs, fc, p->t0 + static_cast<double>(fs) * p->h));
        }
        if (f1 != kNoFail) {
            decode(f1, fs, fc);
            return fail(ctx, PIRK_EINTEGRATION, "growth-bound radius integration: " +
                                                    integ_msg(fs, fc, p->t0 + static_cast<double>(fs) * p->h));
        }
        for (uint64_t s = 0; s < S; ++s)
            if (flags[s] != kNoFail)
                return fail(ctx, PIRK_ENEGRADIUS, "growth-bound: deviation went negative (" + fstr(vals[s]) +
                                                      ") at component " + std::to_string(flags[s]) +
                                                      "; contraction matrix is invalid");
        fill_report(rep, n, 0, total, 7 * n * sizeof(double), dev_bytes, exact_mode(ctx), setup_s, integ_s,
                    0.0, launches);
    }
    if (rep) rep->workers = workers;
    return PIRK_OK;
}

// Large-model (chain / heat kernels) MM and GB driver.
pirk_status run_large(pirk_ctx* ctx, const pirk_model* m, int method, const pirk_problem* p,
                      pirk_tube* tube, pirk_report* rep) {
    {   // heat3d CTMM with only the final box: field-pipelined transfers
        Plan pl;
        plan_steps(p->t0, p->t1, p->h, pl);
        std::vector<uint64_t> ss;
        std::vector<double> st;
        record_schedule(p->t0, p->t1, p->h, p->tube_stride, pl, ss, st);
        static const bool pipelined = [] {
            const char* v = std::getenv("PIRK_PIPELINE");
            return !(v && std::strcmp(v, "0") == 0);
        }();
        if (pipelined && is_heat(m) && method == PIRK_METHOD_MM && ss.size() == 1 && tube && tube->lower &&
            tube->upper && tube->max_slots >= 1 && m->dim >= (1ull << 22) && !exact_mode(ctx) &&
            m->grid % 2 == 0 && heat_single_field_ok() && heat_plan_strip_ok(m, p, pl))
            return run_heat_mm_pipelined(ctx, m, p, tube, rep);
    }
    const auto t_setup = Clock::now();
    const uint64_t launches0 = ctx->launches;
    pirk_engine e;
    e.cache_state = true;
    pirk_status st = engine_init(ctx, m, method, p, &e);
    if (st != PIRK_OK) return st;
    std::vector<uint64_t> slot_steps;
    std::vector<double> slot_times;
    record_schedule(p->t0, p->t1, p->h, p->tube_stride, e.plan, slot_steps, slot_times);
    const uint64_t S = slot_steps.size();
    if (tube && tube->max_slots < S)
        return fail(ctx, PIRK_EINVAL, "tube: max_slots " + std::to_string(tube->max_slots) +
                                          " < record slots " + std::to_string(S));
    DevBuf<unsigned long long> slot_flag;  // per slot: order (MM) / negative radius (GB)
    DevBuf<double> slot_val;
    CK(ctx, slot_flag.alloc(ctx, S));
    CK(ctx, slot_val.alloc(ctx, S));
    CK(ctx, cudaMemsetAsync(slot_flag.p, 0xff, S * sizeof(unsigned long long), ctx->stream));
    CK(ctx, cudaStreamSynchronize(ctx->stream));
    const double setup_s = since(t_setup);

    const auto t_int = Clock::now();
    const uint64_t n = e.n;
    SlotStreamer rec;
    CK(ctx, rec.init(ctx, n, 1));
    for (uint64_t s = 0; s < S; ++s) {
        st = engine_advance(&e, slot_steps[s] - e.done);
        if (st != PIRK_OK) return st;
        CK(ctx, rec.deliver());  // slot s-1 to the callback while these steps run
        const double* out_lo = e.s0();
        const double* out_hi = e.s1();
        if (method == PIRK_METHOD_MM) {
            CK(ctx, launch_order_check(e.s0(), e.s1(), n, slot_flag.p + s, ctx->stream));
        } else {
            // the free ping-pong buffers receive the clamped box
            CK(ctx, launch_gb_box(e.s0(), e.s1(), e.o0(), e.o1(), n, slot_flag.p + s, ctx->stream));
            CK(ctx, launch_gb_negval(e.s1(), slot_flag.p + s, slot_val.p + s, ctx->stream));
            ctx->launches++;
            out_lo = e.o0();
            out_hi = e.o1();
        }
        ctx->launches++;
        if (tube && tube->lower)
            CK(ctx, cudaMemcpyAsync(tube->lower + s * n, out_lo, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        if (tube && tube->upper)
            CK(ctx, cudaMemcpyAsync(tube->upper + s * n, out_hi, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        if (rec.on()) {
            CK(ctx, cudaMemcpyAsync(rec.buf, out_lo, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
            CK(ctx, cudaMemcpyAsync(rec.buf + n, out_hi, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
            CK(ctx, rec.mark(0, ctx->stream));
            rec.set_pending(s, slot_steps[s], slot_times[s]);
        }
    }
    CK(ctx, rec.deliver());
    std::vector<unsigned long long> flags(S);
    std::vector<double> vals(S);
    CK(ctx, cudaMemcpyAsync(ctx->h_flags, e.d_fail.p, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
    CK(ctx, cudaMemcpyAsync(flags.data(), slot_flag.p, S * sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
    CK(ctx, cudaMemcpyAsync(vals.data(), slot_val.p, S * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(ctx, cudaStreamSynchronize(ctx->stream));
    const double integ_s = since(t_int);

    if (tube) {
        tube->n_slots = S;
        if (tube->times)
            for (uint64_t s = 0; s < S; ++s) tube->times[s] = slot_times[s];
    }
    return large_errors(ctx, method, p, e.plan.total, slot_steps, slot_times, ctx->h_flags[0],
                        ctx->h_flags[1], flags, vals, n, 4 * n * sizeof(double), setup_s, integ_s,
                        ctx->launches - launches0, 1, rep);
}

// ------------------------------------------------ multi-lane (state-sharded) driver
//
// A context made by pirk_create_multi owns W lanes (device + compute stream +
// copy stream).  Chains shard contiguous component ranges, heat3d contiguous
// z-slabs (models.cpp:110-112), exactly as sharded.py does across processes.
// Each lane keeps a window of its units plus a 4-unit halo per side (the RK4
// dependency cone of a radius-1 stencil) and exchanges halos every step.  By
// default ONE launch per lane and step computes its owned units and stores the
// first / last 4 of them a second time into the neighbours' halos over NVLink
// peer memory (WindowArgs::mir0/1, mirh0/1):
//
//   lane stream:  wait(neighbours' step k-1) | owned units (+ edge units to the neighbours)
//
// PIRK_LANE_SCHEDULE=split runs the boundary units as separate launches first
// (their stores overlap the interior launch); PIRK_LANE_HALO=copy, or lanes
// without peer access, send them with copy-engine peer copies instead:
//
//   lane stream:  wait(halos of step k-1) | boundary units (+ peer stores) | interior ....
//   lane copies:                          | (copy mode) send boundary -> neighbours' halos
//
// In the split schedules the boundary units (the ones the neighbours need next
// step) are computed first, their transfer overlaps the interior, and the next
// step waits only for the copies (double-buffered events: a lane waits on
// its neighbours' step-(k-1) records, never on the current ones).  Every unit
// is computed once from the same inputs as on one device, so the result is
// bit-identical for any lane count, and lanes on the SAME device (a repeated
// device id) run the identical code path with device-local copies -- which is
// how the path is tested on a one-GPU box.
struct LaneRef {
    int device;
    cudaStream_t s, xs;
    std::vector<CachedBlock>* cache;
};

LaneRef lane_ref(pirk_ctx* ctx, int r) {
    if (r == 0) return {ctx->device, ctx->stream, ctx->own_xstream, &ctx->cache};
    PirkLane& l = ctx->peers[static_cast<size_t>(r - 1)];
    return {l.device, l.stream, l.xstream, &l.cache};
}

struct ShardState {
    LaneRef L{};
    uint64_t b = 0, e = 0, wb = 0, we = 0;  // owned units [b, e), window [wb, we)
    DevBuf<double> a0, a1, b0, b1;
    DevBuf<unsigned long long> fail, slot_flag, box_flag;
    DevBuf<double> slot_val;
    int cur = 0;
    cudaEvent_t bnd = nullptr, sent[2] = {nullptr, nullptr};
    double* in0() { return cur ? b0.p : a0.p; }
    double* in1() { return cur ? b1.p : a1.p; }
    double* out0() { return cur ? a0.p : b0.p; }
    double* out1() { return cur ? a1.p : b1.p; }
    ~ShardState() {
        for (cudaEvent_t ev : {bnd, sent[0], sent[1]})
            if (ev) cudaEventDestroy(ev);
    }
};

// lanes a run of `units` partition units can use: >= 8 units per lane, so a
// 4-unit halo always comes from the adjacent lane alone
int usable_lanes(const pirk_ctx* ctx, uint64_t units) {
    const uint64_t w = std::min<uint64_t>(static_cast<uint64_t>(ctx->lanes()), units / 8);
    return w < 1 ? 1 : static_cast<int>(w);
}

pirk_status run_large_multi(pirk_ctx* ctx, const pirk_model* m, int method, const pirk_problem* p,
                            pirk_tube* tube, pirk_report* rep) {
    const auto t_setup = Clock::now();
    const uint64_t launches0 = ctx->launches;
    Plan plan;
    plan_steps(p->t0, p->t1, p->h, plan);
    if (plan.total >= (1ull << 23))
        return fail(ctx, PIRK_EINVAL, "step count exceeds the device failure-key range (2^23)");
    const uint64_t n = m->dim;
    const uint64_t unit = is_heat(m) ? m->grid * m->grid : 1;
    const uint64_t units = n / unit;
    if (2 * n >= (1ull << kFailCompBits))
        return fail(ctx, PIRK_EINVAL, "dimension exceeds the device failure-key range");
    const int W = usable_lanes(ctx, units);
    std::vector<uint64_t> slot_steps;
    std::vector<double> slot_times;
    record_schedule(p->t0, p->t1, p->h, p->tube_stride, plan, slot_steps, slot_times);
    const uint64_t S = slot_steps.size();
    if (tube && tube->max_slots < S)
        return fail(ctx, PIRK_EINVAL, "tube: max_slots " + std::to_string(tube->max_slots) +
                                          " < record slots " + std::to_string(S));
    double p0 = 0.0, p1 = 0.0;
    if (m->input_dim > 0) {
        if (method == PIRK_METHOD_MM) {
            p0 = p->input_lower[0];
            p1 = p->input_upper[0];
        } else {  // interval.cpp:25-37 center / half-width
            p0 = 0.5 * (p->input_upper[0] + p->input_lower[0]);
            p1 = 0.5 * (p->input_upper[0] - p->input_lower[0]);
        }
    }
    const ChainModel cm = chain_model(m, method, p0, p1);
    const HeatModel hm = heat_model(m, method);
    const bool cache = state_cache_on();
    std::unique_ptr<ShardState[]> sh(new ShardState[static_cast<size_t>(W)]);
    uint64_t dev_bytes = 0;
    for (int r = 0; r < W; ++r) {
        ShardState& z = sh[static_cast<size_t>(r)];
        z.L = lane_ref(ctx, r);
        z.b = units * static_cast<uint64_t>(r) / static_cast<uint64_t>(W);
        z.e = units * static_cast<uint64_t>(r + 1) / static_cast<uint64_t>(W);
        z.wb = z.b >= 4 ? z.b - 4 : 0;
        z.we = std::min(z.e + 4, units);
        const size_t wn = (z.we - z.wb) * unit;
        CK(ctx, cudaSetDevice(z.L.device));
        for (DevBuf<double>* d : {&z.a0, &z.a1, &z.b0, &z.b1})
            CK(ctx, cache ? d->alloc_state(ctx, *z.L.cache, wn) : d->alloc(ctx, wn));
        dev_bytes += 4 * wn * sizeof(double);
        CK(ctx, z.fail.alloc(ctx, 2));
        CK(ctx, z.slot_flag.alloc(ctx, S));
        CK(ctx, z.slot_val.alloc(ctx, S));
        CK(ctx, z.box_flag.alloc(ctx, 1));
        for (cudaEvent_t* ev : {&z.bnd, &z.sent[0], &z.sent[1]})
            CK(ctx, cudaEventCreateWithFlags(ev, cudaEventDisableTiming));
        CK(ctx, cudaMemsetAsync(z.fail.p, 0xff, 2 * sizeof(unsigned long long), z.L.s));
        CK(ctx, cudaMemsetAsync(z.slot_flag.p, 0xff, S * sizeof(unsigned long long), z.L.s));
        CK(ctx, cudaMemsetAsync(z.box_flag.p, 0xff, sizeof(unsigned long long), z.L.s));
        CK(ctx, cudaMemcpyAsync(z.a0.p, p->init_lower + z.wb * unit, wn * sizeof(double), cudaMemcpyHostToDevice, z.L.s));
        CK(ctx, cudaMemcpyAsync(z.a1.p, p->init_upper + z.wb * unit, wn * sizeof(double), cudaMemcpyHostToDevice, z.L.s));
        const size_t own = (z.b - z.wb) * unit;
        CK(ctx, launch_box_check(z.a0.p + own, z.a1.p + own, (z.e - z.b) * unit, z.box_flag.p, z.L.s));
        ctx->launches++;
        if (method == PIRK_METHOD_GB) {
            CK(ctx, launch_center_radius(z.a0.p, z.a1.p, wn, z.L.s));
            ctx->launches++;
        }
    }
    const double setup_s = since(t_setup);
    const auto t_int = Clock::now();
    const bool ex = exact_mode(ctx);
    // Halo transfer: the boundary launch itself stores its units into the
    // neighbour's halo over NVLink peer memory (WindowArgs::mir0/1) -- one
    // kernel computes and sends; PIRK_LANE_HALO=copy (or lanes without peer
    // access) sends them with cudaMemcpyPeerAsync on the copy stream instead.
    static const bool halo_copy_env = [] {
        const char* v = std::getenv("PIRK_LANE_HALO");
        return v && std::strcmp(v, "copy") == 0;
    }();
    const bool fused = ctx->peer_stores && !halo_copy_env;
    // Fused halos, by default as ONE launch per lane and step over its owned
    // units whose first / last 4 units also go to the neighbours (a windowed
    // launch has a fixed cost -- the 4-unit cone on both sides and the CTA
    // set-up over every tile -- so two thin boundary launches per step cost
    // more than the overlap they buy: tools/peer_probe.py, heat3d g=1600 over
    // 8 lanes 4.94 vs 5.69 ms per step).  PIRK_LANE_SCHEDULE=split keeps the
    // boundary-first launches.
    static const bool split_env = [] {
        const char* v = std::getenv("PIRK_LANE_SCHEDULE");
        return v && std::strcmp(v, "split") == 0;
    }();
    const bool slab = fused && !split_env;
    auto launch = [&](ShardState& z, const StepConsts& sc, uint64_t k, uint64_t ob, uint64_t oe,
                      ShardState* mlo = nullptr, ShardState* mhi = nullptr) -> cudaError_t {
        if (ob >= oe) return cudaSuccess;
        const size_t off = (ob - z.wb) * unit;
        WindowArgs w{z.in0(), z.in1(), z.out0() + off, z.out1() + off, z.wb, z.we, ob, oe};
        // mirror targets: unit ob at the same place of the neighbour's output
        // window (for the high neighbour that place lies before its window;
        // only units >= its window start are stored)
        if (mlo) {
            const long long moff = (static_cast<long long>(ob) - static_cast<long long>(mlo->wb)) * unit;
            w.mir0 = mlo->out0() + moff;
            w.mir1 = mlo->out1() + moff;
            w.mir_lo_end = z.b + 4;
        }
        if (mhi) {
            const long long moff = (static_cast<long long>(ob) - static_cast<long long>(mhi->wb)) * unit;
            w.mirh0 = mhi->out0() + moff;
            w.mirh1 = mhi->out1() + moff;
            w.mir_hi_begin = z.e - 4;
        }
        ctx->launches++;
        if (is_chain(m))
            return ex ? launch_chain_step<true>(cm, w, sc, k, z.fail.p, z.L.s)
                      : launch_chain_step<false>(cm, w, sc, k, z.fail.p, z.L.s);
        return ex ? launch_heat_step<true>(hm, w, sc, k, z.fail.p, z.L.s)
                  : launch_heat_step<false>(hm, w, sc, k, z.fail.p, z.L.s);
    };
    const size_t halo_bytes = 4 * unit * sizeof(double);
    SlotStreamer rec;
    CK(ctx, rec.init(ctx, n, W));
    uint64_t done = 0;
    for (uint64_t s = 0; s < S; ++s) {
        for (; done < slot_steps[s]; ++done) {
            const uint64_t k = done;
            const StepConsts sc = host_step(p->t0, p->t1, p->h, k, plan.total);
            for (int r = 0; r < W; ++r) {
                ShardState& z = sh[static_cast<size_t>(r)];
                const bool left = r > 0, right = r + 1 < W;
                CK(ctx, cudaSetDevice(z.L.device));
                if (k > 0) {  // this step's inputs include the halos the neighbours sent last step
                    if (left) CK(ctx, cudaStreamWaitEvent(z.L.s, sh[static_cast<size_t>(r - 1)].sent[(k - 1) & 1], 0));
                    if (right) CK(ctx, cudaStreamWaitEvent(z.L.s, sh[static_cast<size_t>(r + 1)].sent[(k - 1) & 1], 0));
                }
                // 1. boundary units, the ones the neighbours read next step
                //    (fused: written into the neighbours' halos by the same launch)
                ShardState* yl = left ? &sh[static_cast<size_t>(r - 1)] : nullptr;
                ShardState* yr = right ? &sh[static_cast<size_t>(r + 1)] : nullptr;
                if (slab) {  // one launch: owned units, edges also into the neighbours' halos
                    CK(ctx, launch(z, sc, k, z.b, z.e, yl, yr));
                    if (left || right) CK(ctx, cudaEventRecord(z.sent[k & 1], z.L.s));
                    continue;
                }
                if (left) CK(ctx, launch(z, sc, k, z.b, z.b + 4, fused ? yl : nullptr));
                if (right) CK(ctx, launch(z, sc, k, z.e - 4, z.e, nullptr, fused ? yr : nullptr));
                if (fused && (left || right)) CK(ctx, cudaEventRecord(z.sent[k & 1], z.L.s));
                // 2. else their peer copies, on the copy stream
                if (!fused && (left || right)) {
                    CK(ctx, cudaEventRecord(z.bnd, z.L.s));
                    CK(ctx, cudaStreamWaitEvent(z.L.xs, z.bnd, 0));
                    if (left) {
                        ShardState& y = sh[static_cast<size_t>(r - 1)];
                        const size_t so = (z.b - z.wb) * unit, dof = (z.b - y.wb) * unit;
                        CK(ctx, cudaMemcpyPeerAsync(y.out0() + dof, y.L.device, z.out0() + so, z.L.device, halo_bytes, z.L.xs));
                        CK(ctx, cudaMemcpyPeerAsync(y.out1() + dof, y.L.device, z.out1() + so, z.L.device, halo_bytes, z.L.xs));
                    }
                    if (right) {
                        ShardState& y = sh[static_cast<size_t>(r + 1)];
                        const size_t so = (z.e - 4 - z.wb) * unit, dof = (z.e - 4 - y.wb) * unit;
                        CK(ctx, cudaMemcpyPeerAsync(y.out0() + dof, y.L.device, z.out0() + so, z.L.device, halo_bytes, z.L.xs));
                        CK(ctx, cudaMemcpyPeerAsync(y.out1() + dof, y.L.device, z.out1() + so, z.L.device, halo_bytes, z.L.xs));
                    }
                    CK(ctx, cudaEventRecord(z.sent[k & 1], z.L.xs));
                }
                // 3. the interior, overlapping the copies
                CK(ctx, launch(z, sc, k, left ? z.b + 4 : z.b, right ? z.e - 4 : z.e));
            }
            for (int r = 0; r < W; ++r) sh[static_cast<size_t>(r)].cur ^= 1;
        }
        CK(ctx, rec.deliver());  // slot s-1 to the callback while these steps run
        for (int r = 0; r < W; ++r) {  // record slot s on every lane's owned units
            ShardState& z = sh[static_cast<size_t>(r)];
            CK(ctx, cudaSetDevice(z.L.device));
            const size_t own = (z.b - z.wb) * unit, cnt = (z.e - z.b) * unit;
            const double* lo = z.in0() + own;
            const double* hi = z.in1() + own;
            if (method == PIRK_METHOD_MM) {
                CK(ctx, launch_order_check(lo, hi, cnt, z.slot_flag.p + s, z.L.s));
            } else {  // the next step's output buffers (owned part) take the clamped box
                CK(ctx, launch_gb_box(lo, hi, z.out0() + own, z.out1() + own, cnt, z.slot_flag.p + s, z.L.s));
                CK(ctx, launch_gb_negval(hi, z.slot_flag.p + s, z.slot_val.p + s, z.L.s));
                ctx->launches++;
                lo = z.out0() + own;
                hi = z.out1() + own;
            }
            ctx->launches++;
            if (tube && tube->lower)
                CK(ctx, cudaMemcpyAsync(tube->lower + s * n + z.b * unit, lo, cnt * sizeof(double), cudaMemcpyDeviceToHost, z.L.s));
            if (tube && tube->upper)
                CK(ctx, cudaMemcpyAsync(tube->upper + s * n + z.b * unit, hi, cnt * sizeof(double), cudaMemcpyDeviceToHost, z.L.s));
            if (rec.on()) {
                CK(ctx, cudaMemcpyAsync(rec.buf + z.b * unit, lo, cnt * sizeof(double), cudaMemcpyDeviceToHost, z.L.s));
                CK(ctx, cudaMemcpyAsync(rec.buf + n + z.b * unit, hi, cnt * sizeof(double), cudaMemcpyDeviceToHost, z.L.s));
                CK(ctx, rec.mark(r, z.L.s));
            }
        }
        if (rec.on()) rec.set_pending(s, slot_steps[s], slot_times[s]);
    }
    CK(ctx, cudaSetDevice(ctx->device));
    CK(ctx, rec.deliver());
    unsigned long long f0 = kNoFail, f1 = kNoFail, box = kNoFail;
    std::vector<unsigned long long> flags(S, kNoFail), lf(S);
    std::vector<double> vals(S, 0.0), lv(S);
    for (int r = 0; r < W; ++r) {
        ShardState& z = sh[static_cast<size_t>(r)];
        CK(ctx, cudaSetDevice(z.L.device));
        unsigned long long hf[3];
        CK(ctx, cudaMemcpyAsync(hf, z.fail.p, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, z.L.s));
        CK(ctx, cudaMemcpyAsync(hf + 2, z.box_flag.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost, z.L.s));
        CK(ctx, cudaMemcpyAsync(lf.data(), z.slot_flag.p, S * sizeof(unsigned long long), cudaMemcpyDeviceToHost, z.L.s));
        CK(ctx, cudaMemcpyAsync(lv.data(), z.slot_val.p, S * sizeof(double), cudaMemcpyDeviceToHost, z.L.s));
        CK(ctx, cudaStreamSynchronize(z.L.s));
        CK(ctx, cudaStreamSynchronize(z.L.xs));
        // failure keys carry global components; slot / box flags are lane-local
        f0 = std::min(f0, hf[0]);
        f1 = std::min(f1, hf[1]);
        const unsigned long long base = z.b * unit;
        if (hf[2] != kNoFail) box = std::min(box, hf[2] + base);
        for (uint64_t s = 0; s < S; ++s)
            if (lf[s] != kNoFail && lf[s] + base < flags[s]) {
                flags[s] = lf[s] + base;
                vals[s] = lv[s];
            }
    }
    CK(ctx, cudaSetDevice(ctx->device));
    const double integ_s = since(t_int);
    if (box != kNoFail) {  // IntervalVector validation (interval.cpp:14-22) comes first
        const bool nonfinite = !std::isfinite(p->init_lower[box]) || !std::isfinite(p->init_upper[box]);
        return fail(ctx, PIRK_EINVAL, std::string(nonfinite ? "interval: non-finite bound at component "
                                                            : "interval: lower > upper at component ") +
                                          std::to_string(box));
    }
    if (tube) {
        tube->n_slots = S;
        if (tube->times)
            for (uint64_t s = 0; s < S; ++s) tube->times[s] = slot_times[s];
    }
    return large_errors(ctx, method, p, plan.total, slot_steps, slot_times, f0, f1, flags, vals, n, dev_bytes,
                        setup_s, integ_s, ctx->launches - launches0, W, rep);
}

#include "user_models.cuh"

// Small-model MM / GB: one device thread per integration.
pirk_status run_small(pirk_ctx* ctx, const pirk_model* m, int method, const pirk_problem* p,
                      pirk_tube* tube, pirk_report* rep) {
    const auto t_setup = Clock::now();
    const uint64_t launches0 = ctx->launches;
    Plan plan;
    plan_steps(p->t0, p->t1, p->h, plan);
    std::vector<uint64_t> slot_steps;
    std::vector<double> slot_times;
    record_schedule(p->t0, p->t1, p->h, p->tube_stride, plan, slot_steps, slot_times);
    const uint64_t S = slot_steps.size();
    if (tube && tube->max_slots < S)
        return fail(ctx, PIRK_EINVAL, "tube: max_slots too small");
    const uint64_t n = m->dim, ni = m->input_dim;
    const SmallModel sm = small_model(m);
    const bool ex = exact_mode(ctx);
    UserBuild* ub = nullptr;  // user-defined evaluators (NVRTC kernels)
    if (is_user(m)) {
        const pirk_status us = user_kernels(ctx, m, &ub);
        if (us != PIRK_OK) return us;
    }
    std::vector<double> host_rec0, host_rec1;
    unsigned long long f0 = kNoFail, f1 = kNoFail;
    double setup_s = 0.0;
    const auto t_int = Clock::now();
    if (method == PIRK_METHOD_MM) {
        // x0 = [lower | upper], p = [p_lo | p_hi] (reach.cpp:150-161)
        std::vector<double> x0(2 * n), pp(2 * ni + 1, 0.0);
        for (uint64_t i = 0; i < n; ++i) { x0[i] = p->init_lower[i]; x0[n + i] = p->init_upper[i]; }
        for (uint64_t j = 0; j < ni; ++j) { pp[j] = p->input_lower[j]; pp[ni + j] = p->input_upper[j]; }
        DevBuf<double> dx, dp, drec;
        DevBuf<unsigned long long> dfail;
        CK(ctx, dx.alloc(ctx, 2 * n));
        CK(ctx, dp.alloc(ctx, pp.size()));
        CK(ctx, drec.alloc(ctx, S * 2 * n));
        CK(ctx, dfail.alloc(ctx, 1));
        CK(ctx, cudaMemcpyAsync(dx.p, x0.data(), 2 * n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        CK(ctx, cudaMemcpyAsync(dp.p, pp.data(), pp.size() * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        CK(ctx, cudaMemsetAsync(dfail.p, 0xff, sizeof(unsigned long long), ctx->stream));
        setup_s = since(t_setup);
        CK(ctx, ub ? user_launch_small(ub, 2, dx.p, dp.p, p->t0, p->t1, p->h, plan.total, p->tube_stride, drec.p, dfail.p, ctx->stream)
              : ex ? launch_small_integrate<true>(sm, 2, dx.p, dp.p, p->t0, p->t1, p->h, plan.total, p->tube_stride, drec.p, dfail.p, ctx->stream)
                   : launch_small_integrate<false>(sm, 2, dx.p, dp.p, p->t0, p->t1, p->h, plan.total, p->tube_stride, drec.p, dfail.p, ctx->stream));
        ctx->launches++;
        host_rec0.resize(S * 2 * n);
        CK(ctx, cudaMemcpyAsync(host_rec0.data(), drec.p, S * 2 * n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        CK(ctx, cudaMemcpyAsync(&f0, dfail.p, sizeof f0, cudaMemcpyDeviceToHost, ctx->stream));
        CK(ctx, cudaStreamSynchronize(ctx->stream));
    } else {
        // center/radius of the initial and input boxes (interval.cpp:25-37)
        std::vector<double> c0(n), r0(n), pc(ni + 1, 0.0), w(ni + 1, 0.0);
        for (uint64_t i = 0; i < n; ++i) {
            c0[i] = 0.5 * (p->init_upper[i] + p->init_lower[i]);
            r0[i] = 0.5 * (p->init_upper[i] - p->init_lower[i]);
        }
        for (uint64_t j = 0; j < ni; ++j) {
            pc[j] = 0.5 * (p->input_upper[j] + p->input_lower[j]);
            w[j] = 0.5 * (p->input_upper[j] - p->input_lower[j]);
        }
        DevBuf<double> dc, dr, dpc, dw, drec0, drec1;
        DevBuf<unsigned long long> dfail;
        CK(ctx, dc.alloc(ctx, n)); CK(ctx, dr.alloc(ctx, n)); CK(ctx, dpc.alloc(ctx, ni + 1)); CK(ctx, dw.alloc(ctx, ni + 1));
        CK(ctx, drec0.alloc(ctx, S * n)); CK(ctx, drec1.alloc(ctx, S * n)); CK(ctx, dfail.alloc(ctx, 2));
        CK(ctx, cudaMemcpyAsync(dc.p, c0.data(), n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        CK(ctx, cudaMemcpyAsync(dr.p, r0.data(), n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        CK(ctx, cudaMemcpyAsync(dpc.p, pc.data(), (ni + 1) * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        CK(ctx, cudaMemcpyAsync(dw.p, w.data(), (ni + 1) * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        CK(ctx, cudaMemsetAsync(dfail.p, 0xff, 2 * sizeof(unsigned long long), ctx->stream));
        setup_s = since(t_setup);
        for (int which = 0; which < 2; ++which) {
            const double* x0 = which ? dr.p : dc.p;
            const double* pp = which ? dw.p : dpc.p;
            double* rec = which ? drec1.p : drec0.p;
            CK(ctx, ub ? user_launch_small(ub, which, x0, pp, p->t0, p->t1, p->h, plan.total, p->tube_stride, rec, dfail.p + which, ctx->stream)
                  : ex ? launch_small_integrate<true>(sm, which, x0, pp, p->t0, p->t1, p->h, plan.total, p->tube_stride, rec, dfail.p + which, ctx->stream)
                       : launch_small_integrate<false>(sm, which, x0, pp, p->t0, p->t1, p->h, plan.total, p->tube_stride, rec, dfail.p + which, ctx->stream));
            ctx->launches++;
        }
        host_rec0.resize(S * n);
        host_rec1.resize(S * n);
        unsigned long long ff[2];
        CK(ctx, cudaMemcpyAsync(host_rec0.data(), drec0.p, S * n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        CK(ctx, cudaMemcpyAsync(host_rec1.data(), drec1.p, S * n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        CK(ctx, cudaMemcpyAsync(ff, dfail.p, sizeof ff, cudaMemcpyDeviceToHost, ctx->stream));
        CK(ctx, cudaStreamSynchronize(ctx->stream));
        f0 = ff[0];
        f1 = ff[1];
    }
    const double integ_s = since(t_int);
    const auto t_red = Clock::now();
    if (tube) {
        tube->n_slots = S;
        if (tube->times)
            for (uint64_t s = 0; s < S; ++s) tube->times[s] = slot_times[s];
    }
    auto decode = [](unsigned long long key, uint64_t& step, uint64_t& comp) {
        step = key >> kFailCompBits;
        comp = key & ((1ull << kFailCompBits) - 1);
    };
    if (method == PIRK_METHOD_MM) {
        uint64_t fs = 0, fc = 0;
        if (f0 != kNoFail) decode(f0, fs, fc);
        for (uint64_t s = 0; s < S; ++s) {
            if (f0 != kNoFail && fs < slot_steps[s])
                return fail(ctx, PIRK_EINTEGRATION, "mixed-monotonicity embedding integration: " +
                                                        integ_msg(fs, fc, p->t0 + static_cast<double>(fs) * p->h));
            const double* xx = host_rec0.data() + s * 2 * n;
            for (uint64_t i = 0; i < n; ++i)  // reach.cpp:181-186
                if (xx[i] > xx[n + i])
                    return fail(ctx, PIRK_EORDER, "mixed-monotonicity: embedding order violated at step " +
                                                      std::to_string(slot_steps[s]) + ", t = " + fstr(slot_times[s]) +
                                                      ", component " + std::to_string(i));
            if (tube && tube->lower) std::memcpy(tube->lower + s * n, xx, n * sizeof(double));
            if (tube && tube->upper) std::memcpy(tube->upper + s * n, xx + n, n * sizeof(double));
            if (ctx->record_fn) ctx->record_fn(ctx->record_user, s, slot_steps[s], slot_times[s], xx, xx + n, n);
        }
        fill_report(rep, n, 0, plan.total, 7 * 2 * n * sizeof(double), 4 * 2 * n * sizeof(double),
                    ex, setup_s, integ_s, since(t_red), ctx->launches - launches0);
    } else {
        uint64_t fs = 0, fc = 0;
        if (f0 != kNoFail) {
            decode(f0, fs, fc);
            return fail(ctx, PIRK_EINTEGRATION, "growth-bound center integration: " +
                                                    integ_msg(fs, fc, p->t0 + static_cast<double>(fs) * p->h));
        }
        if (f1 != kNoFail) {
            decode(f1, fs, fc);
            return fail(ctx, PIRK_EINTEGRATION, "growth-bound radius integration: " +
                                                    integ_msg(fs, fc, p->t0 + static_cast<double>(fs) * p->h));
        }
        for (uint64_t s = 0; s < S; ++s) {  // reach.cpp:121-134
            double* r = host_rec1.data() + s * n;
            const double* c = host_rec0.data() + s * n;
            for (uint64_t i = 0; i < n; ++i) {
                if (r[i] < 0.0) {
                    if (r[i] < -1e-12)
                        return fail(ctx, PIRK_ENEGRADIUS, "growth-bound: deviation went negative (" + fstr(r[i]) +
                                                              ") at component " + std::to_string(i) +
                                                              "; contraction matrix is invalid");
                    r[i] = 0.0;
                }
                if (tube && tube->lower) tube->lower[s * n + i] = c[i] - r[i];
                if (tube && tube->upper) tube->upper[s * n + i] = c[i] + r[i];
            }
            if (ctx->record_fn) {
                std::vector<double> lo(n), hi(n);
                for (uint64_t i = 0; i < n; ++i) {
                    lo[i] = c[i] - r[i];
                    hi[i] = c[i] + r[i];
                }
                ctx->record_fn(ctx->record_user, s, slot_steps[s], slot_times[s], lo.data(), hi.data(), n);
            }
        }
        fill_report(rep, n, 0, plan.total, 7 * n * sizeof(double), 4 * n * sizeof(double), ex,
                    setup_s, integ_s, since(t_red), ctx->launches - launches0);
    }
    return PIRK_OK;
}

// Monte Carlo (reach.cpp:246-323): samples [s_begin, s_end) split over the
// context's lanes (pirk_create_multi), each lane one launch of the
// one-sample-per-thread kernel on its own device/stream; the per-lane hulls
// (order-preserving keys) are min/max-folded on the host -- exact and
// order-independent, the single-process form of the NCCL MIN/MAX all-reduce.
pirk_status run_mc(pirk_ctx* ctx, const pirk_model* m, const pirk_problem* p, uint64_t seed,
                   uint64_t s_begin, uint64_t s_end, uint64_t m_total, pirk_tube* tube,
                   bool fold_into, pirk_report* rep, const double* box_lo, const double* box_hi,
                   double* fraction) {
    const auto t_setup = Clock::now();
    const uint64_t launches0 = ctx->launches;
    UserBuild* ub = nullptr;
    pirk_model um;  // a catalog model beyond the compiled MC kernels: its field as NVRTC source
    if (!is_user(m) && !small_ok(m) && catalog_mc_program(ctx, m, um)) m = &um;
    if (is_user(m)) {
        if (m->dim > kUserMcMax)
            return fail(ctx, PIRK_EUNSUPPORTED, "monte_carlo: device kernel supports user models with n <= " +
                                                    std::to_string(kUserMcMax) + " (got " + std::to_string(m->dim) + ")");
        const pirk_status us = user_kernels(ctx, m, &ub);
        if (us != PIRK_OK) return us;
    } else if (!small_ok(m)) {
        return fail(ctx, PIRK_EUNSUPPORTED, "monte_carlo: device kernel supports n <= " +
                                                std::to_string(kSmallMax) + " (got " + std::to_string(m->dim) + ")");
    }
    Plan plan;
    plan_steps(p->t0, p->t1, p->h, plan);
    const bool coverage = fraction != nullptr;
    std::vector<uint64_t> slot_steps;
    std::vector<double> slot_times;
    record_schedule(p->t0, p->t1, p->h, coverage ? 0 : p->tube_stride, plan, slot_steps, slot_times);
    const uint64_t S = slot_steps.size();
    if (tube && tube->max_slots < S) return fail(ctx, PIRK_EINVAL, "tube: max_slots too small");
    if (s_end - s_begin >= (1ull << 34) || plan.total >= (1ull << 20))
        return fail(ctx, PIRK_EINVAL, "monte_carlo: sample count or step count exceeds the device key range");
    const uint64_t n = m->dim, ni = m->input_dim;
    const SmallModel sm = small_model(m);
    const size_t nb = 4 * n + 2 * (ni + 1);
    std::vector<double> hb(nb, 0.0);
    for (uint64_t i = 0; i < n; ++i) {
        hb[i] = p->init_lower[i];
        hb[n + i] = p->init_upper[i];
        if (coverage) {
            hb[2 * n + i] = box_lo[i];
            hb[3 * n + i] = box_hi[i];
        }
    }
    for (uint64_t j = 0; j < ni; ++j) {
        hb[4 * n + j] = p->input_lower[j];
        hb[4 * n + ni + 1 + j] = p->input_upper[j];
    }
    const uint64_t count = s_end - s_begin;
    const int W = static_cast<int>(std::min<uint64_t>(static_cast<uint64_t>(ctx->lanes()), count));
    struct McLane {
        LaneRef L{};
        uint64_t sb = 0, se = 0;
        DevBuf<double> dbox;  // lo, hi, box_lo, box_hi, plo, phi
        DevBuf<unsigned long long> dhull, dflags;
        std::vector<unsigned long long> hull;
        unsigned long long fl[2] = {kNoFail, 0};
    };
    std::unique_ptr<McLane[]> ln(new McLane[static_cast<size_t>(W)]);
    for (int r = 0; r < W; ++r) {
        McLane& z = ln[static_cast<size_t>(r)];
        z.L = lane_ref(ctx, r);
        z.sb = s_begin + count * static_cast<uint64_t>(r) / static_cast<uint64_t>(W);
        z.se = s_begin + count * static_cast<uint64_t>(r + 1) / static_cast<uint64_t>(W);
        CK(ctx, cudaSetDevice(z.L.device));
        CK(ctx, z.dbox.alloc(ctx, nb));
        CK(ctx, z.dhull.alloc(ctx, S * 2 * n));
        CK(ctx, z.dflags.alloc(ctx, 2));
        CK(ctx, cudaMemcpyAsync(z.dbox.p, hb.data(), nb * sizeof(double), cudaMemcpyHostToDevice, z.L.s));
        for (uint64_t s = 0; s < S; ++s) {  // hull init +inf / -inf as ordered keys (reach.cpp:218-221)
            CK(ctx, cudaMemsetAsync(z.dhull.p + s * 2 * n, 0xff, n * sizeof(unsigned long long), z.L.s));
            CK(ctx, cudaMemsetAsync(z.dhull.p + s * 2 * n + n, 0x00, n * sizeof(unsigned long long), z.L.s));
        }
        CK(ctx, cudaMemsetAsync(z.dflags.p, 0xff, sizeof(unsigned long long), z.L.s));
        CK(ctx, cudaMemsetAsync(z.dflags.p + 1, 0x00, sizeof(unsigned long long), z.L.s));
    }
    const double setup_s = since(t_setup);
    const auto t_int = Clock::now();
    for (int r = 0; r < W; ++r) {
        McLane& z = ln[static_cast<size_t>(r)];
        McArgs a{};
        a.lo = z.dbox.p;
        a.hi = z.dbox.p + n;
        a.plo = z.dbox.p + 4 * n;
        a.phi = z.dbox.p + 4 * n + ni + 1;
        a.seed = seed;
        a.s_begin = z.sb;
        a.s_end = z.se;
        a.t0 = p->t0;
        a.t1 = p->t1;
        a.h = p->h;
        a.total = plan.total;
        a.stride = coverage ? 0 : p->tube_stride;
        a.slots = S;
        a.hull = z.dhull.p;
        a.fail = z.dflags.p;
        if (coverage) {
            a.box_lo = z.dbox.p + 2 * n;
            a.box_hi = z.dbox.p + 3 * n;
            a.outside = z.dflags.p + 1;
        }
        CK(ctx, cudaSetDevice(z.L.device));
        CK(ctx, ub ? user_launch_mc(ub, a, z.L.s)
                   : exact_mode(ctx) ? launch_monte_carlo<true>(sm, a, z.L.s)
                                     : launch_monte_carlo<false>(sm, a, z.L.s));
        ctx->launches++;
        z.hull.resize(S * 2 * n);
        CK(ctx, cudaMemcpyAsync(z.hull.data(), z.dhull.p, z.hull.size() * sizeof(unsigned long long),
                                cudaMemcpyDeviceToHost, z.L.s));
        CK(ctx, cudaMemcpyAsync(z.fl, z.dflags.p, sizeof z.fl, cudaMemcpyDeviceToHost, z.L.s));
    }
    for (int r = 0; r < W; ++r) {
        CK(ctx, cudaSetDevice(ln[static_cast<size_t>(r)].L.device));
        CK(ctx, cudaStreamSynchronize(ln[static_cast<size_t>(r)].L.s));
    }
    CK(ctx, cudaSetDevice(ctx->device));
    const double integ_s = since(t_int);
    const auto t_red = Clock::now();
    // the lowest failing sample over all lanes (its lane's key is lane-relative)
    uint64_t fail_sample = ~0ull, fail_step = 0, fail_comp = 0;
    unsigned long long outside = 0;
    for (int r = 0; r < W; ++r) {
        const McLane& z = ln[static_cast<size_t>(r)];
        if (z.fl[0] != kNoFail) {
            const uint64_t smp = z.sb + (z.fl[0] >> 30);
            if (smp < fail_sample) {
                fail_sample = smp;
                fail_step = (z.fl[0] >> 10) & 0xfffff;
                fail_comp = z.fl[0] & 0x3ff;
            }
        }
        outside += z.fl[1];
    }
    if (fail_sample != ~0ull)
        return fail(ctx, PIRK_EINTEGRATION, "monte-carlo sample " + std::to_string(fail_sample) + " integration: " +
                                                integ_msg(fail_step, fail_comp, p->t0 + static_cast<double>(fail_step) * p->h));
    if (coverage) {
        *fraction = static_cast<double>(outside) / static_cast<double>(count);
        return PIRK_OK;
    }
    std::vector<double> slo, shi;  // the record callback's copy of a slot
    if (tube) {
        tube->n_slots = S;
        for (uint64_t s = 0; s < S; ++s) {
            if (tube->times) tube->times[s] = slot_times[s];
            if (ctx->record_fn && !fold_into) {
                slo.assign(n, 0.0);
                shi.assign(n, 0.0);
            }
            for (uint64_t i = 0; i < n; ++i) {
                unsigned long long klo = ln[0].hull[s * 2 * n + i], khi = ln[0].hull[s * 2 * n + n + i];
                for (int r = 1; r < W; ++r) {  // HullAccumulator::merge (reach.cpp:232-241) on keys
                    klo = std::min(klo, ln[static_cast<size_t>(r)].hull[s * 2 * n + i]);
                    khi = std::max(khi, ln[static_cast<size_t>(r)].hull[s * 2 * n + n + i]);
                }
                const double lo = ord_val(klo);
                const double hi = ord_val(khi);
                if (fold_into) {
                    if (tube->lower && lo < tube->lower[s * n + i]) tube->lower[s * n + i] = lo;
                    if (tube->upper && hi > tube->upper[s * n + i]) tube->upper[s * n + i] = hi;
                } else {
                    if (tube->lower) tube->lower[s * n + i] = lo;
                    if (tube->upper) tube->upper[s * n + i] = hi;
                }
                if (!slo.empty()) {
                    slo[i] = lo;
                    shi[i] = hi;
                }
            }
            if (!slo.empty()) ctx->record_fn(ctx->record_user, s, slot_steps[s], slot_times[s], slo.data(), shi.data(), n);
        }
    }
    // reach.cpp:273-275 with `outer` = lanes
    const uint64_t peak = static_cast<uint64_t>(W) * (7 * n * sizeof(double) + 2 * S * n * sizeof(double)) +
                          2 * S * n * sizeof(double);
    fill_report(rep, n, m_total, plan.total, peak, static_cast<uint64_t>(W) * (nb * sizeof(double) + S * 2 * n * 8),
                exact_mode(ctx), setup_s, integ_s, since(t_red), ctx->launches - launches0);
    if (rep) rep->workers = W;
    return PIRK_OK;
}

}  // namespace

// ================================================================== C ABI

extern "C" {

int32_t pirk_abi_version(void) { return PIRK_ABI_VERSION; }

pirk_status pirk_create(int device, pirk_ctx** out) { return pirk_create_multi(1, &device, out); }

pirk_status pirk_create_multi(int n_lanes, const int* devices, pirk_ctx** out) {
    if (!out || n_lanes < 1 || !devices) return PIRK_EINVAL;
    *out = nullptr;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) return PIRK_ECUDA;
    for (int r = 0; r < n_lanes; ++r)
        if (devices[r] < 0 || devices[r] >= count) return PIRK_EINVAL;
    pirk_ctx* ctx = new (std::nothrow) pirk_ctx;
    if (!ctx) return PIRK_ENOMEM;
    const int device = devices[0];
    ctx->device = device;
    if (cudaSetDevice(device) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->own_xstream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaMalloc(reinterpret_cast<void**>(&ctx->d_flags), 16 * sizeof(unsigned long long)) != cudaSuccess ||
        cudaMallocHost(reinterpret_cast<void**>(&ctx->h_flags), 16 * sizeof(unsigned long long)) != cudaSuccess) {
        pirk_destroy(ctx);
        return PIRK_ECUDA;
    }
    ctx->stream = ctx->own_stream;
    for (int r = 1; r < n_lanes; ++r) {
        PirkLane l;
        l.device = devices[r];
        ctx->peers.push_back(l);
        PirkLane& lr = ctx->peers.back();
        if (cudaSetDevice(lr.device) != cudaSuccess ||
            cudaStreamCreateWithFlags(&lr.stream, cudaStreamNonBlocking) != cudaSuccess ||
            cudaStreamCreateWithFlags(&lr.xstream, cudaStreamNonBlocking) != cudaSuccess) {
            pirk_destroy(ctx);
            return PIRK_ECUDA;
        }
    }
    // halos move between adjacent lanes: direct NVLink peer access where the
    // devices differ (cudaMemcpyPeerAsync falls back to staging otherwise)
    for (int r = 0; r + 1 < n_lanes; ++r) {
        const int a = devices[r], b = devices[r + 1];
        if (a == b) continue;
        for (int dir = 0; dir < 2; ++dir) {
            const int from = dir ? b : a, to = dir ? a : b;
            int ok = 0;
            if (cudaDeviceCanAccessPeer(&ok, from, to) == cudaSuccess && ok) {
                cudaSetDevice(from);
                const cudaError_t pe = cudaDeviceEnablePeerAccess(to, 0);
                if (pe == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                else if (pe != cudaSuccess) {
                    cudaGetLastError();
                    ctx->peer_stores = false;
                }
            } else {
                ctx->peer_stores = false;  // halos then move by copy engine (staged by the driver)
            }
        }
    }
    cudaSetDevice(device);
    *out = ctx;
    return PIRK_OK;
}

int32_t pirk_lane_count(const pirk_ctx* ctx) { return ctx ? ctx->lanes() : 0; }

int32_t pirk_device_count(void) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return count;
}

int32_t pirk_lane_device(const pirk_ctx* ctx, int32_t lane) {
    if (!ctx || lane < 0 || lane >= ctx->lanes()) return -1;
    return lane == 0 ? ctx->device : ctx->peers[static_cast<size_t>(lane - 1)].device;
}

pirk_status pirk_set_record_callback(pirk_ctx* ctx, pirk_record_fn fn, void* user) {
    if (!ctx) return PIRK_EINVAL;
    LOCK(ctx);
    ctx->record_fn = fn;
    ctx->record_user = user;
    return PIRK_OK;
}

pirk_status pirk_release_cache(pirk_ctx* ctx) {
    if (!ctx) return PIRK_EINVAL;
    LOCK(ctx);
    ctx->flush_all();
    return PIRK_OK;
}

void pirk_destroy(pirk_ctx* ctx) {
    if (!ctx) return;
    {
        LOCK(ctx);
        ctx->flush_all();
        for (PirkLane& l : ctx->peers) {
            cudaSetDevice(l.device);
            if (l.stream) cudaStreamDestroy(l.stream);
            if (l.xstream) cudaStreamDestroy(l.xstream);
        }
        cudaSetDevice(ctx->device);
        if (ctx->d_flags) cudaFree(ctx->d_flags);
        if (ctx->h_flags) cudaFreeHost(ctx->h_flags);
        if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
        if (ctx->own_xstream) cudaStreamDestroy(ctx->own_xstream);
    }
    delete ctx;
}

const char* pirk_last_error(const pirk_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

pirk_status pirk_set_mode(pirk_ctx* ctx, int32_t mode) {
    if (!ctx || (mode != PIRK_MODE_EXACT && mode != PIRK_MODE_FAST)) return PIRK_EINVAL;
    LOCK(ctx);
    ctx->mode = mode;
    return PIRK_OK;
}

pirk_status pirk_set_stream(pirk_ctx* ctx, void* stream) {
    if (!ctx) return PIRK_EINVAL;
    LOCK(ctx);
    ctx->stream = static_cast<cudaStream_t>(stream);  // NULL = the CUDA default stream
    return PIRK_OK;
}

void* pirk_get_stream(pirk_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

uint64_t pirk_launch_count(const pirk_ctx* ctx) { return ctx ? ctx->launches : 0; }

pirk_status pirk_plan_steps(double t0, double t1, double h, uint64_t* full_steps,
                            int32_t* has_remainder) {
    Plan p;
    if (!plan_steps(t0, t1, h, p)) return PIRK_EINVAL;
    if (full_steps) *full_steps = p.full;
    if (has_remainder) *has_remainder = p.rem ? 1 : 0;
    return PIRK_OK;
}

uint64_t pirk_record_schedule(double t0, double t1, double h, uint64_t stride, uint64_t* steps_out,
                              double* times_out) {
    Plan p;
    if (!plan_steps(t0, t1, h, p)) return 0;
    std::vector<uint64_t> steps;
    std::vector<double> times;
    record_schedule(t0, t1, h, stride, p, steps, times);
    for (size_t i = 0; i < steps.size(); ++i) {
        if (steps_out) steps_out[i] = steps[i];
        if (times_out) times_out[i] = times[i];
    }
    return steps.size();
}

pirk_status pirk_sample_count(uint64_t n, double epsilon, double delta, uint64_t* out) {
    // reach.cpp:55-63
    if (n == 0 || !(epsilon > 0.0) || !(epsilon < 1.0) || !(delta > 0.0) || !(delta < 1.0))
        return PIRK_EINVAL;
    const double nn = 2.0 * static_cast<double>(n);
    *out = static_cast<uint64_t>(std::ceil(nn / epsilon * std::log(nn / delta)));
    return PIRK_OK;
}

int32_t pirk_supports(const pirk_model* m, int32_t method) {
    if (!m) return 0;
    if (m->kind == PIRK_USER) {
        if (!m->program) return 0;
        const uint32_t f = m->program->flags;
        if (method == PIRK_METHOD_MM) return (f & PIRK_HAS_DECOMPOSITION) ? 1 : 0;
        if (method == PIRK_METHOD_GB) return (f & PIRK_HAS_GROWTH) ? 1 : 0;
        return ((f & PIRK_HAS_RHS) && m->dim <= kUserMcMax) ? 1 : 0;
    }
    if (method == 2 && !small_ok(m)) return catalog_mc_source_ok(m) ? 1 : 0;
    if (method == PIRK_METHOD_MM) {
        if (m->decomp == PIRK_DECOMP_NONE) return 0;
        if (is_chain(m) || is_heat(m)) return m->decomp == PIRK_DECOMP_NATIVE;
        if (!small_ok(m)) return 0;
        if (m->decomp == PIRK_DECOMP_JACOBIAN)
            return m->kind == PIRK_LAUB_LOOMIS || m->kind == PIRK_ARCH_QUAD || m->kind == PIRK_VDP;
        return m->kind != PIRK_LAUB_LOOMIS && m->kind != PIRK_ARCH_QUAD && m->kind != PIRK_VDP;
    }
    if (method == PIRK_METHOD_GB) {
        if (!has_growth(m)) return 0;
        return is_chain(m) || is_heat(m) || small_ok(m);
    }
    return small_ok(m) ? 1 : 0;  // 2 = Monte Carlo
}

static pirk_status reach_mm_gb(pirk_ctx* ctx, const pirk_model* m, const pirk_problem* p,
                               pirk_tube* tube, pirk_report* rep, int method) {
    if (!ctx) return PIRK_EINVAL;
    LOCK(ctx);
    ctx->err.clear();
    if (cudaSetDevice(ctx->device) != cudaSuccess) return fail(ctx, PIRK_ECUDA, "cudaSetDevice failed");
    pirk_status st = PIRK_OK;
    const bool large = m && (is_chain(m) || is_heat(m));
    if (!check_problem(ctx, m, p, !large, st)) return st;
    if (method == PIRK_METHOD_MM) {
        if (!has_decomposition(m))
            return fail(ctx, PIRK_EINVAL, "mixed_monotonicity: model has no decomposition function");
        if (!pirk_supports(m, PIRK_METHOD_MM))
            return fail(ctx, PIRK_EUNSUPPORTED, "mixed_monotonicity: no device kernel for this model/decomposition");
    } else {
        if (!has_growth(m)) return fail(ctx, PIRK_EINVAL, "growth_bound: model has no deviation dynamics");
        if (is_user(m) && !(m->program->flags & PIRK_INPUT_AFFINE))  // reach.cpp:70-71
            return fail(ctx, PIRK_EINVAL, "growth_bound: model is not input-affine");
        if (!pirk_supports(m, PIRK_METHOD_GB))
            return fail(ctx, PIRK_EUNSUPPORTED, "growth_bound: no device kernel for this model");
    }
    try {
        if (is_user(m) && m->dim > kUserSmallMax) return run_user_large(ctx, m, method, p, tube, rep);
        if (!large) return run_small(ctx, m, method, p, tube, rep);
        if (ctx->lanes() > 1 && usable_lanes(ctx, is_heat(m) ? m->grid : m->dim) > 1)
            return run_large_multi(ctx, m, method, p, tube, rep);
        return run_large(ctx, m, method, p, tube, rep);
    } catch (const std::bad_alloc&) {
        return fail(ctx, PIRK_ENOMEM, "host allocation failed");
    }
}

pirk_status pirk_mixed_monotonicity(pirk_ctx* ctx, const pirk_model* model,
                                    const pirk_problem* problem, pirk_tube* tube,
                                    pirk_report* report) {
    return reach_mm_gb(ctx, model, problem, tube, report, PIRK_METHOD_MM);
}

pirk_status pirk_growth_bound(pirk_ctx* ctx, const pirk_model* model, const pirk_problem* problem,
                              pirk_tube* tube, pirk_report* report) {
    return reach_mm_gb(ctx, model, problem, tube, report, PIRK_METHOD_GB);
}

pirk_status pirk_monte_carlo(pirk_ctx* ctx, const pirk_model* m, const pirk_problem* p,
                             const pirk_mc_spec* spec, pirk_tube* tube, pirk_report* report) {
    if (!ctx || !spec) return PIRK_EINVAL;
    LOCK(ctx);
    ctx->err.clear();
    if (cudaSetDevice(ctx->device) != cudaSuccess) return fail(ctx, PIRK_ECUDA, "cudaSetDevice failed");
    pirk_status st = PIRK_OK;
    if (!check_problem(ctx, m, p, true, st)) return st;
    if (is_user(m) && !(m->program->flags & PIRK_HAS_RHS))
        return fail(ctx, PIRK_EINVAL, "monte_carlo: model has no vector field");
    uint64_t count = spec->samples_override;
    if (count == 0) {
        if (pirk_sample_count(m->dim, spec->epsilon, spec->delta, &count) != PIRK_OK) {
            if (!(spec->epsilon > 0.0) || !(spec->epsilon < 1.0))
                return fail(ctx, PIRK_EINVAL, "sample_count: epsilon must be in (0, 1)");
            return fail(ctx, PIRK_EINVAL, "sample_count: delta must be in (0, 1)");
        }
    }
    try {
        return run_mc(ctx, m, p, spec->seed, 0, count, count, tube, false, report, nullptr, nullptr, nullptr);
    } catch (const std::bad_alloc&) {
        return fail(ctx, PIRK_ENOMEM, "host allocation failed");
    }
}

pirk_status pirk_monte_carlo_range(pirk_ctx* ctx, const pirk_model* m, const pirk_problem* p,
                                   uint64_t seed, uint64_t s_begin, uint64_t s_end,
                                   pirk_tube* tube, pirk_report* report) {
    if (!ctx) return PIRK_EINVAL;
    LOCK(ctx);
    ctx->err.clear();
    if (cudaSetDevice(ctx->device) != cudaSuccess) return fail(ctx, PIRK_ECUDA, "cudaSetDevice failed");
    pirk_status st = PIRK_OK;
    if (!check_problem(ctx, m, p, true, st)) return st;
    if (s_end < s_begin) return fail(ctx, PIRK_EINVAL, "monte_carlo_range: s_end < s_begin");
    if (s_end == s_begin) {
        if (tube) tube->n_slots = pirk_record_schedule(p->t0, p->t1, p->h, p->tube_stride, nullptr, tube->times);
        return PIRK_OK;
    }
    try {
        return run_mc(ctx, m, p, seed, s_begin, s_end, s_end - s_begin, tube, true, report, nullptr, nullptr, nullptr);
    } catch (const std::bad_alloc&) {
        return fail(ctx, PIRK_ENOMEM, "host allocation failed");
    }
}

pirk_status pirk_coverage_estimate(pirk_ctx* ctx, const pirk_model* m, const pirk_problem* p,
                                   const double* box_lower, const double* box_upper,
                                   uint64_t fresh_samples, uint64_t seed, double* fraction) {
    if (!ctx || !fraction) return PIRK_EINVAL;
    LOCK(ctx);
    ctx->err.clear();
    pirk_status st = PIRK_OK;
    if (!check_problem(ctx, m, p, true, st)) return st;
    if (!box_lower || !box_upper) return fail(ctx, PIRK_EINVAL, "coverage_estimate: tube has no entries");
    if (fresh_samples == 0) return fail(ctx, PIRK_EINVAL, "coverage_estimate: fresh_samples must be positive");
    try {
        return run_mc(ctx, m, p, seed, 0, fresh_samples, fresh_samples, nullptr, false, nullptr,
                      box_lower, box_upper, fraction);
    } catch (const std::bad_alloc&) {
        return fail(ctx, PIRK_ENOMEM, "host allocation failed");
    }
}

pirk_status pirk_engine_create(pirk_ctx* ctx, const pirk_model* m, int32_t method,
                               const pirk_problem* p, pirk_engine** out) {
    if (!ctx || !out) return PIRK_EINVAL;
    LOCK(ctx);
    *out = nullptr;
    ctx->err.clear();
    if (cudaSetDevice(ctx->device) != cudaSuccess) return fail(ctx, PIRK_ECUDA, "cudaSetDevice failed");
    pirk_status st = PIRK_OK;
    if (!check_problem(ctx, m, p, false, st)) return st;
    if (!(is_chain(m) || is_heat(m)) || !pirk_supports(m, method))
        return fail(ctx, PIRK_EUNSUPPORTED, "engine: only the chain and heat3d kernels run as engines");
    pirk_engine* e = new (std::nothrow) pirk_engine;
    if (!e) return PIRK_ENOMEM;
    st = engine_init(ctx, m, method, p, e);
    if (st != PIRK_OK) {
        delete e;
        return st;
    }
    *out = e;
    return PIRK_OK;
}

pirk_status pirk_engine_advance(pirk_engine* e, uint64_t nsteps) {
    if (!e) return PIRK_EINVAL;
    LOCK(e->ctx);
    return engine_advance(e, nsteps);
}

pirk_status pirk_engine_status(pirk_engine* e, uint64_t* steps_done) {
    if (!e) return PIRK_EINVAL;
    LOCK(e->ctx);
    pirk_ctx* ctx = e->ctx;
    unsigned long long f[2];
    CK(ctx, cudaMemcpyAsync(f, e->d_fail.p, sizeof f, cudaMemcpyDeviceToHost, ctx->stream));
    CK(ctx, cudaStreamSynchronize(ctx->stream));
    if (steps_done) *steps_done = e->done;
    for (int i = 0; i < 2; ++i) {
        if (f[i] != kNoFail) {
            const uint64_t s = f[i] >> kFailCompBits, c = f[i] & ((1ull << kFailCompBits) - 1);
            return fail(ctx, PIRK_EINTEGRATION, integ_msg(s, c, e->t0 + static_cast<double>(s) * e->h));
        }
    }
    return PIRK_OK;
}

pirk_status pirk_engine_read(pirk_engine* e, double* lower, double* upper) {
    if (!e) return PIRK_EINVAL;
    LOCK(e->ctx);
    pirk_ctx* ctx = e->ctx;
    const uint64_t n = e->n;
    const double* lo = e->s0();
    const double* hi = e->s1();
    if (e->method == PIRK_METHOD_GB) {
        CK(ctx, cudaMemsetAsync(ctx->d_flags, 0xff, sizeof(unsigned long long), ctx->stream));
        CK(ctx, launch_gb_box(e->s0(), e->s1(), e->o0(), e->o1(), n, ctx->d_flags, ctx->stream));
        ctx->launches++;
        lo = e->o0();
        hi = e->o1();
    }
    if (lower) CK(ctx, cudaMemcpyAsync(lower, lo, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    if (upper) CK(ctx, cudaMemcpyAsync(upper, hi, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(ctx, cudaStreamSynchronize(ctx->stream));
    return PIRK_OK;
}

void pirk_engine_destroy(pirk_engine* e) {
    if (!e) return;
    std::lock_guard<std::recursive_mutex> lk(e->ctx->mu);
    delete e;
}

namespace {
pirk_status step_window_impl(pirk_ctx* ctx, const pirk_model* m, int32_t method, const pirk_window* win,
                             const pirk_mirror* mir, const double* p0, const double* p1, double t,
                             double hk, uint64_t step_index, uint64_t* fail_ptr) {
    if (!ctx || !win) return PIRK_EINVAL;
    LOCK(ctx);
    pirk_status st = PIRK_OK;
    if (!check_model(ctx, m, st)) return st;
    if (!(is_chain(m) || is_heat(m)) || !pirk_supports(m, method))
        return fail(ctx, PIRK_EUNSUPPORTED, "step_window: only the chain and heat3d kernels are windowed");
    const uint64_t unit = is_heat(m) ? m->grid * m->grid : 1;
    const uint64_t units = m->dim / unit;
    const uint64_t wb = win->win_begin, we = win->win_begin + win->win_len;
    if (we > units || win->out_begin < wb || win->out_end > we || win->out_begin > win->out_end)
        return fail(ctx, PIRK_EINVAL, "step_window: window outside the state");
    const uint64_t need_lo = win->out_begin >= 4 ? win->out_begin - 4 : 0;
    const uint64_t need_hi = (win->out_end + 4 <= units) ? win->out_end + 4 : units;
    if (wb > need_lo || we < need_hi)
        return fail(ctx, PIRK_EINVAL, "step_window: window must cover the output range +-4 units");
    double q0 = 0.0, q1 = 0.0;
    if (m->input_dim > 0) {
        if (!p0 || !p1) return fail(ctx, PIRK_EINVAL, "step_window: inputs missing");
        q0 = p0[0];
        q1 = p1[0];
    }
    StepConsts sc;  // rk4.cpp:38-39
    sc.t = t;
    sc.hk = hk;
    sc.h2 = 0.5 * hk;
    sc.h6 = hk / 6.0;
    const ChainModel cm = chain_model(m, method, q0, q1);
    const HeatModel hm = heat_model(m, method);
    WindowArgs w{win->in0, win->in1, win->out0, win->out1, wb, we, win->out_begin, win->out_end};
    if (mir) {
        if ((mir->lo0 == nullptr) != (mir->lo1 == nullptr) || (mir->hi0 == nullptr) != (mir->hi1 == nullptr))
            return fail(ctx, PIRK_EINVAL, "step_window_mirror: a mirror side needs both fields");
        if (mir->lo0) {
            w.mir0 = mir->lo0;
            w.mir1 = mir->lo1;
            w.mir_lo_end = mir->lo_end;
        }
        if (mir->hi0) {
            w.mirh0 = mir->hi0;
            w.mirh1 = mir->hi1;
            w.mir_hi_begin = mir->hi_begin;
        }
    }
    CK(ctx, step_launch(ctx, ctx->stream, m, cm, hm, w, sc, step_index,
                        reinterpret_cast<unsigned long long*>(fail_ptr)));
    return PIRK_OK;
}

// driver entry points (no link-time libcuda dependency)
struct DriverFns {
    decltype(&cuStreamWaitValue32) wait32 = nullptr;
    decltype(&cuMemGetAddressRange) range = nullptr;
    bool ok = false;
};
const DriverFns& driver_fns() {
    static DriverFns f = [] {
        DriverFns d;
        cudaDriverEntryPointQueryResult q1, q2;
        void* a = nullptr;
        void* b = nullptr;
        if (cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", &a, 12000, cudaEnableDefault, &q1) ==
                cudaSuccess &&
            q1 == cudaDriverEntryPointSuccess &&
            cudaGetDriverEntryPointByVersion("cuMemGetAddressRange", &b, 12000, cudaEnableDefault, &q2) ==
                cudaSuccess &&
            q2 == cudaDriverEntryPointSuccess) {
            d.wait32 = reinterpret_cast<decltype(&cuStreamWaitValue32)>(a);
            d.range = reinterpret_cast<decltype(&cuMemGetAddressRange)>(b);
            d.ok = true;
        }
        cudaGetLastError();
        return d;
    }();
    return f;
}

// pirk_ipc_open mappings: handle bytes -> (base, count), process-wide
struct IpcMap {
    std::mutex mu;
    std::map<std::string, std::pair<void*, int>> by_handle;
    std::map<void*, std::string> by_base;
};
IpcMap& ipc_map() {
    static IpcMap m;
    return m;
}
}  // namespace

pirk_status pirk_step_window(pirk_ctx* ctx, const pirk_model* m, int32_t method,
                             const pirk_window* win, const double* p0, const double* p1,
                             double t, double hk, uint64_t step_index, uint64_t* fail_ptr) {
    return step_window_impl(ctx, m, method, win, nullptr, p0, p1, t, hk, step_index, fail_ptr);
}

pirk_status pirk_step_window_mirror(pirk_ctx* ctx, const pirk_model* m, int32_t method,
                                    const pirk_window* win, const pirk_mirror* mirror,
                                    const double* p0, const double* p1, double t, double hk,
                                    uint64_t step_index, uint64_t* fail_ptr) {
    if (!mirror) return ctx ? fail(ctx, PIRK_EINVAL, "step_window_mirror: mirror missing") : PIRK_EINVAL;
    return step_window_impl(ctx, m, method, win, mirror, p0, p1, t, hk, step_index, fail_ptr);
}

pirk_status pirk_ipc_export(const void* dptr, unsigned char handle[64], uint64_t* offset) {
    if (!dptr || !handle || !offset) return PIRK_EINVAL;
    const DriverFns& d = driver_fns();
    if (!d.ok) return PIRK_ECUDA;
    CUdeviceptr base = 0;
    size_t size = 0;
    if (d.range(&base, &size, reinterpret_cast<CUdeviceptr>(dptr)) != CUDA_SUCCESS) return PIRK_EINVAL;
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)) != cudaSuccess) {
        cudaGetLastError();
        return PIRK_ECUDA;
    }
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    std::memcpy(handle, &h, 64);
    *offset = static_cast<uint64_t>(reinterpret_cast<CUdeviceptr>(dptr) - base);
    return PIRK_OK;
}

pirk_status pirk_ipc_open(int device, const unsigned char handle[64], void** base) {
    if (!handle || !base) return PIRK_EINVAL;
    *base = nullptr;
    IpcMap& m = ipc_map();
    std::lock_guard<std::mutex> lk(m.mu);
    std::string key(reinterpret_cast<const char*>(handle), 64);
    key += std::to_string(device);
    auto it = m.by_handle.find(key);
    if (it != m.by_handle.end()) {
        it->second.second++;
        *base = it->second.first;
        return PIRK_OK;
    }
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, 64);
    void* p = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    cudaSetDevice(prev);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return PIRK_ECUDA;
    }
    m.by_handle[key] = {p, 1};
    m.by_base[p] = key;
    *base = p;
    return PIRK_OK;
}

pirk_status pirk_ipc_close(void* base) {
    if (!base) return PIRK_EINVAL;
    IpcMap& m = ipc_map();
    std::lock_guard<std::mutex> lk(m.mu);
    auto it = m.by_base.find(base);
    if (it == m.by_base.end()) return PIRK_EINVAL;
    auto& ent = m.by_handle[it->second];
    if (--ent.second > 0) return PIRK_OK;
    m.by_handle.erase(it->second);
    m.by_base.erase(it);
    return cudaIpcCloseMemHandle(base) == cudaSuccess ? PIRK_OK : (cudaGetLastError(), PIRK_ECUDA);
}

pirk_status pirk_wait_flag(pirk_ctx* ctx, const uint32_t* flag, uint32_t value) {
    if (!ctx || !flag) return PIRK_EINVAL;
    LOCK(ctx);
    const DriverFns& d = driver_fns();
    if (!d.ok) return fail(ctx, PIRK_ECUDA, "wait_flag: driver entry point cuStreamWaitValue32 missing");
    if (d.wait32(reinterpret_cast<CUstream>(ctx->stream), reinterpret_cast<CUdeviceptr>(flag), value,
                 CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
        return fail(ctx, PIRK_ECUDA, "wait_flag: cuStreamWaitValue32 failed");
    return PIRK_OK;
}

pirk_status pirk_signal_flag(pirk_ctx* ctx, uint32_t* flag, uint32_t value) {
    if (!ctx || !flag) return PIRK_EINVAL;
    LOCK(ctx);
    ctx->launches++;
    CK(ctx, launch_signal_flag(flag, value, ctx->stream));
    return PIRK_OK;
}

pirk_status pirk_program_create(const char* source, uint64_t dim, uint64_t input_dim, uint32_t flags,
                                pirk_program** out) {
    if (!out) return PIRK_EINVAL;
    *out = nullptr;
    if (!source || dim == 0) return PIRK_EINVAL;
    pirk_program* pg = new (std::nothrow) pirk_program;
    if (!pg) return PIRK_ENOMEM;
    pg->source = source;
    pg->dim = dim;
    pg->input_dim = input_dim;
    pg->flags = flags;
    *out = pg;
    return PIRK_OK;
}

pirk_status pirk_program_compile(pirk_program* pg, int32_t mode, char* log, size_t log_len,
                                 uint64_t* cubin_bytes) {
    if (!pg || (mode != PIRK_MODE_EXACT && mode != PIRK_MODE_FAST)) return PIRK_EINVAL;
    std::lock_guard<std::mutex> lk(pg->mu);
    UserBuild& b = pg->build[mode == PIRK_MODE_EXACT ? 0 : 1];
    const bool ok = user_compile(pg, mode, b);
    if (log && log_len) {
        std::snprintf(log, log_len, "%s", b.log.c_str());
    }
    if (cubin_bytes) *cubin_bytes = ok ? b.cubin.size() : 0;
    return ok ? PIRK_OK : PIRK_EINVAL;
}

pirk_status pirk_program_cubin(const pirk_program* pg, int32_t mode, void* buf, uint64_t len) {
    if (!pg || !buf || (mode != PIRK_MODE_EXACT && mode != PIRK_MODE_FAST)) return PIRK_EINVAL;
    const UserBuild& b = pg->build[mode == PIRK_MODE_EXACT ? 0 : 1];
    if (!b.ok || len < b.cubin.size()) return PIRK_EINVAL;
    std::memcpy(buf, b.cubin.data(), b.cubin.size());
    return PIRK_OK;
}

pirk_status pirk_program_set_stencil(pirk_program* pg, uint64_t radius) {
    if (!pg || radius > kUserStencilMax) return PIRK_EINVAL;
    std::lock_guard<std::mutex> lk(pg->mu);
    if (pg->build[0].tried || pg->build[1].tried) return PIRK_EINVAL;  // before the first compile
    pg->stencil = radius;
    return PIRK_OK;
}

void pirk_program_destroy(pirk_program* pg) { delete pg; }

}  // extern "C"
