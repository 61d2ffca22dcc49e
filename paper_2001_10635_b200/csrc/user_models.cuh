// user_models.cuh -- host side of user-defined models (pirk_program), included
// by engine.cu inside its anonymous namespace.
//
// A pirk_program holds the caller's CUDA source for f / d / g (the reference's
// SystemModel evaluators, system_model.hpp:14-43; conventions in user_rt.cuh).
// It is compiled with NVRTC for sm_100a the first time a context uses it in a
// given arithmetic mode (exact: --fmad=false) and loaded as a context-
// independent cudaLibrary_t, so every lane/device of a context can launch it.
// A compile error is the model being invalid: PIRK_EINVAL with the NVRTC log.

bool is_user(const pirk_model* m) { return m->kind == PIRK_USER; }
pirk_program* user_program(const pirk_model* m) { return const_cast<pirk_program*>(m->program); }
bool user_has(const pirk_model* m, uint32_t f) { return m->program && (m->program->flags & f) != 0; }

#define NVRTC_CK(expr, what)                                           \
    do {                                                               \
        nvrtcResult r_ = (expr);                                       \
        if (r_ != NVRTC_SUCCESS) {                                     \
            b.log += std::string(what) + ": " + nvrtcGetErrorString(r_); \
            return false;                                              \
        }                                                              \
    } while (0)

// NVRTC compile of prelude + user source + kernels (cached per mode).
bool user_compile(pirk_program* pg, int mode, UserBuild& b) {
    if (b.tried) return b.ok;
    b.tried = true;
    const std::string src = std::string(kUserPrelude) + "\n#line 1 \"user_model.cu\"\n" + pg->source +
                            "\n#line 1 \"pirk_user_kernels\"\n" + kUserKernels;
    nvrtcProgram prog = nullptr;
    NVRTC_CK(nvrtcCreateProgram(&prog, src.c_str(), "pirk_user.cu", 0, nullptr, nullptr), "nvrtcCreateProgram");
    std::vector<std::string> opt = {
        "--gpu-architecture=sm_100a", "--std=c++17", "-default-device",
        mode == PIRK_MODE_EXACT ? "--fmad=false" : "--fmad=true",
        "-DPIRK_N=" + std::to_string(pg->dim) + "ull", "-DPIRK_NI=" + std::to_string(pg->input_dim) + "ull",
        "-DPIRK_HAS_RHS=" + std::to_string((pg->flags & PIRK_HAS_RHS) ? 1 : 0),
        "-DPIRK_HAS_DECOMP=" + std::to_string((pg->flags & PIRK_HAS_DECOMPOSITION) ? 1 : 0),
        "-DPIRK_HAS_GROWTH=" + std::to_string((pg->flags & PIRK_HAS_GROWTH) ? 1 : 0),
        "-DPIRK_STENCIL=" + std::to_string(pg->stencil)};
    std::vector<const char*> ov;
    for (const std::string& o : opt) ov.push_back(o.c_str());
    const nvrtcResult cr = nvrtcCompileProgram(prog, static_cast<int>(ov.size()), ov.data());
    size_t log_size = 0;
    nvrtcGetProgramLogSize(prog, &log_size);
    if (log_size > 1) {
        std::string lg(log_size, '\0');
        nvrtcGetProgramLog(prog, &lg[0]);
        lg.resize(std::strlen(lg.c_str()));
        b.log += lg;
    }
    if (cr != NVRTC_SUCCESS) {
        b.log = "user model: NVRTC compile failed (" + std::string(nvrtcGetErrorString(cr)) + "):\n" + b.log;
        nvrtcDestroyProgram(&prog);
        return false;
    }
    size_t n = 0;
    nvrtcGetCUBINSize(prog, &n);
    b.cubin.resize(n);
    nvrtcGetCUBIN(prog, b.cubin.data());
    nvrtcDestroyProgram(&prog);
    b.ok = true;
    return true;
}

// Compiled and loaded kernels of `m`'s program for the context's mode.
pirk_status user_kernels(pirk_ctx* ctx, const pirk_model* m, UserBuild** out) {
    pirk_program* pg = user_program(m);
    std::lock_guard<std::mutex> lk(pg->mu);
    UserBuild& b = pg->build[ctx->mode == PIRK_MODE_EXACT ? 0 : 1];
    if (!user_compile(pg, ctx->mode, b)) return fail(ctx, PIRK_EINVAL, b.log);
    if (!b.lib) {
        CK(ctx, cudaLibraryLoadData(&b.lib, b.cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
        CK(ctx, cudaLibraryGetKernel(&b.k_small, b.lib, "pirk_user_small"));
        CK(ctx, cudaLibraryGetKernel(&b.k_stage, b.lib, "pirk_user_stage"));
        CK(ctx, cudaLibraryGetKernel(&b.k_mc, b.lib, "pirk_user_mc"));
        if (pg->stencil > 0) CK(ctx, cudaLibraryGetKernel(&b.k_tile, b.lib, "pirk_user_tile"));
    }
    *out = &b;
    return PIRK_OK;
}

cudaError_t user_launch_small(UserBuild* b, int which, const double* x0, const double* p, double t0, double t1,
                              double h, unsigned long long total, unsigned long long stride, double* rec,
                              unsigned long long* fail, cudaStream_t stream) {
    void* args[] = {&which, &x0, &p, &t0, &t1, &h, &total, &stride, &rec, &fail};
    return cudaLaunchKernel(reinterpret_cast<const void*>(b->k_small), dim3(1), dim3(32), args, 0, stream);
}

// McArgs and user_rt.cuh's UserMcArgs share their layout.
cudaError_t user_launch_mc(UserBuild* b, const McArgs& a, cudaStream_t stream) {
    if (a.s_end <= a.s_begin) return cudaSuccess;
    const unsigned long long count = a.s_end - a.s_begin;
    McArgs copy = a;
    void* args[] = {&copy};
    return cudaLaunchKernel(reinterpret_cast<const void*>(b->k_mc),
                            dim3(static_cast<unsigned>((count + 127) / 128)), dim3(128), args, 0, stream);
}

cudaError_t user_launch_stage(UserBuild* b, int which, int stage, double t0, double t1, double h,
                              unsigned long long step, unsigned long long total, double* x, const double* ui,
                              double* uo, double* acc, const double* p, unsigned long long D,
                              unsigned long long* fail, cudaStream_t stream) {
    void* args[] = {&which, &stage, &t0, &t1, &h, &step, &total, &x, &ui, &uo, &acc, &p, &D, &fail};
    return cudaLaunchKernel(reinterpret_cast<const void*>(b->k_stage), dim3(static_cast<unsigned>((D + 255) / 256)),
                            dim3(256), args, 0, stream);
}

size_t user_tile_smem(uint64_t radius) { return 8 * (kUserTile + 8 * radius) * sizeof(double); }

cudaError_t user_launch_tile(UserBuild* b, uint64_t radius, int which, double t0, double t1, double h,
                             unsigned long long step, unsigned long long total, const double* in0,
                             const double* in1, double* out0, double* out1, const double* p, unsigned long long n,
                             unsigned long long* fail, cudaStream_t stream) {
    const size_t smem = user_tile_smem(radius);
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (!(b->tile_devices & (1ull << (dev & 63)))) {  // dynamic shared memory opt-in, per device
        e = cudaKernelSetAttributeForDevice(b->k_tile, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(smem), dev);
        if (e != cudaSuccess) return e;
        b->tile_devices |= 1ull << (dev & 63);
    }
    void* args[] = {&which, &t0, &t1, &h, &step, &total, &in0, &in1, &out0, &out1, &p, &n, &fail};
    return cudaLaunchKernel(reinterpret_cast<const void*>(b->k_tile),
                            dim3(static_cast<unsigned>((n + kUserTile - 1) / kUserTile)), dim3(kUserTileThreads),
                            args, smem, stream);
}

// MM / GB of a user model with n > kUserSmallMax: one thread per component,
// four stage launches per RK4 step (pirk_user_stage), any stencil the
// evaluators read.  Slots go straight to the caller's tube; GB composes the
// box on the host after both integrations (reach.cpp:103-134).
pirk_status run_user_large(pirk_ctx* ctx, const pirk_model* m, int method, const pirk_problem* p,
                           pirk_tube* tube, pirk_report* rep) {
    const auto t_setup = Clock::now();
    const uint64_t launches0 = ctx->launches;
    UserBuild* ub = nullptr;
    pirk_status st = user_kernels(ctx, m, &ub);
    if (st != PIRK_OK) return st;
    Plan plan;
    plan_steps(p->t0, p->t1, p->h, plan);
    if (plan.total >= (1ull << 23))
        return fail(ctx, PIRK_EINVAL, "step count exceeds the device failure-key range (2^23)");
    std::vector<uint64_t> slot_steps;
    std::vector<double> slot_times;
    record_schedule(p->t0, p->t1, p->h, p->tube_stride, plan, slot_steps, slot_times);
    const uint64_t S = slot_steps.size();
    if (tube && tube->max_slots < S) return fail(ctx, PIRK_EINVAL, "tube: max_slots too small");
    const uint64_t n = m->dim, ni = m->input_dim;
    const bool mm = method == PIRK_METHOD_MM;
    const uint64_t D = mm ? 2 * n : n;
    // radius-r stencil models: one fused step per launch on ping-pong field
    // buffers (X holds [field 0 | field 1], UA the other copy)
    const bool tiled = user_program(m)->stencil > 0 && ub->k_tile;
    DevBuf<double> X, UA, UB, ACC, P;
    DevBuf<unsigned long long> dfail, sflag;
    CK(ctx, X.alloc(ctx, D));
    CK(ctx, UA.alloc(ctx, D));
    CK(ctx, UB.alloc(ctx, D));
    CK(ctx, ACC.alloc(ctx, D));
    CK(ctx, P.alloc(ctx, 2 * ni + 1));
    CK(ctx, dfail.alloc(ctx, 2));
    CK(ctx, sflag.alloc(ctx, S));
    CK(ctx, cudaMemsetAsync(dfail.p, 0xff, 2 * sizeof(unsigned long long), ctx->stream));
    CK(ctx, cudaMemsetAsync(sflag.p, 0xff, S * sizeof(unsigned long long), ctx->stream));
    std::vector<double> hc, hr;  // GB: host centres and radii, slots x n
    SlotStreamer rec;  // MM: slots stream to the record callback during the run
    if (mm) CK(ctx, rec.init(ctx, n, 1));
    const double setup_s = since(t_setup);
    const auto t_int = Clock::now();
    for (int pass = 0; pass < (mm ? 1 : 2); ++pass) {
        const int which = mm ? 2 : pass;
        std::vector<double> x0(D), pp(2 * ni + 1, 0.0);
        for (uint64_t i = 0; i < n; ++i) {
            if (mm) {  // [lower | upper], [p_lo | p_hi] (reach.cpp:150-161)
                x0[i] = p->init_lower[i];
                x0[n + i] = p->init_upper[i];
            } else {  // centre / half-width (interval.cpp:25-37)
                x0[i] = pass == 0 ? 0.5 * (p->init_upper[i] + p->init_lower[i])
                                  : 0.5 * (p->init_upper[i] - p->init_lower[i]);
            }
        }
        for (uint64_t j = 0; j < ni; ++j) {
            if (mm) {
                pp[j] = p->input_lower[j];
                pp[ni + j] = p->input_upper[j];
            } else {
                pp[j] = pass == 0 ? 0.5 * (p->input_upper[j] + p->input_lower[j])
                                  : 0.5 * (p->input_upper[j] - p->input_lower[j]);
            }
        }
        CK(ctx, cudaMemcpyAsync(X.p, x0.data(), D * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        CK(ctx, cudaMemcpyAsync(P.p, pp.data(), pp.size() * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        if (!mm) (pass == 0 ? hc : hr).resize(S * n);
        uint64_t done = 0;
        for (uint64_t s = 0; s < S; ++s) {
            for (; done < slot_steps[s]; ++done) {
                if (tiled) {  // X -> UA in one launch, then swap (the copy back keeps X the state)
                    const uint64_t nn = n;
                    CK(ctx, user_launch_tile(ub, user_program(m)->stencil, which, p->t0, p->t1, p->h, done,
                                             plan.total, X.p, X.p + nn, UA.p, UA.p + nn, P.p, nn,
                                             dfail.p + pass, ctx->stream));
                    ctx->launches++;
                    std::swap(X.p, UA.p);
                    continue;
                }
                const double* ins[4] = {X.p, UA.p, UB.p, UA.p};
                double* outs[4] = {UA.p, UB.p, UA.p, nullptr};
                for (int stg = 0; stg < 4; ++stg) {
                    CK(ctx, user_launch_stage(ub, which, stg, p->t0, p->t1, p->h, done, plan.total, X.p, ins[stg],
                                              outs[stg], ACC.p, P.p, D, dfail.p + pass, ctx->stream));
                    ctx->launches++;
                }
            }
            if (mm) {
                CK(ctx, rec.deliver());
                CK(ctx, launch_order_check(X.p, X.p + n, n, sflag.p + s, ctx->stream));  // reach.cpp:181-186
                ctx->launches++;
                if (tube && tube->lower)
                    CK(ctx, cudaMemcpyAsync(tube->lower + s * n, X.p, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
                if (tube && tube->upper)
                    CK(ctx, cudaMemcpyAsync(tube->upper + s * n, X.p + n, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
                if (rec.on()) {
                    CK(ctx, cudaMemcpyAsync(rec.buf, X.p, 2 * n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
                    CK(ctx, rec.mark(0, ctx->stream));
                    rec.set_pending(s, slot_steps[s], slot_times[s]);
                }
            } else {
                double* dst = (pass == 0 ? hc : hr).data() + s * n;
                CK(ctx, cudaMemcpyAsync(dst, X.p, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
            }
        }
        CK(ctx, cudaStreamSynchronize(ctx->stream));
    }
    CK(ctx, rec.deliver());
    unsigned long long hf[2];
    std::vector<unsigned long long> flags(S);
    CK(ctx, cudaMemcpyAsync(hf, dfail.p, sizeof hf, cudaMemcpyDeviceToHost, ctx->stream));
    CK(ctx, cudaMemcpyAsync(flags.data(), sflag.p, S * sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
    CK(ctx, cudaStreamSynchronize(ctx->stream));
    const double integ_s = since(t_int);
    if (tube) {
        tube->n_slots = S;
        if (tube->times)
            for (uint64_t s = 0; s < S; ++s) tube->times[s] = slot_times[s];
    }
    std::vector<double> vals(S, 0.0);
    if (!mm) {  // clamp / negative radius (reach.cpp:121-134), then the box
        for (uint64_t s = 0; s < S; ++s) {
            for (uint64_t i = 0; i < n && flags[s] == kNoFail; ++i) {
                double& r = hr[s * n + i];
                if (r < 0.0) {
                    if (r < -1e-12) {
                        flags[s] = i;
                        vals[s] = r;
                        break;
                    }
                    r = 0.0;
                }
            }
            if (tube && tube->lower)
                for (uint64_t i = 0; i < n; ++i) tube->lower[s * n + i] = hc[s * n + i] - hr[s * n + i];
            if (tube && tube->upper)
                for (uint64_t i = 0; i < n; ++i) tube->upper[s * n + i] = hc[s * n + i] + hr[s * n + i];
            if (ctx->record_fn && flags[s] == kNoFail) {
                std::vector<double> lo(n), hi(n);
                for (uint64_t i = 0; i < n; ++i) {
                    lo[i] = hc[s * n + i] - hr[s * n + i];
                    hi[i] = hc[s * n + i] + hr[s * n + i];
                }
                ctx->record_fn(ctx->record_user, s, slot_steps[s], slot_times[s], lo.data(), hi.data(), n);
            }
        }
    }
    return large_errors(ctx, method, p, plan.total, slot_steps, slot_times, hf[0], hf[1], flags, vals, n,
                        4 * D * sizeof(double), setup_s, integ_s, ctx->launches - launches0, 1, rep);
}

// ----------------------------------------------------- catalog fields as source
//
// Monte Carlo of a catalog model with n > kSmallMax (the compiled MC kernels
// hold a sample in registers for n <= 64): its vector field is generated as
// user-model source with the constants the reference's make_* computes
// (models.cpp:47-133, SURVEY.md 8d chain) printed as exact hex-float literals,
// and runs on pirk_user_mc (n <= kUserMcMax).  Same expressions, same order:
// bit-identical to the reference in exact mode.

std::string hexf(double v) {
    char b[64];
    std::snprintf(b, sizeof b, "%a", v);
    return b;
}

bool catalog_mc_source_ok(const pirk_model* m) {
    return (m->kind == PIRK_TRAFFIC || m->kind == PIRK_HEAT3D || m->kind == PIRK_CHAIN || m->kind == PIRK_ZERO) &&
           m->dim <= kUserMcMax;
}

std::string catalog_source(const pirk_model* m) {
    const double* P = m->params;
    std::string s;
    if (m->kind == PIRK_TRAFFIC) {  // models.cpp:55-75
        s = "namespace cat { constexpr double V = " + hexf(P[0]) + ", W = " + hexf(P[1]) + ", C = " + hexf(P[2]) +
            ", XBAR = " + hexf(P[3]) + ", BETA = " + hexf(P[5]) + ", INV_T = " + hexf(1.0 / P[4]) + "; }\n";
        s += R"(
__device__ double flux(double from, double into) {
    return pirk_min(cat::C, pirk_min(cat::V * from, cat::W * (cat::XBAR - into) / cat::BETA));
}
__device__ double pirk_rhs(u64 i, double, const double* x, const double* p) {
    const double in = (i == 0) ? cat::BETA * p[0] : cat::BETA * flux(x[i - 1], x[i]);
    const double out = (i + 1 == PIRK_N) ? pirk_min(cat::C, cat::V * x[i]) : flux(x[i], x[i + 1]);
    return cat::INV_T * (in - out);
}
)";
    } else if (m->kind == PIRK_HEAT3D) {  // models.cpp:99-127
        const double delta = 1.0 / static_cast<double>(m->grid - 1);
        s = "namespace cat { constexpr u64 G = " + std::to_string(m->grid) + "ull; constexpr double KK = " +
            hexf(P[0] / (delta * delta)) + ", ROBIN = " + hexf(2.0 * delta * P[1]) + "; }\n";
        s += R"(
__device__ double pirk_rhs(u64 i, double, const double* x, const double*) {
    using namespace cat;
    const u64 ix = i % G, iy = (i / G) % G, iz = i / (G * G);
    const double self = x[i];
    double acc = 0.0;
    if (ix > 0) acc += x[i - 1] - self;
    else acc += (x[i + 1] - self) - ROBIN * self;
    if (ix + 1 < G) acc += x[i + 1] - self;
    if (iy > 0) acc += x[i - G] - self;
    if (iy + 1 < G) acc += x[i + G] - self;
    if (iz > 0) acc += x[i - G * G] - self;
    if (iz + 1 < G) acc += x[i + G * G] - self;
    return KK * acc;
}
)";
    } else if (m->kind == PIRK_CHAIN) {  // f = d(x, p, x, p)
        s = "namespace cat { constexpr double A = " + hexf(P[0]) + ", B = " + hexf(P[1]) + ", CC = " + hexf(P[2]) +
            "; }\n";
        s += R"(
__device__ double chain_s(double z) { return z / (1.0 + fabs(z)); }
__device__ double pirk_rhs(u64 i, double, const double* x, const double* p) {
    const double sl = (i == 0) ? 0.0 : chain_s(x[i - 1]);
    const double sr = (i + 1 == PIRK_N) ? 0.0 : chain_s(x[i + 1]);
    return ((-cat::A) * x[i] + cat::B * sl - cat::CC * sr) + p[0];
}
)";
    } else {  // PIRK_ZERO, models.cpp:621-623
        s = "__device__ double pirk_rhs(u64, double, const double*, const double*) { return 0.0; }\n";
    }
    return s;
}

// Point `um` at the (cached, per context) program of `m`'s generated field.
bool catalog_mc_program(pirk_ctx* ctx, const pirk_model* m, pirk_model& um) {
    if (!catalog_mc_source_ok(m)) return false;
    const std::string src = catalog_source(m);
    std::unique_ptr<pirk_program>& pg = ctx->catalog_programs[src];
    if (!pg) {
        pg.reset(new pirk_program);
        pg->source = src;
        pg->dim = m->dim;
        pg->input_dim = m->input_dim;
        pg->flags = PIRK_HAS_RHS;
    }
    um = *m;
    um.kind = PIRK_USER;
    um.program = pg.get();
    return true;
}
