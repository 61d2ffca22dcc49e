/*
 * pirk_oracle.c -- TEST INFRASTRUCTURE ONLY (see pirk_oracle.h).
 *
 * CPU restatement of the reference's hot path.  Every function cites the
 * reference file:line (relative to /root/reference/proj) it restates.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load the
 * shared library built from this file.
 */
#include "pirk_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ rng.hpp */

uint64_t po_mix64(uint64_t z) { /* rng.hpp:11-16 */
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

double po_u01(uint64_t seed, uint64_t stream, uint64_t index) { /* rng.hpp:19-23 */
    uint64_t z = po_mix64(po_mix64(po_mix64(seed) ^ (stream * 0xd1342543de82ef95ull)) ^
                          (index * 0xaf251af3b0f025b5ull));
    return (double)(z >> 11) * 0x1.0p-53;
}

double po_uniform_in(double lo, double hi, double u) { /* rng.hpp:26-29 */
    if (lo == hi) return lo;
    return lo + u * (hi - lo);
}

/* --------------------------------------------------------- step planning */

int po_plan_steps(double t0, double t1, double h, uint64_t* full_steps, int* has_remainder) {
    /* rk4.cpp:8-17 */
    if (!(h > 0.0)) return PO_EINVAL;
    if (!(t0 < t1)) return PO_EINVAL;
    const double span = t1 - t0;
    const uint64_t full = (uint64_t)floor(span / h + 1e-9);
    const double remainder = span - (double)full * h;
    *full_steps = full;
    *has_remainder = remainder > 1e-9 * h;
    return PO_OK;
}

static uint64_t plan_total(double t0, double t1, double h) {
    uint64_t full = 0;
    int rem = 0;
    if (po_plan_steps(t0, t1, h, &full, &rem) != PO_OK) return 0;
    return full + (rem ? 1 : 0);
}

uint64_t po_record_schedule(double t0, double t1, double h, uint64_t stride,
                            uint64_t* steps_out, double* times_out) {
    /* reach.cpp:28-39 */
    const uint64_t total = plan_total(t0, t1, h);
    uint64_t n = 0;
    if (stride > 0) {
        if (steps_out) steps_out[n] = 0;
        if (times_out) times_out[n] = t0;
        ++n;
        for (uint64_t k = stride; k < total; k += stride) {
            if (steps_out) steps_out[n] = k;
            if (times_out) times_out[n] = t0 + (double)k * h;
            ++n;
        }
    }
    if (steps_out) steps_out[n] = total;
    if (times_out) times_out[n] = t1;
    return n + 1;
}

int po_sample_count(uint64_t n, double epsilon, double delta, uint64_t* out) {
    /* reach.cpp:55-63 */
    if (n == 0) return PO_EINVAL;
    if (!(epsilon > 0.0) || !(epsilon < 1.0)) return PO_EINVAL;
    if (!(delta > 0.0) || !(delta < 1.0)) return PO_EINVAL;
    const double nn = 2.0 * (double)n;
    *out = (uint64_t)ceil(nn / epsilon * log(nn / delta));
    return PO_OK;
}

/* ------------------------------------------------------------------ models */

static double dmin(double a, double b) { return (b < a) ? b : a; } /* std::min */

/* traffic flux, models.cpp:59-61 */
static double traffic_flux(const double* P, double from, double into) {
    const double v = P[0], w = P[1], c = P[2], xbar = P[3], beta = P[5];
    return dmin(c, dmin(v * from, w * (xbar - into) / beta));
}

static double traffic_rhs(const po_model* m, uint64_t i, const double* x, const double* p) {
    /* models.cpp:55, 64-75 */
    const double* P = m->params;
    const double v = P[0], c = P[2], beta = P[5];
    const double inv_t = 1.0 / P[4];
    const uint64_t n = m->dim;
    const double in = (i == 0) ? beta * p[0] : beta * traffic_flux(P, x[i - 1], x[i]);
    const double out = (i + 1 == n) ? dmin(c, v * x[i]) : traffic_flux(P, x[i], x[i + 1]);
    return inv_t * (in - out);
}

static double traffic_growth(const po_model* m, uint64_t i, const double* r, const double* w) {
    /* models.cpp:78-87 */
    const double* P = m->params;
    const double v = P[0], wc = P[1], beta = P[5];
    const double inv_t = 1.0 / P[4];
    const double a_prev = beta * v * inv_t;
    const double a_next = (wc / beta) * inv_t;
    const double a_in = beta * inv_t;
    double g = (i == 0) ? a_in * w[0] : a_prev * r[i - 1];
    if (i + 1 < m->dim) g += a_next * r[i + 1];
    return g;
}

static double heat_rhs(const po_model* m, uint64_t i, const double* x) {
    /* models.cpp:99-127 */
    const uint64_t g = m->grid, g2 = g * g;
    const double alpha = m->params[0], exchange = m->params[1];
    const double delta = 1.0 / (double)(g - 1);
    const double k = alpha / (delta * delta);
    const double robin = 2.0 * delta * exchange;
    const uint64_t ix = i % g, iy = (i / g) % g, iz = i / g2;
    const double self = x[i];
    double acc = 0.0;
    if (ix > 0)
        acc += x[i - 1] - self;
    else
        acc += (x[i + 1] - self) - robin * self;
    if (ix + 1 < g) acc += x[i + 1] - self;
    if (iy > 0) acc += x[i - g] - self;
    if (iy + 1 < g) acc += x[i + g] - self;
    if (iz > 0) acc += x[i - g2] - self;
    if (iz + 1 < g) acc += x[i + g2] - self;
    return k * acc;
}

/* Synthetic coupled chain:
 *   f_i = -a x_i + b s(x_{i-1}) - c s(x_{i+1}) + p,  s(z) = z / (1 + |z|),
 *   x_{-1} = x_n = 0;   d_i reads x_{i+1} from the hatted copy.
 * Expression order (left to right) is part of the contract: the reference
 * oracle in oracle/ref_shim.cpp builds the SystemModel with the same lambda. */
static double chain_s(double z) { return z / (1.0 + fabs(z)); }

static double chain_d(const po_model* m, uint64_t i, const double* x, const double* p,
                      const double* xh) {
    const double a = m->params[0], b = m->params[1], c = m->params[2];
    const uint64_t n = m->dim;
    const double sl = (i == 0) ? 0.0 : chain_s(x[i - 1]);
    const double sr = (i + 1 == n) ? 0.0 : chain_s(xh[i + 1]);
    return ((-a) * x[i] + b * sl - c * sr) + p[0];
}

static double laub_loomis_rhs(uint64_t i, const double* x) {
    /* models.cpp:470-485 */
    switch (i) {
        case 0: return 1.4 * x[2] - 0.9 * x[0];
        case 1: return 2.5 * x[4] - 1.5 * x[1];
        case 2: return 0.6 * x[6] - 0.8 * x[1] * x[2];
        case 3: return 2.0 - 1.3 * x[2] * x[3];
        case 4: return 0.7 * x[0] - x[3] * x[4];
        case 5: return 0.3 * x[0] - 3.1 * x[5];
        default: return 1.8 * x[5] - 1.5 * x[1] * x[6];
    }
}

static double arch_quad_rhs(const po_model* m, uint64_t i, const double* x) {
    /* models.cpp:515-555 */
    const double mass = m->params[0], gravity = m->params[1];
    const double jx = m->params[2], jy = m->params[3], jz = m->params[4];
    const double kx = (jy - jz) / jx, ky = (jz - jx) / jy, kz = (jx - jy) / jz;
    const double s7 = sin(x[6]), c7 = cos(x[6]);
    const double s8 = sin(x[7]), c8 = cos(x[7]);
    const double s9 = sin(x[8]), c9 = cos(x[8]);
    switch (i) {
        case 0:
            return c8 * c9 * x[3] + (s7 * s8 * c9 - c7 * s9) * x[4] +
                   (c7 * s8 * c9 + s7 * s9) * x[5];
        case 1:
            return c8 * s9 * x[3] + (s7 * s8 * s9 + c7 * c9) * x[4] +
                   (c7 * s8 * s9 - s7 * c9) * x[5];
        case 2: return s8 * x[3] - s7 * c8 * x[4] - c7 * c8 * x[5];
        case 3: return x[11] * x[4] - x[10] * x[5] - gravity * s8;
        case 4: return x[9] * x[5] - x[11] * x[3] + gravity * c8 * s7;
        case 5: {
            const double thrust = mass * gravity - 10.0 * (x[2] - 1.0) + 3.0 * x[5];
            return x[10] * x[3] - x[9] * x[4] + gravity * c8 * c7 - thrust / mass;
        }
        case 6: return x[9] + s7 * (s8 / c8) * x[10] + c7 * (s8 / c8) * x[11];
        case 7: return c7 * x[10] - s7 * x[11];
        case 8: return s7 / c8 * x[10] + c7 / c8 * x[11];
        case 9: return kx * x[10] * x[11] - (x[6] + x[9]) / jx;
        case 10: return ky * x[9] * x[11] - (x[7] + x[10]) / jy;
        default: return kz * x[9] * x[10];
    }
}

static double vdp_rhs(const po_model* m, uint64_t i, const double* x) {
    /* models.cpp:452-456 */
    const double mu = m->params[0];
    if (i == 0) return x[1];
    return mu * (1.0 - x[0] * x[0]) * x[1] - x[0];
}

double po_rhs(const po_model* m, uint64_t i, double t, const double* x, const double* p) {
    (void)t;
    switch (m->kind) {
        case PO_ZERO: return 0.0;                                  /* models.cpp:621-623 */
        case PO_SCALAR_DECAY: return -x[0] + p[0];                 /* models.cpp:634-636 */
        case PO_SCALAR_LINEAR: return m->params[0] * x[0];         /* models.cpp:648-650 */
        case PO_TRAFFIC: return traffic_rhs(m, i, x, p);
        case PO_HEAT3D: return heat_rhs(m, i, x);
        case PO_CHAIN: return chain_d(m, i, x, p, x);
        case PO_LAUB_LOOMIS: return laub_loomis_rhs(i, x);
        case PO_ARCH_QUAD: return arch_quad_rhs(m, i, x);
        case PO_VDP: return vdp_rhs(m, i, x);
        default: return NAN;
    }
}

/* Dense growth matrices: models.cpp:457-460 (vdp), 488-500 (laub-loomis),
 * 557-611 (arch-quadrotor).  Row-major n x n. */
int po_growth_matrix(const po_model* m, double* C) {
    const uint64_t n = m->dim;
    memset(C, 0, sizeof(double) * n * n);
    if (m->kind == PO_VDP) {
        const double mu = m->params[0], op_x = m->params[1], op_y = m->params[2];
        C[0 * 2 + 1] = 1.0;
        C[1 * 2 + 0] = 2.0 * mu * op_x * op_y + 1.0;
        C[1 * 2 + 1] = mu;
        return 1;
    }
    if (m->kind == PO_LAUB_LOOMIS) {
        const double xm = 5.0;
        const double rows[7][7] = {
            {-0.9, 0, 1.4, 0, 0, 0, 0},     {0, -1.5, 0, 0, 2.5, 0, 0},
            {0, 0.8 * xm, 0, 0, 0, 0, 0.6}, {0, 0, 1.3 * xm, 0, 0, 0, 0},
            {0.7, 0, 0, xm, 0, 0, 0},       {0.3, 0, 0, 0, 0, -3.1, 0},
            {0, 1.5 * xm, 0, 0, 0, 1.8, 0},
        };
        memcpy(C, rows, sizeof(rows));
        return 1;
    }
    if (m->kind == PO_ARCH_QUAD) {
        const double mass = m->params[0], gravity = m->params[1];
        const double jx = m->params[2], jy = m->params[3], jz = m->params[4];
        const double kx = (jy - jz) / jx, ky = (jz - jx) / jy, kz = (jx - jy) / jz;
        const double vb = 5.0, ab = 0.5, rb = 2.0;
        const double tanb = tan(ab);
        const double secb = 1.0 / cos(ab);
        const double sec2b = secb * secb;
        const double akx = fabs(kx), aky = fabs(ky), akz = fabs(kz);
#define CC(r, c) C[(r) * 12 + (c)]
        for (int row = 0; row < 3; ++row) {
            CC(row, 3) = CC(row, 4) = CC(row, 5) = 1.0;
            CC(row, 6) = CC(row, 7) = 6.0 * vb;
            if (row < 2) CC(row, 8) = 6.0 * vb;
        }
        CC(3, 4) = rb; CC(3, 5) = rb; CC(3, 7) = gravity; CC(3, 10) = vb; CC(3, 11) = vb;
        CC(4, 3) = rb; CC(4, 5) = rb; CC(4, 6) = gravity; CC(4, 7) = gravity;
        CC(4, 9) = vb; CC(4, 11) = vb;
        CC(5, 2) = 10.0 / mass; CC(5, 3) = rb; CC(5, 4) = rb; CC(5, 5) = -3.0 / mass;
        CC(5, 6) = gravity; CC(5, 7) = gravity; CC(5, 9) = vb; CC(5, 10) = vb;
        CC(6, 6) = 2.0 * tanb * rb; CC(6, 7) = 2.0 * sec2b * rb; CC(6, 9) = 1.0;
        CC(6, 10) = tanb; CC(6, 11) = tanb;
        CC(7, 6) = 2.0 * rb; CC(7, 10) = 1.0; CC(7, 11) = 1.0;
        CC(8, 6) = 2.0 * secb * rb; CC(8, 7) = 2.0 * secb * tanb * rb;
        CC(8, 10) = secb; CC(8, 11) = secb;
        CC(9, 6) = 1.0 / jx; CC(9, 9) = -1.0 / jx; CC(9, 10) = akx * rb; CC(9, 11) = akx * rb;
        CC(10, 7) = 1.0 / jy; CC(10, 9) = aky * rb; CC(10, 10) = -1.0 / jy;
        CC(10, 11) = aky * rb;
        CC(11, 9) = akz * rb; CC(11, 10) = akz * rb;
#undef CC
        return 1;
    }
    return 0;
}

/* growth_from_matrix evaluator, system_model.cpp:107-121 (acc from 0.0, all j). */
static double dense_growth(const double* C, uint64_t n, uint64_t i, const double* r) {
    double acc = 0.0;
    for (uint64_t j = 0; j < n; ++j) acc += C[i * n + j] * r[j];
    return acc;
}

/* Small-model growth matrix cache (n <= 12). */
typedef struct {
    const po_model* m;
    double C[144];
    int has;
} po_cache;

static void cache_init(po_cache* pc, const po_model* m) {
    pc->m = m;
    pc->has = 0;
    if (m->dim <= 12) pc->has = po_growth_matrix(m, pc->C);
}

static double growth_c(const po_cache* pc, uint64_t i, double t, const double* r,
                       const double* w) {
    const po_model* m = pc->m;
    (void)t;
    switch (m->kind) {
        case PO_ZERO: return 0.0;                       /* models.cpp:624 (growth = rhs) */
        case PO_SCALAR_DECAY: return -r[0] + w[0];      /* models.cpp:637-638 */
        case PO_SCALAR_LINEAR: return m->params[0] * r[0]; /* models.cpp:651-652 */
        case PO_TRAFFIC: return traffic_growth(m, i, r, w);
        case PO_HEAT3D: return heat_rhs(m, i, r);       /* models.cpp:130 */
        default:
            if (pc->has) return dense_growth(pc->C, m->dim, i, r);
            return NAN;
    }
}

double po_growth(const po_model* m, uint64_t i, double t, const double* r, const double* w) {
    po_cache pc;
    cache_init(&pc, m);
    return growth_c(&pc, i, t, r, w);
}

static double decomp_c(const po_cache* pc, uint64_t i, double t, const double* x,
                       const double* p, const double* xh, const double* ph) {
    const po_model* m = pc->m;
    (void)ph;
    if (m->decomp == PO_DECOMP_JACOBIAN) {
        double acc = po_rhs(m, i, t, x, p);
        const uint64_t n = m->dim;
        for (uint64_t j = 0; j < n; ++j) {
            const double cij = pc->C[i * n + j];
            if (j == i || cij == 0.0) continue;
            acc = acc + cij * (x[j] - xh[j]);
        }
        return acc;
    }
    if (m->kind == PO_CHAIN) return chain_d(m, i, x, p, xh);
    /* cooperative(rhs), models.cpp:20-27 */
    return po_rhs(m, i, t, x, p);
}

double po_decomp(const po_model* m, uint64_t i, double t, const double* x, const double* p,
                 const double* xh, const double* ph) {
    po_cache pc;
    cache_init(&pc, m);
    return decomp_c(&pc, i, t, x, p, xh, ph);
}

/* ------------------------------------------------------- generic RK4 engine */

/* The three integrands the methods use: plain f (MC, GB center), the growth
 * dynamics (GB radius) and the 2n embedding (system_model.cpp:56-77). */
enum { SYS_F = 0, SYS_G = 1, SYS_EMBED = 2 };

typedef struct {
    const po_cache* pc;
    int which;
    uint64_t dim; /* integrated dimension */
} po_sys;

static double sys_eval(const po_sys* s, uint64_t i, double t, const double* x, const double* p) {
    const po_model* m = s->pc->m;
    switch (s->which) {
        case SYS_F: return po_rhs(m, i, t, x, p);
        case SYS_G: return growth_c(s->pc, i, t, x, p);
        default: {
            /* system_model.cpp:67-75 */
            const uint64_t n = m->dim, ni = m->input_dim;
            const double* xl = x;
            const double* xu = x + n;
            const double* pl = p;
            const double* pu = p + ni;
            if (i < n) return decomp_c(s->pc, i, t, xl, pl, xu, pu);
            return decomp_c(s->pc, i - n, t, xu, pu, xl, pl);
        }
    }
}

typedef void (*po_observer)(void* user, uint64_t step, double t, const double* x, uint64_t dim);

/* rk4_serial.cpp:10-61, with Rk4Engine::run's recording rule (rk4.cpp:96-111). */
static int rk4_run(const po_sys* s, const double* x0, const double* p, double t0, double t1,
                   double h, uint64_t stride, po_observer obs, void* user, double* work,
                   uint64_t* err_step, uint64_t* err_comp, double* err_t) {
    const uint64_t n = s->dim;
    const uint64_t total = plan_total(t0, t1, h);
    if (total == 0) return PO_EINVAL;
    double* x = work;
    double* k0 = x + n;
    double* k1 = k0 + n;
    double* k2 = k1 + n;
    double* k3 = k2 + n;
    double* u1 = k3 + n;
    double* u2 = u1 + n;
    memcpy(x, x0, n * sizeof(double));
    if (stride > 0 && obs) obs(user, 0, t0, x, n);
    for (uint64_t k = 0; k < total; ++k) {
        const double t = t0 + (double)k * h;                 /* rk4.cpp:99 */
        const double hk = (k + 1 == total) ? t1 - t : h;     /* rk4.cpp:100 */
        const double h2 = 0.5 * hk;
        const double h6 = hk / 6.0;
        for (uint64_t i = 0; i < n; ++i) {
            k0[i] = sys_eval(s, i, t, x, p);
            u1[i] = x[i] + h2 * k0[i];
        }
        for (uint64_t i = 0; i < n; ++i) {
            k1[i] = sys_eval(s, i, t + h2, u1, p);
            u2[i] = x[i] + h2 * k1[i];
        }
        for (uint64_t i = 0; i < n; ++i) {
            k2[i] = sys_eval(s, i, t + h2, u2, p);
            u1[i] = x[i] + hk * k2[i];
        }
        for (uint64_t i = 0; i < n; ++i) {
            k3[i] = sys_eval(s, i, t + hk, u1, p);
            x[i] = x[i] + h6 * (k0[i] + 2.0 * k1[i] + 2.0 * k2[i] + k3[i]);
        }
        /* rk4.cpp:72-75: first non-finite component of the step */
        for (uint64_t i = 0; i < n; ++i) {
            if (!isfinite(x[i])) {
                if (err_step) *err_step = k;
                if (err_comp) *err_comp = i;
                if (err_t) *err_t = t;
                return PO_EINTEGRATION;
            }
        }
        if (!obs) continue;
        if (k + 1 == total)
            obs(user, total, t1, x, n);
        else if (stride > 0 && (k + 1) % stride == 0)
            obs(user, k + 1, t0 + (double)(k + 1) * h, x, n);
    }
    return PO_OK;
}

typedef struct {
    double* states;
    double* times;
    uint64_t slot;
    uint64_t dim;
} collect_ctx;

static void collect_obs(void* user, uint64_t step, double t, const double* x, uint64_t dim) {
    (void)step;
    collect_ctx* c = (collect_ctx*)user;
    if (c->times) c->times[c->slot] = t;
    if (c->states) memcpy(c->states + c->slot * dim, x, dim * sizeof(double));
    c->slot++;
}

int po_integrate(const po_model* m, const double* x0, const double* p, double t0, double t1,
                 double h, uint64_t stride, double* times_out, double* states_out,
                 uint64_t* err_step, uint64_t* err_comp, double* err_t) {
    po_cache pc;
    cache_init(&pc, m);
    po_sys s = {&pc, SYS_F, m->dim};
    double* work = (double*)malloc(7 * m->dim * sizeof(double));
    if (!work) return PO_ENOMEM;
    collect_ctx c = {states_out, times_out, 0, m->dim};
    const int rc = rk4_run(&s, x0, p, t0, t1, h, stride, collect_obs, &c, work, err_step,
                           err_comp, err_t);
    free(work);
    return rc;
}

/* ----------------------------------------------------------------- methods */

static int validate(const po_model* m, const double* lo, const double* hi, const double* plo,
                    const double* phi, double t0, double t1, double h, char* err, int errlen) {
    /* system_model.cpp:10-32 + IntervalVector ctor, interval.cpp:10-23 */
    if (m->dim == 0) {
        snprintf(err, errlen, "problem: model has no dynamics");
        return PO_EINVAL;
    }
    for (uint64_t i = 0; i < m->dim; ++i) {
        if (!isfinite(lo[i]) || !isfinite(hi[i]) || lo[i] > hi[i]) {
            snprintf(err, errlen, "interval: invalid bound at component %llu",
                     (unsigned long long)i);
            return PO_EINVAL;
        }
    }
    for (uint64_t j = 0; j < m->input_dim; ++j) {
        if (!plo || !phi || !isfinite(plo[j]) || !isfinite(phi[j]) || plo[j] > phi[j]) {
            snprintf(err, errlen, "problem: invalid input box");
            return PO_EINVAL;
        }
    }
    if (!(t0 < t1)) {
        snprintf(err, errlen, "problem: t0 must be earlier than t1");
        return PO_EINVAL;
    }
    if (!(h > 0.0)) {
        snprintf(err, errlen, "problem: step size h must be positive");
        return PO_EINVAL;
    }
    return PO_OK;
}

typedef struct {
    uint64_t n;
    double* times;
    double* out_lo;
    double* out_hi;
    uint64_t slot;
    int failed;
    uint64_t fail_step;
    double fail_t;
    uint64_t fail_comp;
} mm_ctx;

static void mm_obs(void* user, uint64_t step, double t, const double* xx, uint64_t dim) {
    /* reach.cpp:177-189: split, order check, box */
    (void)dim;
    mm_ctx* c = (mm_ctx*)user;
    if (c->failed) return;
    const uint64_t n = c->n;
    for (uint64_t i = 0; i < n; ++i) {
        if (xx[i] > xx[n + i]) {
            c->failed = 1;
            c->fail_step = step;
            c->fail_t = t;
            c->fail_comp = i;
            return;
        }
    }
    c->times[c->slot] = t;
    memcpy(c->out_lo + c->slot * n, xx, n * sizeof(double));
    memcpy(c->out_hi + c->slot * n, xx + n, n * sizeof(double));
    c->slot++;
}

/* Order-checking observer aborts via this wrapper: the reference throws from
 * inside the observer (reach.cpp:181-186), which ends the integration. */
static int rk4_run_mm(const po_sys* s, const double* x0, const double* p, double t0, double t1,
                      double h, uint64_t stride, mm_ctx* c, double* work, uint64_t* es,
                      uint64_t* ec, double* et) {
    /* Same loop as rk4_run, stopping after a failed observation. */
    const uint64_t n = s->dim;
    const uint64_t total = plan_total(t0, t1, h);
    double* x = work;
    double* k0 = x + n;
    double* k1 = k0 + n;
    double* k2 = k1 + n;
    double* k3 = k2 + n;
    double* u1 = k3 + n;
    double* u2 = u1 + n;
    memcpy(x, x0, n * sizeof(double));
    if (stride > 0) {
        mm_obs(c, 0, t0, x, n);
        if (c->failed) return PO_EORDER;
    }
    for (uint64_t k = 0; k < total; ++k) {
        const double t = t0 + (double)k * h;
        const double hk = (k + 1 == total) ? t1 - t : h;
        const double h2 = 0.5 * hk;
        const double h6 = hk / 6.0;
        for (uint64_t i = 0; i < n; ++i) {
            k0[i] = sys_eval(s, i, t, x, p);
            u1[i] = x[i] + h2 * k0[i];
        }
        for (uint64_t i = 0; i < n; ++i) {
            k1[i] = sys_eval(s, i, t + h2, u1, p);
            u2[i] = x[i] + h2 * k1[i];
        }
        for (uint64_t i = 0; i < n; ++i) {
            k2[i] = sys_eval(s, i, t + h2, u2, p);
            u1[i] = x[i] + hk * k2[i];
        }
        for (uint64_t i = 0; i < n; ++i) {
            k3[i] = sys_eval(s, i, t + hk, u1, p);
            x[i] = x[i] + h6 * (k0[i] + 2.0 * k1[i] + 2.0 * k2[i] + k3[i]);
        }
        for (uint64_t i = 0; i < n; ++i) {
            if (!isfinite(x[i])) {
                *es = k;
                *ec = i;
                *et = t;
                return PO_EINTEGRATION;
            }
        }
        if (k + 1 == total)
            mm_obs(c, total, t1, x, n);
        else if (stride > 0 && (k + 1) % stride == 0)
            mm_obs(c, k + 1, t0 + (double)(k + 1) * h, x, n);
        if (c->failed) return PO_EORDER;
    }
    return PO_OK;
}

int po_mixed_monotonicity(const po_model* m, const double* lo, const double* hi,
                          const double* plo, const double* phi, double t0, double t1,
                          double h, uint64_t stride, double* times, double* out_lo,
                          double* out_hi, char* err, int errlen) {
    /* reach.cpp:139-196 */
    int rc = validate(m, lo, hi, plo, phi, t0, t1, h, err, errlen);
    if (rc) return rc;
    if (m->decomp == PO_DECOMP_NONE) {
        snprintf(err, errlen, "mixed_monotonicity: model has no decomposition function");
        return PO_EINVAL;
    }
    const uint64_t n = m->dim, ni = m->input_dim;
    po_cache pc;
    cache_init(&pc, m);
    po_sys s = {&pc, SYS_EMBED, 2 * n};
    double* x0 = (double*)malloc(2 * n * sizeof(double));
    double* p = (double*)malloc((2 * ni + 1) * sizeof(double));
    double* work = (double*)malloc(7 * 2 * n * sizeof(double));
    if (!x0 || !p || !work) {
        free(x0); free(p); free(work);
        return PO_ENOMEM;
    }
    for (uint64_t i = 0; i < n; ++i) { /* reach.cpp:150-155 */
        x0[i] = lo[i];
        x0[n + i] = hi[i];
    }
    for (uint64_t j = 0; j < ni; ++j) { /* reach.cpp:156-161 */
        p[j] = plo[j];
        p[ni + j] = phi[j];
    }
    mm_ctx c = {n, times, out_lo, out_hi, 0, 0, 0, 0.0, 0};
    uint64_t es = 0, ec = 0;
    double et = 0.0;
    rc = rk4_run_mm(&s, x0, p, t0, t1, h, stride, &c, work, &es, &ec, &et);
    if (rc == PO_EORDER) {
        snprintf(err, errlen,
                 "mixed-monotonicity: embedding order violated at step %llu, t = %f, "
                 "component %llu",
                 (unsigned long long)c.fail_step, c.fail_t, (unsigned long long)c.fail_comp);
    } else if (rc == PO_EINTEGRATION) {
        snprintf(err, errlen,
                 "mixed-monotonicity embedding integration: integration produced a "
                 "non-finite value at step %llu, component %llu, t = %f",
                 (unsigned long long)es, (unsigned long long)ec, et);
    }
    free(x0); free(p); free(work);
    return rc;
}

int po_growth_bound(const po_model* m, const double* lo, const double* hi,
                    const double* plo, const double* phi, double t0, double t1, double h,
                    uint64_t stride, double* times, double* out_lo, double* out_hi,
                    char* err, int errlen) {
    /* reach.cpp:65-137 */
    int rc = validate(m, lo, hi, plo, phi, t0, t1, h, err, errlen);
    if (rc) return rc;
    const uint64_t n = m->dim, ni = m->input_dim;
    po_cache pc;
    cache_init(&pc, m);
    const int has_growth = m->kind <= PO_HEAT3D || pc.has;
    if (!has_growth) {
        snprintf(err, errlen, "growth_bound: model has no deviation dynamics");
        return PO_EINVAL;
    }
    const uint64_t slots = po_record_schedule(t0, t1, h, stride, NULL, times);
    double* c0 = (double*)malloc(n * sizeof(double));
    double* r0 = (double*)malloc(n * sizeof(double));
    double* pc_ = (double*)malloc((ni + 1) * sizeof(double));
    double* w = (double*)malloc((ni + 1) * sizeof(double));
    double* work = (double*)malloc(7 * n * sizeof(double));
    double* centers = (double*)malloc(slots * n * sizeof(double));
    double* radii = (double*)malloc(slots * n * sizeof(double));
    for (uint64_t i = 0; i < n; ++i) { /* interval.cpp:25-37 */
        c0[i] = 0.5 * (hi[i] + lo[i]);
        r0[i] = 0.5 * (hi[i] - lo[i]);
    }
    for (uint64_t j = 0; j < ni; ++j) {
        pc_[j] = 0.5 * (phi[j] + plo[j]);
        w[j] = 0.5 * (phi[j] - plo[j]);
    }
    uint64_t es = 0, ec = 0;
    double et = 0.0;
    po_sys sf = {&pc, SYS_F, n};
    collect_ctx cc = {centers, NULL, 0, n};
    rc = rk4_run(&sf, c0, pc_, t0, t1, h, stride, collect_obs, &cc, work, &es, &ec, &et);
    if (rc == PO_EINTEGRATION) {
        snprintf(err, errlen,
                 "growth-bound center integration: integration produced a non-finite value "
                 "at step %llu, component %llu, t = %f",
                 (unsigned long long)es, (unsigned long long)ec, et);
    } else if (rc == PO_OK) {
        po_sys sg = {&pc, SYS_G, n};
        collect_ctx cr = {radii, NULL, 0, n};
        rc = rk4_run(&sg, r0, w, t0, t1, h, stride, collect_obs, &cr, work, &es, &ec, &et);
        if (rc == PO_EINTEGRATION)
            snprintf(err, errlen,
                     "growth-bound radius integration: integration produced a non-finite "
                     "value at step %llu, component %llu, t = %f",
                     (unsigned long long)es, (unsigned long long)ec, et);
    }
    if (rc == PO_OK) {
        for (uint64_t s = 0; s < slots && rc == PO_OK; ++s) { /* reach.cpp:121-134 */
            double* r = radii + s * n;
            const double* c = centers + s * n;
            for (uint64_t i = 0; i < n; ++i) {
                if (r[i] < 0.0) {
                    if (r[i] < -1e-12) {
                        snprintf(err, errlen,
                                 "growth-bound: deviation went negative (%f) at component "
                                 "%llu; contraction matrix is invalid",
                                 r[i], (unsigned long long)i);
                        rc = PO_ENEGRADIUS;
                        break;
                    }
                    r[i] = 0.0;
                }
                out_lo[s * n + i] = c[i] - r[i]; /* interval.cpp:49-50 */
                out_hi[s * n + i] = c[i] + r[i];
            }
        }
    }
    free(c0); free(r0); free(pc_); free(w); free(work); free(centers); free(radii);
    return rc;
}

typedef struct {
    double* out_lo;
    double* out_hi;
    uint64_t slot;
    uint64_t n;
} hull_ctx;

static void hull_obs(void* user, uint64_t step, double t, const double* x, uint64_t dim) {
    /* HullAccumulator::fold, reach.cpp:222-230 */
    (void)step; (void)t;
    hull_ctx* h = (hull_ctx*)user;
    double* lo = h->out_lo + h->slot * dim;
    double* hi = h->out_hi + h->slot * dim;
    for (uint64_t i = 0; i < dim; ++i) {
        if (x[i] < lo[i]) lo[i] = x[i];
        if (x[i] > hi[i]) hi[i] = x[i];
    }
    h->slot++;
}

static void draw_sample(const po_model* m, const double* lo, const double* hi,
                        const double* plo, const double* phi, uint64_t seed, uint64_t s,
                        double* x0, double* p) {
    /* reach.cpp:202-212 */
    const uint64_t n = m->dim;
    for (uint64_t i = 0; i < n; ++i) x0[i] = po_uniform_in(lo[i], hi[i], po_u01(seed, s, i));
    for (uint64_t j = 0; j < m->input_dim; ++j)
        p[j] = po_uniform_in(plo[j], phi[j], po_u01(seed, s, n + j));
}

int po_monte_carlo(const po_model* m, const double* lo, const double* hi, const double* plo,
                   const double* phi, double t0, double t1, double h, uint64_t stride,
                   uint64_t seed, uint64_t s_begin, uint64_t s_end, double* times,
                   double* out_lo, double* out_hi, char* err, int errlen) {
    /* reach.cpp:246-323 (sample loop restricted to [s_begin, s_end)) */
    int rc = validate(m, lo, hi, plo, phi, t0, t1, h, err, errlen);
    if (rc) return rc;
    const uint64_t n = m->dim;
    po_record_schedule(t0, t1, h, stride, NULL, times);
    po_cache pc;
    cache_init(&pc, m);
    po_sys s = {&pc, SYS_F, n};
    double* x0 = (double*)malloc(n * sizeof(double));
    double* p = (double*)malloc((m->input_dim + 1) * sizeof(double));
    double* work = (double*)malloc(7 * n * sizeof(double));
    for (uint64_t smp = s_begin; smp < s_end; ++smp) {
        draw_sample(m, lo, hi, plo, phi, seed, smp, x0, p);
        hull_ctx hc = {out_lo, out_hi, 0, n};
        uint64_t es = 0, ec = 0;
        double et = 0.0;
        rc = rk4_run(&s, x0, p, t0, t1, h, stride, hull_obs, &hc, work, &es, &ec, &et);
        if (rc == PO_EINTEGRATION) {
            snprintf(err, errlen,
                     "monte-carlo sample %llu integration: integration produced a non-finite "
                     "value at step %llu, component %llu, t = %f",
                     (unsigned long long)smp, (unsigned long long)es, (unsigned long long)ec,
                     et);
            break;
        }
    }
    free(x0); free(p); free(work);
    return rc;
}

int po_coverage_estimate(const po_model* m, const double* lo, const double* hi,
                         const double* plo, const double* phi, double t0, double t1,
                         double h, const double* box_lo, const double* box_hi,
                         uint64_t fresh, uint64_t seed, double* fraction) {
    /* reach.cpp:325-358 */
    const uint64_t n = m->dim;
    po_cache pc;
    cache_init(&pc, m);
    po_sys s = {&pc, SYS_F, n};
    double* x0 = (double*)malloc(n * sizeof(double));
    double* p = (double*)malloc((m->input_dim + 1) * sizeof(double));
    double* work = (double*)malloc(7 * n * sizeof(double));
    double* xf = (double*)malloc(n * sizeof(double));
    uint64_t outside = 0;
    int rc = PO_OK;
    for (uint64_t smp = 0; smp < fresh; ++smp) {
        draw_sample(m, lo, hi, plo, phi, seed, smp, x0, p);
        collect_ctx c = {xf, NULL, 0, n};
        rc = rk4_run(&s, x0, p, t0, t1, h, 0, collect_obs, &c, work, NULL, NULL, NULL);
        if (rc) break;
        for (uint64_t i = 0; i < n; ++i) { /* interval.cpp:55-62 */
            if (xf[i] < box_lo[i] || xf[i] > box_hi[i]) {
                ++outside;
                break;
            }
        }
    }
    *fraction = (double)outside / (double)fresh;
    free(x0); free(p); free(work); free(xf);
    return rc;
}

/* -------------------------------------------------- windowed step (sharding) */

int po_step_window(const po_model* m, int method, const double* in0, const double* in1,
                   double* out0, double* out1, uint64_t win_begin, uint64_t win_len,
                   uint64_t out_begin, uint64_t out_end, const double* p0, const double* p1,
                   double t, double hk) {
    /* integrate_step (rk4.cpp:30-76) of the 2-field system, evaluated on a
     * global-size scratch whose non-window entries are NaN so that any read
     * outside the window poisons the result (and the bit-exact comparison). */
    const uint64_t n = m->dim;
    const uint64_t unit = (m->kind == PO_HEAT3D) ? m->grid * m->grid : 1; /* comps per unit */
    const uint64_t units = n / unit;
    if (win_begin + win_len > units || out_begin < win_begin ||
        out_end > win_begin + win_len || out_begin > out_end)
        return PO_EINVAL;
    const uint64_t N = 2 * n, ni = m->input_dim;
    double* buf = (double*)malloc(7 * N * sizeof(double));
    double* p = (double*)malloc((2 * ni + 1) * sizeof(double));
    if (!buf || !p) {
        free(buf); free(p);
        return PO_ENOMEM;
    }
    double* x = buf;
    double *k0 = x + N, *k1 = k0 + N, *k2 = k1 + N, *k3 = k2 + N, *u1 = k3 + N, *u2 = u1 + N;
    for (uint64_t i = 0; i < 7 * N; ++i) buf[i] = NAN;
    const uint64_t c0 = win_begin * unit, c1 = (win_begin + win_len) * unit;
    memcpy(x + c0, in0, (c1 - c0) * sizeof(double));
    memcpy(x + n + c0, in1, (c1 - c0) * sizeof(double));
    for (uint64_t j = 0; j < ni; ++j) {
        p[j] = p0 ? p0[j] : 0.0;
        p[ni + j] = p1 ? p1[j] : 0.0;
    }
    po_cache pc;
    cache_init(&pc, m);
    /* Per-field evaluators.  method 0: embedding (system_model.cpp:67-75);
     * method 1: growth bound, field 0 = center under f(.,pc), field 1 = radius
     * under g(.,w) (reach.cpp:103-114). */
    const double h2 = 0.5 * hk, h6 = hk / 6.0;
    /* stage s valid range in units: shrink by s+1 at window edges that are
     * not global boundaries */
    for (int stage = 0; stage < 4; ++stage) {
        const uint64_t shrink = (uint64_t)stage + 1;
        uint64_t a = win_begin, b = win_begin + win_len;
        if (a > 0) a += shrink;
        if (b < units) b = (b >= shrink) ? b - shrink : 0;
        if (stage == 3) {
            a = out_begin;
            b = out_end;
        }
        const double* src = (stage == 0) ? x : (stage == 2) ? u2 : u1;
        double* kdst = (stage == 0) ? k0 : (stage == 1) ? k1 : (stage == 2) ? k2 : k3;
        const double tt = (stage == 0) ? t : (stage == 3) ? t + hk : t + h2;
        for (uint64_t i = a * unit; i < b * unit; ++i) {
            for (int f = 0; f < 2; ++f) {
                const uint64_t gi = (uint64_t)f * n + i;
                double kv;
                if (method == 0) {
                    kv = (f == 0) ? decomp_c(&pc, i, tt, src, p, src + n, p + ni)
                                  : decomp_c(&pc, i, tt, src + n, p + ni, src, p);
                } else {
                    kv = (f == 0) ? po_rhs(m, i, tt, src, p) : growth_c(&pc, i, tt, src + n, p + ni);
                }
                kdst[gi] = kv;
            }
        }
        /* stage updates, written after all evaluations of the stage */
        for (uint64_t i = a * unit; i < b * unit; ++i) {
            for (int f = 0; f < 2; ++f) {
                const uint64_t gi = (uint64_t)f * n + i;
                if (stage == 0) u1[gi] = x[gi] + h2 * k0[gi];
                else if (stage == 1) u2[gi] = x[gi] + h2 * k1[gi];
                else if (stage == 2) u1[gi] = x[gi] + hk * k2[gi];
            }
        }
        if (stage == 2) {
            /* the final stage reads u1 over its (narrower) range only; the
             * u1 entries outside stage 2's range still hold stage-0 values,
             * poison them to keep the window discipline honest */
            for (uint64_t i = 0; i < a * unit; ++i) { u1[i] = NAN; u1[n + i] = NAN; }
            for (uint64_t i = b * unit; i < n; ++i) { u1[i] = NAN; u1[n + i] = NAN; }
        }
    }
    for (uint64_t i = out_begin * unit; i < out_end * unit; ++i) {
        for (int f = 0; f < 2; ++f) {
            const uint64_t gi = (uint64_t)f * n + i;
            const double v = x[gi] + h6 * (k0[gi] + 2.0 * k1[gi] + 2.0 * k2[gi] + k3[gi]);
            double* o = (f == 0) ? out0 : out1;
            o[i - out_begin * unit] = v;
        }
    }
    free(buf);
    free(p);
    return PO_OK;
}
