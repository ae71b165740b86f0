/*
 * pwadv_oracle.c — CPU restatement of the reference PW-advection hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This file is the parity checker for the CUDA
 * path and the timed CPU baseline of bench.py; nothing in the product
 * (paper_2010_01545_b200/) links, loads or calls it. Only tests/,
 * __graft_entry__.smoke() and bench.py (cpu_baseline leg, --impl reference)
 * may use it.
 *
 * What it restates (reference = /root/reference, pwadvect 0.1.0):
 *   - su/sv/sw formulas           pkg/src/pwadvect/kernel.py:73-112
 *   - operand wiring              pkg/src/pwadvect/kernel.py:117-128
 *   - level-0 zero / top branch   pkg/src/pwadvect/kernel.py:146-161
 *   - run_reference scatter       pkg/src/pwadvect/kernel.py:175-185
 *   - X-slab engines              pkg/src/pwadvect/schedules.py:65-75, 207-232
 *   - wrap_halos (X then Y)       pkg/src/pwadvect/grid.py:203-208
 *   - Knuth MMIX LCG + skip-ahead pkg/src/pwadvect/grid.py:21-23, 164-200
 *   - random fill (u,v,w stream)  pkg/src/pwadvect/grid.py:223-239
 *
 * Arithmetic contract: every +, -, * is one IEEE-754 binary64 round-to-
 * nearest operation with the reference's association (Python evaluates
 * a*b*(c+d) as (a*b)*(c+d)). Build with -ffp-contract=off and without
 * -ffast-math so no FMA contraction or reassociation happens.
 *
 * Parity pin: checked bit-for-bit against the reference's goldens.json
 * digests and against fixtures produced by importing the reference
 * (tests/golden/make_golden.py) — see tests/test_oracle.py.
 */
#include <stdint.h>
#include <stddef.h>
#include <string.h>
#include <pthread.h>

#define ORACLE_LCG_MULT 6364136223846793005ULL
#define ORACLE_LCG_INC 1442695040888963407ULL

int oracle_version(void) { return 1; }

/* Padded (nx+2, ny+2, nz) C-order, k fastest: grid.py:61-64. */
#define IX(i, j, k) ((((size_t)(i)) * (size_t)(ny + 2) + (size_t)(j)) * (size_t)nz + (size_t)(k))

/*
 * One X slab [x_begin, x_end) of interior columns (1-based i), full Y range.
 * Writes levels 0..nz-1 of each interior column (level 0 = +0.0, exactly as
 * compute_block's zeros_like leaves it, kernel.py:151). Halo columns of the
 * outputs are not touched (caller provides zeroed outputs, as zeros_sources).
 */
void oracle_advect_slab(const double *u, const double *v, const double *w,
                        double *su, double *sv, double *sw,
                        int64_t nx, int64_t ny, int64_t nz,
                        double tcx, double tcy,
                        const double *tzc1, const double *tzc2,
                        int64_t x_begin, int64_t x_end)
{
    (void)nx;
    for (int64_t i = x_begin; i < x_end; ++i) {
        for (int64_t j = 1; j <= ny; ++j) {
            su[IX(i, j, 0)] = 0.0;
            sv[IX(i, j, 0)] = 0.0;
            sw[IX(i, j, 0)] = 0.0;
            for (int64_t k = 1; k < nz; ++k) {
                const int top = (k == nz - 1);
                double s, x, y, a, b;
                /* su: kernel.py:73-84, operands kernel.py:117-120 */
                x = tcx * (u[IX(i - 1, j, k)] * (u[IX(i, j, k)] + u[IX(i - 1, j, k)])
                           - u[IX(i + 1, j, k)] * (u[IX(i, j, k)] + u[IX(i + 1, j, k)]));
                y = tcy * (u[IX(i, j - 1, k)] * (v[IX(i, j - 1, k)] + v[IX(i + 1, j - 1, k)])
                           - u[IX(i, j + 1, k)] * (v[IX(i, j, k)] + v[IX(i + 1, j, k)]));
                s = x + y;
                a = (tzc1[k] * u[IX(i, j, k - 1)]) * (w[IX(i, j, k - 1)] + w[IX(i + 1, j, k - 1)]);
                if (top) {
                    s = s + a;
                } else {
                    b = (tzc2[k] * u[IX(i, j, k + 1)]) * (w[IX(i, j, k)] + w[IX(i + 1, j, k)]);
                    s = s + (a - b);
                }
                su[IX(i, j, k)] = s;

                /* sv: kernel.py:87-98, operands kernel.py:121-124 */
                x = tcx * (v[IX(i - 1, j, k)] * (u[IX(i - 1, j, k)] + u[IX(i - 1, j + 1, k)])
                           - v[IX(i + 1, j, k)] * (u[IX(i, j, k)] + u[IX(i, j + 1, k)]));
                y = tcy * (v[IX(i, j - 1, k)] * (v[IX(i, j, k)] + v[IX(i, j - 1, k)])
                           - v[IX(i, j + 1, k)] * (v[IX(i, j, k)] + v[IX(i, j + 1, k)]));
                s = x + y;
                a = (tzc1[k] * v[IX(i, j, k - 1)]) * (w[IX(i, j, k - 1)] + w[IX(i, j + 1, k - 1)]);
                if (top) {
                    s = s + a;
                } else {
                    b = (tzc2[k] * v[IX(i, j, k + 1)]) * (w[IX(i, j, k)] + w[IX(i, j + 1, k)]);
                    s = s + (a - b);
                }
                sv[IX(i, j, k)] = s;

                /* sw: kernel.py:101-112, operands kernel.py:125-128 */
                x = tcx * (w[IX(i - 1, j, k)] * (u[IX(i - 1, j, k - 1)] + u[IX(i - 1, j, k)])
                           - w[IX(i + 1, j, k)] * (u[IX(i, j, k - 1)] + u[IX(i, j, k)]));
                y = tcy * (w[IX(i, j - 1, k)] * (v[IX(i, j - 1, k - 1)] + v[IX(i, j - 1, k)])
                           - w[IX(i, j + 1, k)] * (v[IX(i, j, k - 1)] + v[IX(i, j, k)]));
                s = x + y;
                a = (tzc1[k] * w[IX(i, j, k - 1)]) * (w[IX(i, j, k)] + w[IX(i, j, k - 1)]);
                if (top) {
                    s = s + a;
                } else {
                    b = (tzc2[k] * w[IX(i, j, k + 1)]) * (w[IX(i, j, k)] + w[IX(i, j, k + 1)]);
                    s = s + (a - b);
                }
                sw[IX(i, j, k)] = s;
            }
        }
    }
}

typedef struct {
    const double *u, *v, *w;
    double *su, *sv, *sw;
    int64_t nx, ny, nz;
    double tcx, tcy;
    const double *tzc1, *tzc2;
    int64_t x_begin, x_end;
} slab_job;

static void *slab_worker(void *p)
{
    slab_job *j = (slab_job *)p;
    oracle_advect_slab(j->u, j->v, j->w, j->su, j->sv, j->sw, j->nx, j->ny, j->nz,
                       j->tcx, j->tcy, j->tzc1, j->tzc2, j->x_begin, j->x_end);
    return NULL;
}

/*
 * Whole-grid evaluation on `engines` host threads over balanced X slabs
 * (partition_domain, schedules.py:65-75: widths differ by <= 1, wider first).
 * Output is independent of the thread count (each slab is disjoint).
 * Returns 0, or -1 for bad arguments.
 */
int oracle_advect(const double *u, const double *v, const double *w,
                  double *su, double *sv, double *sw,
                  int64_t nx, int64_t ny, int64_t nz,
                  double tcx, double tcy, const double *tzc1, const double *tzc2,
                  int engines)
{
    if (nx < 1 || ny < 1 || nz < 2) return -1;
    if (engines < 1) engines = 1;
    if (engines > nx) engines = (int)nx;
    if (engines > 1024) engines = 1024;
    if (engines == 1) {
        oracle_advect_slab(u, v, w, su, sv, sw, nx, ny, nz, tcx, tcy, tzc1, tzc2, 1, nx + 1);
        return 0;
    }
    pthread_t tid[1024];
    slab_job jobs[1024];
    int64_t base = nx / engines, rem = nx % engines, x = 1;
    for (int e = 0; e < engines; ++e) {
        int64_t width = base + (e < rem ? 1 : 0);
        slab_job jb = {u, v, w, su, sv, sw, nx, ny, nz, tcx, tcy, tzc1, tzc2, x, x + width};
        jobs[e] = jb;
        x += width;
    }
    int joined[1024];
    for (int e = 0; e < engines; ++e) {
        joined[e] = pthread_create(&tid[e], NULL, slab_worker, &jobs[e]) == 0;
        if (!joined[e]) slab_worker(&jobs[e]);
    }
    for (int e = 0; e < engines; ++e)
        if (joined[e]) pthread_join(tid[e], NULL);
    return 0;
}

/* Periodic wrap, X first then Y over all i (grid.py:203-208). */
void oracle_wrap_halos(double *f, int64_t nx, int64_t ny, int64_t nz)
{
    size_t plane = (size_t)(ny + 2) * (size_t)nz;
    memcpy(f + 0 * plane, f + (size_t)nx * plane, plane * sizeof(double));
    memcpy(f + (size_t)(nx + 1) * plane, f + 1 * plane, plane * sizeof(double));
    for (int64_t i = 0; i < nx + 2; ++i) {
        memcpy(f + IX(i, 0, 0), f + IX(i, ny, 0), (size_t)nz * sizeof(double));
        memcpy(f + IX(i, ny + 1, 0), f + IX(i, 1, 0), (size_t)nz * sizeof(double));
    }
}

/* (A, C) such that state_{n+steps} = A*state_n + C (mod 2^64), grid.py:172-181. */
static void lcg_jump(uint64_t steps, uint64_t *a_out, uint64_t *c_out)
{
    uint64_t a_s = 1, c_s = 0, a_step = ORACLE_LCG_MULT, c_step = ORACLE_LCG_INC;
    while (steps) {
        if (steps & 1) {
            a_s = a_s * a_step;
            c_s = c_s * a_step + c_step;
        }
        c_step = c_step * a_step + c_step;
        a_step = a_step * a_step;
        steps >>= 1;
    }
    *a_out = a_s;
    *c_out = c_s;
}

/*
 * Values start..start+count-1 of lcg_doubles(seed, .) (grid.py:164-200):
 * value n = (state_{n+1} >> 11) * 2^-53 with state_0 = seed.
 */
void oracle_lcg_doubles(uint64_t seed, uint64_t start, int64_t count, double *out)
{
    uint64_t a, c;
    lcg_jump(start, &a, &c);
    uint64_t s = a * seed + c;
    for (int64_t n = 0; n < count; ++n) {
        s = s * ORACLE_LCG_MULT + ORACLE_LCG_INC;
        out[n] = (double)(s >> 11) * 0x1.0p-53;
    }
}

/*
 * fill_fields(dims, GeneratorSpec.random(seed)) (grid.py:223-239), plus the
 * BASELINE.json value mapping when `baseline` != 0:
 * x -> x*20.0 - 10.0 (mul then sub, no FMA) and w = 0 at levels 0 and nz-1,
 * applied to the interior before the periodic wrap.
 */
void oracle_fill_random(double *u, double *v, double *w,
                        int64_t nx, int64_t ny, int64_t nz, uint64_t seed, int baseline)
{
    double *f[3] = {u, v, w};
    uint64_t cells = (uint64_t)nx * (uint64_t)ny * (uint64_t)nz;
    for (int n = 0; n < 3; ++n) {
        uint64_t a, c;
        lcg_jump((uint64_t)n * cells, &a, &c);
        uint64_t s = a * seed + c;
        for (int64_t i = 1; i <= nx; ++i)
            for (int64_t j = 1; j <= ny; ++j)
                for (int64_t k = 0; k < nz; ++k) {
                    s = s * ORACLE_LCG_MULT + ORACLE_LCG_INC;
                    double d = (double)(s >> 11) * 0x1.0p-53;
                    if (baseline) {
                        d = d * 20.0 - 10.0;
                        if (n == 2 && (k == 0 || k == nz - 1)) d = 0.0;
                    }
                    f[n][IX(i, j, k)] = d;
                }
        oracle_wrap_halos(f[n], nx, ny, nz);
    }
}

/*
 * BASELINE coefficients: t = lcg_doubles(seed+1, 4*nz);
 * tzc1 = 1e-3 + 4e-3*t[0:nz], tzc2 = 1e-3 + 4e-3*t[nz:2nz],
 * tzd1/tzd2 from t[2nz:4nz] (recorded, unused by the formulas).
 */
void oracle_baseline_coefficients(uint64_t seed, int64_t nz, double *tzc1, double *tzc2,
                                  double *tzd1, double *tzd2)
{
    double *dst[4] = {tzc1, tzc2, tzd1, tzd2};
    uint64_t s = seed + 1;
    for (int m = 0; m < 4; ++m)
        for (int64_t k = 0; k < nz; ++k) {
            s = s * ORACLE_LCG_MULT + ORACLE_LCG_INC;
            double t = (double)(s >> 11) * 0x1.0p-53;
            if (dst[m]) dst[m][k] = 1e-3 + 4e-3 * t;
        }
}

/*
 * A box of the same fill (light-cone checks): box cell
 * (a, b, k), a in [0, bnx), b in [0, bny), holds global padded cell
 * (i0 + a, j0 + b, k) of a gnx x gny x nz fill. Global coordinates are taken
 * periodically at any distance (the wrap of grid.py:203-208), so a box may
 * straddle the domain edge or be larger than the domain. Each column jumps
 * the LCG to its own offset, so the cost is that of the box, not the grid.
 */
void oracle_fill_box(double *u, double *v, double *w, int64_t gnx, int64_t gny, int64_t nz,
                     uint64_t seed, int baseline, int64_t i0, int64_t j0,
                     int64_t bnx, int64_t bny)
{
    double *f[3] = {u, v, w};
    uint64_t cells = (uint64_t)gnx * (uint64_t)gny * (uint64_t)nz;
    for (int n = 0; n < 3; ++n)
        for (int64_t a = 0; a < bnx; ++a) {
            int64_t gi = ((i0 + a - 1) % gnx + gnx) % gnx;      /* 0-based interior row */
            for (int64_t b = 0; b < bny; ++b) {
                int64_t gj = ((j0 + b - 1) % gny + gny) % gny;
                uint64_t first = (uint64_t)n * cells +
                                 ((uint64_t)gi * (uint64_t)gny + (uint64_t)gj) * (uint64_t)nz;
                uint64_t ja, jc;
                lcg_jump(first, &ja, &jc);
                uint64_t s = ja * seed + jc;
                double *col = f[n] + ((size_t)a * (size_t)bny + (size_t)b) * (size_t)nz;
                for (int64_t k = 0; k < nz; ++k) {
                    s = s * ORACLE_LCG_MULT + ORACLE_LCG_INC;
                    double d = (double)(s >> 11) * 0x1.0p-53;
                    if (baseline) {
                        d = d * 20.0 - 10.0;
                        if (n == 2 && (k == 0 || k == nz - 1)) d = 0.0;
                    }
                    col[k] = d;
                }
            }
        }
}

/*
 * Composed time-step oracle (the reference has no time
 * integration): f <- f + dt*s on every interior cell (mul then
 * add), then wrap_halos. `scratch` holds 3 padded fields for su/sv/sw.
 * With wrap == 0 the halo ring is left as it is (an open box whose valid
 * region shrinks by one cell per side per step: the light-cone check).
 */
static int step_impl(double *u, double *v, double *w, double *scratch,
                     int64_t nx, int64_t ny, int64_t nz, double tcx, double tcy,
                     const double *tzc1, const double *tzc2, double dt, int engines, int wrap)
{
    size_t n = (size_t)(nx + 2) * (size_t)(ny + 2) * (size_t)nz;
    double *su = scratch, *sv = scratch + n, *sw = scratch + 2 * n;
    memset(scratch, 0, 3 * n * sizeof(double));
    int rc = oracle_advect(u, v, w, su, sv, sw, nx, ny, nz, tcx, tcy, tzc1, tzc2, engines);
    if (rc) return rc;
    double *f[3] = {u, v, w};
    double *s[3] = {su, sv, sw};
    for (int m = 0; m < 3; ++m) {
        for (int64_t i = 1; i <= nx; ++i)
            for (int64_t j = 1; j <= ny; ++j)
                for (int64_t k = 0; k < nz; ++k) {
                    f[m][IX(i, j, k)] = f[m][IX(i, j, k)] + dt * s[m][IX(i, j, k)];
                }
        if (wrap) oracle_wrap_halos(f[m], nx, ny, nz);
    }
    return 0;
}

int oracle_step(double *u, double *v, double *w, double *scratch,
                int64_t nx, int64_t ny, int64_t nz, double tcx, double tcy,
                const double *tzc1, const double *tzc2, double dt, int engines)
{
    return step_impl(u, v, w, scratch, nx, ny, nz, tcx, tcy, tzc1, tzc2, dt, engines, 1);
}

int oracle_step_open(double *u, double *v, double *w, double *scratch,
                     int64_t nx, int64_t ny, int64_t nz, double tcx, double tcy,
                     const double *tzc1, const double *tzc2, double dt, int engines)
{
    return step_impl(u, v, w, scratch, nx, ny, nz, tcx, tcy, tzc1, tzc2, dt, engines, 0);
}
