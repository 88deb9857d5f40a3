/* TEST INFRASTRUCTURE ONLY -- plain-C fp64 restatement of the reference hot path.
 * See snls_oracle.h for the contract.  Built with -ffp-contract=off and the reference's
 * operation order so results are bit-identical to the reference (checked by
 * tests/test_oracle.py against oracle/_ref/libsnls_ref.so and tests/golden/).
 * Citations are /root/reference/proj/<file>:<line>. */
#include "snls_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* oracle_last_error(void) { return g_err; }

/* ---- rng.hpp:12-24: UniformStream over std::mt19937_64 (parameters pinned by the C++
 * standard, [rand.predef]) ---------------------------------------------------------- */
typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ULL) |
                               (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

void oracle_uniform_fill(uint64_t seed, double lo, double hi, int64_t n, double* out) {
    mt64 g;
    mt64_seed(&g, seed);
    for (int64_t i = 0; i < n; ++i) {
        const double u = (double)(mt64_next(&g) >> 11) * 0x1.0p-53; /* rng.hpp:16 */
        out[i] = lo + (hi - lo) * u;                                   /* rng.hpp:18 */
    }
}

uint64_t oracle_uniform_bits(uint64_t seed, int64_t skip) {
    mt64 g;
    mt64_seed(&g, seed);
    for (int64_t i = 0; i < skip; ++i) (void)mt64_next(&g);
    return mt64_next(&g);
}

/* ---- tensor.cpp:23-29 ----------------------------------------------------------------- */
int oracle_reflect_index(int i, int n) {
    if (n == 1) return 0;
    const int period = 2 * (n - 1);
    int m = i % period;
    if (m < 0) m += period;
    return m < n ? m : period - m;
}

/* ---- tensor.cpp:31-48 ----------------------------------------------------------------- */
typedef struct {
    int y0, y1, x0, x1;
    double w00, w01, w10, w11, fy, fx;
} taps_t;

static taps_t taps_at(int h, int w, double y, double x) {
    taps_t t;
    const double by = floor(y), bx = floor(x);
    t.fy = y - by;
    t.fx = x - bx;
    t.y0 = oracle_reflect_index((int)by, h);
    t.y1 = oracle_reflect_index((int)by + 1, h);
    t.x0 = oracle_reflect_index((int)bx, w);
    t.x1 = oracle_reflect_index((int)bx + 1, w);
    t.w00 = (1.0 - t.fy) * (1.0 - t.fx);
    t.w01 = (1.0 - t.fy) * t.fx;
    t.w10 = t.fy * (1.0 - t.fx);
    t.w11 = t.fy * t.fx;
    return t;
}

void oracle_bilinear_taps(int h, int w, double y, double x, int* idx4, double* w6) {
    const taps_t t = taps_at(h, w, y, x);
    idx4[0] = t.y0;
    idx4[1] = t.y1;
    idx4[2] = t.x0;
    idx4[3] = t.x1;
    w6[0] = t.w00;
    w6[1] = t.w01;
    w6[2] = t.w10;
    w6[3] = t.w11;
    w6[4] = t.fy;
    w6[5] = t.fx;
}

/* ---- search.cpp:21-32 ----------------------------------------------------------------- */
int oracle_validate(const oracle_cfg* c) {
    if (c->ws < 1 || c->ws % 2 == 0)
        return fail(ORACLE_ECONFIG, "SearchConfig: ws must be odd and positive");
    if (c->ps < 1 || c->ps % 2 == 0)
        return fail(ORACLE_ECONFIG, "SearchConfig: ps must be odd and positive");
    if (c->wt < 0) return fail(ORACLE_ECONFIG, "SearchConfig: wt must be >= 0");
    if (c->stride0 < 1) return fail(ORACLE_ECONFIG, "SearchConfig: stride0 must be >= 1");
    if (!(c->stride1 > 0.0) || !isfinite(c->stride1))
        return fail(ORACLE_ECONFIG, "SearchConfig: stride1 must be positive and finite");
    if (c->topl < 1 || c->topl > (2 * c->wt + 1) * c->ws * c->ws)
        return fail(ORACLE_ECONFIG, "SearchConfig: topl must lie in [1, window slots]");
    if (!isfinite(c->softmax_scale))
        return fail(ORACLE_ECONFIG, "SearchConfig: softmax_scale must be finite");
    return ORACLE_OK;
}

/* ---- search.cpp:43-57 (QueryGrid) ------------------------------------------------------ */
typedef struct {
    int t, nh, nw, stride;
} qgrid;

static qgrid grid_over(int t, int h, int w, int stride) {
    qgrid g = {t, (h - 1) / stride + 1, (w - 1) / stride + 1, stride};
    return g;
}

int64_t oracle_rows(int t, int h, int w, int stride0) {
    const qgrid g = grid_over(t, h, w, stride0);
    return (int64_t)g.t * g.nh * g.nw;
}

static void grid_coords(const qgrid* g, int64_t row, int* qt, int* qy, int* qx) {
    *qx = (int)(row % g->nw) * g->stride;
    const int64_t r = row / g->nw;
    *qy = (int)(r % g->nh) * g->stride;
    *qt = (int)(r / g->nh);
}

/* ---- search.cpp:59-68: frame order 0, -1, +1, -2, +2, ... ------------------------------ */
static int scan_dt(int fpos) { return fpos == 0 ? 0 : ((fpos & 1) ? -((fpos + 1) / 2) : fpos / 2); }

#define VIDX(h, w, f, t_, y_, x_, c_) \
    ((((size_t)(t_) * (size_t)(h) + (size_t)(y_)) * (size_t)(w) + (size_t)(x_)) * (size_t)(f) + (size_t)(c_))

/* ---- search.cpp:72-122 ----------------------------------------------------------------- */
static void shift_to(int h, int w, const double* ff, const double* bf, int qt, int qy, int qx,
                     int dt, double* dy, double* dx, double* links) {
    if (dt == 0) {
        *dy = ff[VIDX(h, w, 2, qt, qy, qx, 0)];
        *dx = ff[VIDX(h, w, 2, qt, qy, qx, 1)];
        return;
    }
    const double* fld = dt > 0 ? ff : bf;
    const int step = dt > 0 ? 1 : -1;
    const int m = dt > 0 ? dt : -dt;
    double sy = 0.0, sx = 0.0;
    for (int k = 0; k < m; ++k) {
        const int fr = qt + step * k;
        double vy, vx;
        if (k == 0) {
            vy = fld[VIDX(h, w, 2, fr, qy, qx, 0)];
            vx = fld[VIDX(h, w, 2, fr, qy, qx, 1)];
        } else {
            const double py = qy + sy;
            const double px = qx + sx;
            const taps_t t = taps_at(h, w, py, px);
            const double a_y = fld[VIDX(h, w, 2, fr, t.y0, t.x0, 0)];
            const double b_y = fld[VIDX(h, w, 2, fr, t.y0, t.x1, 0)];
            const double c_y = fld[VIDX(h, w, 2, fr, t.y1, t.x0, 0)];
            const double d_y = fld[VIDX(h, w, 2, fr, t.y1, t.x1, 0)];
            const double a_x = fld[VIDX(h, w, 2, fr, t.y0, t.x0, 1)];
            const double b_x = fld[VIDX(h, w, 2, fr, t.y0, t.x1, 1)];
            const double c_x = fld[VIDX(h, w, 2, fr, t.y1, t.x0, 1)];
            const double d_x = fld[VIDX(h, w, 2, fr, t.y1, t.x1, 1)];
            vy = t.w00 * a_y + t.w01 * b_y + t.w10 * c_y + t.w11 * d_y;
            vx = t.w00 * a_x + t.w01 * b_x + t.w10 * c_x + t.w11 * d_x;
            if (links) { /* search.cpp:104-117: position + spatial Jacobian of the link */
                double* lk = links + (size_t)(k - 1) * 6;
                lk[0] = py;
                lk[1] = px;
                lk[2] = -(1.0 - t.fx) * a_y - t.fx * b_y + (1.0 - t.fx) * c_y + t.fx * d_y;
                lk[3] = -(1.0 - t.fy) * a_y + (1.0 - t.fy) * b_y - t.fy * c_y + t.fy * d_y;
                lk[4] = -(1.0 - t.fx) * a_x - t.fx * b_x + (1.0 - t.fx) * c_x + t.fx * d_x;
                lk[5] = -(1.0 - t.fy) * a_x + (1.0 - t.fy) * b_x - t.fy * c_x + t.fy * d_x;
            }
        }
        sy += vy;
        sx += vx;
    }
    *dy = sy;
    *dx = sx;
}

int oracle_accumulate_shift(int t, int h, int w, const double* ff, const double* bf, int qt,
                            int qy, int qx, int dt, double* dy, double* dx, double* links) {
    (void)t;
    shift_to(h, w, ff, bf, qt, qy, qx, dt, dy, dx, links);
    return ORACLE_OK;
}

/* ---- search.cpp:124-151: (py, px, channel) accumulation order ------------------------- */
static double patch_sim(int h, int w, int f, const double* q, const double* k, int qt, int qy,
                        int qx, int kt, double ky, double kx, int ps, int metric) {
    const int half = ps / 2;
    double acc = 0.0;
    for (int py = -half; py <= half; ++py) {
        const int ry = oracle_reflect_index(qy + py, h);
        const double sy = ky + (double)py;
        for (int px = -half; px <= half; ++px) {
            const int rx = oracle_reflect_index(qx + px, w);
            const double sx = kx + (double)px;
            const taps_t t = taps_at(h, w, sy, sx);
            const double* qp = q + VIDX(h, w, f, qt, ry, rx, 0);
            const double* k00 = k + VIDX(h, w, f, kt, t.y0, t.x0, 0);
            const double* k01 = k + VIDX(h, w, f, kt, t.y0, t.x1, 0);
            const double* k10 = k + VIDX(h, w, f, kt, t.y1, t.x0, 0);
            const double* k11 = k + VIDX(h, w, f, kt, t.y1, t.x1, 0);
            for (int c = 0; c < f; ++c) {
                const double kv = t.w00 * k00[c] + t.w01 * k01[c] + t.w10 * k10[c] + t.w11 * k11[c];
                if (metric == 0) {
                    acc += qp[c] * kv;
                } else {
                    const double d = qp[c] - kv;
                    acc -= d * d;
                }
            }
        }
    }
    return acc;
}

static int check_flow_finite(const double* fl, size_t n, const char* what) {
    for (size_t i = 0; i < n; ++i)
        if (!isfinite(fl[i])) {
            char msg[96];
            snprintf(msg, sizeof msg, "%s: flow holds a non-finite value", what);
            return fail(ORACLE_EDOMAIN, msg);
        }
    return ORACLE_OK;
}

static int forward_checks(int t, int h, int w, const double* ff, const double* bf,
                          const oracle_cfg* c) {
    int rc = oracle_validate(c); /* search.cpp:175-183 */
    if (rc) return rc;
    const size_t nf = (size_t)t * h * w * 2;
    if ((rc = check_flow_finite(ff, nf, "search fflow"))) return rc;
    return check_flow_finite(bf, nf, "search bflow");
}

/* ---- search.cpp:187-197: ascending-slot insertion; equal values never displace -------- */
static void keep_best(double* vals, int64_t* slots, int l, double v, int64_t s) {
    if (!(v > vals[l - 1])) return;
    int pos = l - 1;
    while (pos > 0 && v > vals[pos - 1]) --pos;
    for (int j = l - 1; j > pos; --j) {
        vals[j] = vals[j - 1];
        slots[j] = slots[j - 1];
    }
    vals[pos] = v;
    slots[pos] = s;
}

/* ---- search.cpp:207-234 ---------------------------------------------------------------- */
static void emit_entries(int h, int w, const double* ff, const double* bf, const oracle_cfg* c,
                         int64_t row, int qt, int qy, int qx, const double* vals,
                         const int64_t* slots, double* sims, double* offsets, double* centers,
                         double* chains) {
    const int ss = c->ws * c->ws, half_ws = c->ws / 2;
    const int cstride = c->wt > 1 ? c->wt - 1 : 0;
    for (int li = 0; li < c->topl; ++li) {
        const int fpos = (int)(slots[li] / ss);
        const int rem = (int)(slots[li] % ss);
        const int dt = scan_dt(fpos), dyi = rem / c->ws, dxi = rem % c->ws;
        double sdy, sdx;
        shift_to(h, w, ff, bf, qt, qy, qx, dt, &sdy, &sdx, NULL);
        const double cy = (double)qy + sdy, cx = (double)qx + sdx;
        const double ky = cy + c->stride1 * (double)(dyi - half_ws);
        const double kx = cx + c->stride1 * (double)(dxi - half_ws);
        const size_t e = (size_t)row * c->topl + li;
        if (sims) sims[e] = vals[li];
        if (offsets) {
            offsets[e * 3 + 0] = (double)dt;
            offsets[e * 3 + 1] = ky - (double)qy;
            offsets[e * 3 + 2] = kx - (double)qx;
        }
        if (centers) {
            centers[e * 3 + 0] = (double)(qt + dt);
            centers[e * 3 + 1] = ky;
            centers[e * 3 + 2] = kx;
        }
        if (chains && cstride > 0 && (dt > 1 || dt < -1))
            shift_to(h, w, ff, bf, qt, qy, qx, dt, &sdy, &sdx, chains + e * (size_t)cstride * 6);
    }
}

/* ---- search.cpp:264-327: fused streaming top-L -------------------------------------- */
int oracle_search_fwd(int t, int h, int w, int f, const double* q, const double* k,
                      const double* ff, const double* bf, const oracle_cfg* c, double* sims,
                      double* offsets, double* centers, double* chains) {
    int rc = forward_checks(t, h, w, ff, bf, c);
    if (rc) return rc;
    const qgrid g = grid_over(t, h, w, c->stride0);
    const int64_t rows = (int64_t)g.t * g.nh * g.nw;
    const int l = c->topl, half_ws = c->ws / 2, nfr = 2 * c->wt + 1;
    const int cstride = c->wt > 1 ? c->wt - 1 : 0;
    if (chains && cstride > 0) memset(chains, 0, sizeof(double) * (size_t)rows * l * cstride * 6);
    double* vals = malloc(sizeof(double) * l);
    int64_t* slots = malloc(sizeof(int64_t) * l);
    int underfull = 0;
    for (int64_t row = 0; row < rows; ++row) {
        for (int i = 0; i < l; ++i) {
            vals[i] = -INFINITY;
            slots[i] = -1;
        }
        int qt, qy, qx;
        grid_coords(&g, row, &qt, &qy, &qx);
        int valid = 0;
        for (int fpos = 0; fpos < nfr; ++fpos) {
            const int dt = scan_dt(fpos), kt = qt + dt;
            if (kt < 0 || kt >= t) continue; /* search.cpp:300 */
            double sdy, sdx;
            shift_to(h, w, ff, bf, qt, qy, qx, dt, &sdy, &sdx, NULL);
            const double cy = (double)qy + sdy, cx = (double)qx + sdx;
            const int64_t base = (int64_t)fpos * c->ws * c->ws;
            for (int dyi = 0; dyi < c->ws; ++dyi) {
                const double ky = cy + c->stride1 * (double)(dyi - half_ws);
                for (int dxi = 0; dxi < c->ws; ++dxi) {
                    const double kx = cx + c->stride1 * (double)(dxi - half_ws);
                    const double v = patch_sim(h, w, f, q, k, qt, qy, qx, kt, ky, kx, c->ps,
                                               c->metric);
                    keep_best(vals, slots, l, v, base + (int64_t)dyi * c->ws + dxi);
                    ++valid;
                }
            }
        }
        if (valid < l) {
            underfull = 1;
            continue;
        }
        emit_entries(h, w, ff, bf, c, row, qt, qy, qx, vals, slots, sims, offsets, centers,
                     chains);
    }
    free(vals);
    free(slots);
    if (underfull)
        return fail(ORACLE_ECONFIG, "search: topl exceeds the valid window entries of some query");
    return ORACLE_OK;
}

/* ---- search.cpp:329-376: the materialised window grid (pre-selection scores) --------- */
int oracle_search_full_grid(int t, int h, int w, int f, const double* q, const double* k,
                            const double* ff, const double* bf, const oracle_cfg* c,
                            double* grid, double* grid_offsets) {
    int rc = forward_checks(t, h, w, ff, bf, c);
    if (rc) return rc;
    const qgrid g = grid_over(t, h, w, c->stride0);
    const int64_t rows = (int64_t)g.t * g.nh * g.nw;
    const int ss = c->ws * c->ws, n = (2 * c->wt + 1) * ss, half_ws = c->ws / 2;
    for (int64_t row = 0; row < rows; ++row) {
        int qt, qy, qx;
        grid_coords(&g, row, &qt, &qy, &qx);
        for (int fpos = 0; fpos < 2 * c->wt + 1; ++fpos) {
            const int dt = scan_dt(fpos), kt = qt + dt;
            double sdy = 0.0, sdx = 0.0;
            const int on = kt >= 0 && kt < t;
            if (on) shift_to(h, w, ff, bf, qt, qy, qx, dt, &sdy, &sdx, NULL);
            const double cy = (double)qy + sdy, cx = (double)qx + sdx;
            for (int dyi = 0; dyi < c->ws; ++dyi) {
                const double ky = cy + c->stride1 * (double)(dyi - half_ws);
                for (int dxi = 0; dxi < c->ws; ++dxi) {
                    const double kx = cx + c->stride1 * (double)(dxi - half_ws);
                    const size_t e = (size_t)row * n + (size_t)fpos * ss + dyi * c->ws + dxi;
                    grid[e] = on ? patch_sim(h, w, f, q, k, qt, qy, qx, kt, ky, kx, c->ps,
                                             c->metric)
                                 : -INFINITY; /* search.cpp:359-361 */
                    if (grid_offsets) {
                        grid_offsets[e * 3 + 0] = (double)dt;
                        grid_offsets[e * 3 + 1] = on ? ky - (double)qy : 0.0;
                        grid_offsets[e * 3 + 2] = on ? kx - (double)qx : 0.0;
                    }
                }
            }
        }
    }
    return ORACLE_OK;
}

/* ---- search.cpp:430-468: (value desc, column asc) selection --------------------------- */
int oracle_top_l(int64_t rows, int cols, const double* full, const double* full_offsets,
                 int topl, double* sel, double* sel_offsets) {
    if (topl < 1 || topl > cols) return fail(ORACLE_ECONFIG, "top_l: L out of range");
    double* vals = malloc(sizeof(double) * topl);
    int64_t* idx = malloc(sizeof(int64_t) * topl);
    int underfull = 0;
    for (int64_t r = 0; r < rows; ++r) {
        const double* src = full + (size_t)r * cols;
        for (int i = 0; i < topl; ++i) {
            vals[i] = -INFINITY;
            idx[i] = -1;
        }
        /* columns arrive ascending, so strict '>' insertion == the tie-broken sort order;
         * -inf never enters, which is the reference's underfull condition */
        for (int col = 0; col < cols; ++col) keep_best(vals, idx, topl, src[col], col);
        if (idx[topl - 1] < 0) {
            underfull = 1;
            continue;
        }
        for (int li = 0; li < topl; ++li) {
            sel[(size_t)r * topl + li] = vals[li];
            for (int cc = 0; cc < 3; ++cc)
                sel_offsets[((size_t)r * topl + li) * 3 + cc] =
                    full_offsets[((size_t)r * cols + idx[li]) * 3 + cc];
        }
    }
    free(vals);
    free(idx);
    if (underfull) return fail(ORACLE_EDOMAIN, "top_l: some row has fewer than L valid entries");
    return ORACLE_OK;
}

/* ---- search.cpp:470-493 ---------------------------------------------------------------- */
int oracle_replay(int t, int h, int w, int f, const double* q, const double* k,
                  const oracle_cfg* c, const double* centers, double* sims) {
    const qgrid g = grid_over(t, h, w, c->stride0);
    const int64_t rows = (int64_t)g.t * g.nh * g.nw;
    for (int64_t row = 0; row < rows; ++row) {
        int qt, qy, qx;
        grid_coords(&g, row, &qt, &qy, &qx);
        for (int li = 0; li < c->topl; ++li) {
            const double* ce = centers + ((size_t)row * c->topl + li) * 3;
            sims[(size_t)row * c->topl + li] =
                patch_sim(h, w, f, q, k, qt, qy, qx, (int)ce[0], ce[1], ce[2], c->ps, c->metric);
        }
    }
    return ORACLE_OK;
}

/* ---- search.cpp:499-667 (backward_entry<false>) and 671-711 (deterministic order) ------- */
int oracle_search_bwd(int t, int h, int w, int f, const double* q, const double* k,
                      const oracle_cfg* c, const double* centers, const double* chains,
                      const double* grad_sims, double* dq, double* dk, double* dff, double* dbf) {
    const qgrid g = grid_over(t, h, w, c->stride0);
    const int64_t rows = (int64_t)g.t * g.nh * g.nw;
    const size_t nv = (size_t)t * h * w * f, nfl = (size_t)t * h * w * 2;
    memset(dq, 0, nv * sizeof(double));
    memset(dk, 0, nv * sizeof(double));
    memset(dff, 0, nfl * sizeof(double));
    memset(dbf, 0, nfl * sizeof(double));
    const int half = c->ps / 2, cstride = c->wt > 1 ? c->wt - 1 : 0;
    for (int64_t row = 0; row < rows; ++row) {
        int qt, qy, qx;
        grid_coords(&g, row, &qt, &qy, &qx);
        for (int li = 0; li < c->topl; ++li) {
            const size_t e = (size_t)row * c->topl + li;
            const double gsel = grad_sims[e];
            if (gsel == 0.0) continue; /* search.cpp:692 */
            const int kt = (int)centers[e * 3 + 0];
            const double ky = centers[e * 3 + 1], kx = centers[e * 3 + 2];
            const int dt = kt - qt;
            double gy = 0.0, gx = 0.0;
            for (int py = -half; py <= half; ++py) {
                const int ry = oracle_reflect_index(qy + py, h);
                const double sy = ky + (double)py;
                for (int px = -half; px <= half; ++px) {
                    const int rx = oracle_reflect_index(qx + px, w);
                    const double sx = kx + (double)px;
                    const taps_t tp = taps_at(h, w, sy, sx);
                    for (int ch = 0; ch < f; ++ch) {
                        const double qv = q[VIDX(h, w, f, qt, ry, rx, ch)];
                        const size_t i00 = VIDX(h, w, f, kt, tp.y0, tp.x0, ch);
                        const size_t i01 = VIDX(h, w, f, kt, tp.y0, tp.x1, ch);
                        const size_t i10 = VIDX(h, w, f, kt, tp.y1, tp.x0, ch);
                        const size_t i11 = VIDX(h, w, f, kt, tp.y1, tp.x1, ch);
                        const double k00 = k[i00], k01 = k[i01], k10 = k[i10], k11 = k[i11];
                        const double kv = tp.w00 * k00 + tp.w01 * k01 + tp.w10 * k10 + tp.w11 * k11;
                        double ds_dq, ds_dk;
                        if (c->metric == 0) {
                            ds_dq = kv;
                            ds_dk = qv;
                        } else {
                            const double diff = qv - kv;
                            ds_dq = -2.0 * diff;
                            ds_dk = 2.0 * diff;
                        }
                        const double gq = gsel * ds_dq, gk = gsel * ds_dk;
                        dq[VIDX(h, w, f, qt, ry, rx, ch)] += gq;
                        dk[i00] += gk * tp.w00;
                        dk[i01] += gk * tp.w01;
                        dk[i10] += gk * tp.w10;
                        dk[i11] += gk * tp.w11;
                        const double dkv_dy = -(1.0 - tp.fx) * k00 - tp.fx * k01 +
                                              (1.0 - tp.fx) * k10 + tp.fx * k11;
                        const double dkv_dx = -(1.0 - tp.fy) * k00 + (1.0 - tp.fy) * k01 -
                                              tp.fy * k10 + tp.fy * k11;
                        gy += gk * dkv_dy;
                        gx += gk * dkv_dx;
                    }
                }
            }
            /* search.cpp:584-666: route (gy, gx) back through the composition chain */
            double* fld = dt >= 0 ? dff : dbf;
            const int step = dt >= 0 ? 1 : -1;
            const int m = dt == 0 ? 1 : (dt > 0 ? dt : -dt);
            double vy = gy, vx = gx;
            const double* chain = chains ? chains + e * (size_t)cstride * 6 : NULL;
            for (int kk = m - 1; kk >= 1; --kk) {
                const double* lk = chain + (size_t)(kk - 1) * 6;
                const taps_t tp = taps_at(h, w, lk[0], lk[1]);
                const int fr = qt + step * kk;
                fld[VIDX(h, w, 2, fr, tp.y0, tp.x0, 0)] += vy * tp.w00;
                fld[VIDX(h, w, 2, fr, tp.y0, tp.x1, 0)] += vy * tp.w01;
                fld[VIDX(h, w, 2, fr, tp.y1, tp.x0, 0)] += vy * tp.w10;
                fld[VIDX(h, w, 2, fr, tp.y1, tp.x1, 0)] += vy * tp.w11;
                fld[VIDX(h, w, 2, fr, tp.y0, tp.x0, 1)] += vx * tp.w00;
                fld[VIDX(h, w, 2, fr, tp.y0, tp.x1, 1)] += vx * tp.w01;
                fld[VIDX(h, w, 2, fr, tp.y1, tp.x0, 1)] += vx * tp.w10;
                fld[VIDX(h, w, 2, fr, tp.y1, tp.x1, 1)] += vx * tp.w11;
                const double ny = vy + lk[2] * vy + lk[4] * vx;
                const double nx = vx + lk[3] * vy + lk[5] * vx;
                vy = ny;
                vx = nx;
            }
            fld[VIDX(h, w, 2, qt, qy, qx, 0)] += vy;
            fld[VIDX(h, w, 2, qt, qy, qx, 1)] += vx;
        }
    }
    return ORACLE_OK;
}

/* ---- aggregate.cpp:16-37 --------------------------------------------------------------- */
int oracle_softmax_rows(int64_t rows, int l, const double* sims, double beta, double* weights) {
    for (int64_t r = 0; r < rows; ++r) {
        const double* s = sims + (size_t)r * l;
        double* wr = weights + (size_t)r * l;
        double m = -INFINITY;
        for (int j = 0; j < l; ++j) {
            const double z = beta * s[j];
            if (!isfinite(z)) return fail(ORACLE_EDOMAIN, "softmax_rows: non-finite input");
            m = (m < z) ? z : m; /* std::max(m, z) */
        }
        double sum = 0.0;
        for (int j = 0; j < l; ++j) {
            const double e = exp(beta * s[j] - m);
            wr[j] = e;
            sum += e;
        }
        for (int j = 0; j < l; ++j) wr[j] /= sum;
    }
    return ORACLE_OK;
}

/* ---- aggregate.cpp:41-100: shapes, hole-free rule and the write set ------------------- */
typedef struct {
    qgrid g;
    int t, h, w, f, half, qmax_y, qmax_x, stride;
} agg_shape;

static int agg_checks(int t, int h, int w, int f, int64_t rows, int l, const oracle_cfg* c,
                      agg_shape* s) {
    int rc = oracle_validate(c);
    if (rc) return rc;
    if (!((c->ps - 1) / 2 < c->stride0))
        return fail(ORACLE_ECONFIG, "aggregate: (ps-1)/2 < stride0 is required for hole-free output");
    s->g = grid_over(t, h, w, c->stride0);
    if (rows != (int64_t)s->g.t * s->g.nh * s->g.nw)
        return fail(ORACLE_EDOMAIN, "aggregate: weight/offset rows do not match the query grid");
    if (l != c->topl)
        return fail(ORACLE_EDOMAIN, "aggregate: weight/offset L does not match the config");
    s->t = t;
    s->h = h;
    s->w = w;
    s->f = f;
    s->half = c->ps / 2;
    s->stride = c->stride0;
    s->qmax_y = (s->g.nh - 1) * c->stride0;
    s->qmax_x = (s->g.nw - 1) * c->stride0;
    return ORACLE_OK;
}

static int clampi(int d, int half) { return d < -half ? -half : (d > half ? half : d); }

static int owner_index(int coord, int stride, int n) { /* aggregate.hpp:91-95 */
    int gi = (coord + (stride - 1) / 2) / stride;
    return gi > n - 1 ? n - 1 : gi;
}

static void cell_span(int gi, int stride, int n, int extent, int* lo, int* hi) {
    const int a = (stride - 1) / 2; /* aggregate.cpp:71-75 */
    *lo = gi == 0 ? 0 : gi * stride - a;
    *hi = gi == n - 1 ? extent - 1 : gi * stride + (stride - 1 - a);
}

/* aggregate.cpp:104-122: one (query, patch pixel) unit, all L neighbours, optionally one. */
static int add_unit(const agg_shape* s, const double* v, const double* weights,
                    const double* offsets, int l, int64_t row, int ti, int qy, int qx, int pyu,
                    int pxu, int only_li, double* acc) {
    for (int li = 0; li < l; ++li) {
        if (only_li >= 0 && li != only_li) continue;
        const size_t e = (size_t)row * l + li;
        const int kt = ti + (int)llround(offsets[e * 3 + 0]);
        if (kt < 0 || kt >= s->t) return 0;
        const double sy = (double)qy + offsets[e * 3 + 1] + (double)pyu;
        const double sx = (double)qx + offsets[e * 3 + 2] + (double)pxu;
        const taps_t tp = taps_at(s->h, s->w, sy, sx);
        const double wv = weights[e];
        const double* a = v + VIDX(s->h, s->w, s->f, kt, tp.y0, tp.x0, 0);
        const double* b = v + VIDX(s->h, s->w, s->f, kt, tp.y0, tp.x1, 0);
        const double* cc = v + VIDX(s->h, s->w, s->f, kt, tp.y1, tp.x0, 0);
        const double* d = v + VIDX(s->h, s->w, s->f, kt, tp.y1, tp.x1, 0);
        for (int ch = 0; ch < s->f; ++ch)
            acc[ch] += wv * (tp.w00 * a[ch] + tp.w01 * b[ch] + tp.w10 * cc[ch] + tp.w11 * d[ch]);
    }
    return 1;
}

/* Fixed-order gather of one output pixel (aggregate.cpp:156-188): footprint contributions
 * with py, px ascending, then the owning query's cell completion.  Returns the number of
 * contributing units, or -1 when an offset leaves the clip. */
static int gather_pixel(const agg_shape* s, const double* v, const double* weights,
                        const double* offsets, int l, int ti, int y, int x, int only_li,
                        double* acc) {
    const int st = s->stride;
    int cnt = 0;
    for (int py = -s->half; py <= s->half; ++py) {
        const int qy = y - py;
        if (qy < 0 || qy > s->qmax_y || qy % st != 0) continue;
        for (int px = -s->half; px <= s->half; ++px) {
            const int qx = x - px;
            if (qx < 0 || qx > s->qmax_x || qx % st != 0) continue;
            const int64_t row = ((int64_t)ti * s->g.nh + qy / st) * s->g.nw + qx / st;
            if (!add_unit(s, v, weights, offsets, l, row, ti, qy, qx, py, px, only_li, acc))
                return -1;
            ++cnt;
        }
    }
    const int qy = owner_index(y, st, s->g.nh) * st;
    const int qx = owner_index(x, st, s->g.nw) * st;
    if (abs(y - qy) > s->half || abs(x - qx) > s->half) {
        const int64_t row = ((int64_t)ti * s->g.nh + qy / st) * s->g.nw + qx / st;
        if (!add_unit(s, v, weights, offsets, l, row, ti, qy, qx, clampi(y - qy, s->half),
                      clampi(x - qx, s->half), only_li, acc))
            return -1;
        ++cnt;
    }
    return cnt;
}

/* ---- aggregate.cpp:124-203 (deterministic gather form) -------------------------------- */
int oracle_wpsum(int t, int h, int w, int f, const double* v, int64_t rows, int l,
                 const double* weights, const double* offsets, const oracle_cfg* c, double* out,
                 int32_t* counts) {
    agg_shape s;
    int rc = agg_checks(t, h, w, f, rows, l, c, &s);
    if (rc) return rc;
    double* acc = malloc(sizeof(double) * f);
    int bad = 0;
    for (int ti = 0; ti < t; ++ti)
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x) {
                for (int ch = 0; ch < f; ++ch) acc[ch] = 0.0;
                const int cnt = gather_pixel(&s, v, weights, offsets, l, ti, y, x, -1, acc);
                const size_t p = ((size_t)ti * h + y) * w + x;
                if (cnt <= 0) {
                    bad = 1;
                    continue;
                }
                if (counts) counts[p] = cnt;
                for (int ch = 0; ch < f; ++ch) out[p * f + ch] = acc[ch] / (double)cnt;
            }
    free(acc);
    if (bad)
        return fail(ORACLE_EDOMAIN, "wpsum: offsets leave the clip or a pixel has no writers");
    return ORACLE_OK;
}

/* ---- aggregate.cpp:285-347 ------------------------------------------------------------- */
int oracle_gather_stack(int t, int h, int w, int f, const double* v, int64_t rows, int l,
                        const double* weights, const double* offsets, const oracle_cfg* c,
                        double* out) {
    agg_shape s;
    int rc = agg_checks(t, h, w, f, rows, l, c, &s);
    if (rc) return rc;
    int bad = 0;
    const size_t plane = (size_t)t * h * w * f;
    for (int li = 0; li < l; ++li)
        for (int ti = 0; ti < t; ++ti)
            for (int y = 0; y < h; ++y)
                for (int x = 0; x < w; ++x) {
                    double* o = out + li * plane + (((size_t)ti * h + y) * w + x) * f;
                    for (int ch = 0; ch < f; ++ch) o[ch] = 0.0;
                    if (gather_pixel(&s, v, weights, offsets, l, ti, y, x, li, o) < 0) bad = 1;
                }
    if (bad) return fail(ORACLE_EDOMAIN, "gather_stack: offsets leave the clip");
    return ORACLE_OK;
}

/* ---- aggregate.cpp:351-408 (backward_query<false>) ------------------------------------ */
static void backprop_query(const agg_shape* s, const double* go, const int32_t* counts,
                           const double* v, const double* weights, const double* offsets, int l,
                           int64_t row, double* dv, double* dw) {
    int ti, qy, qx;
    grid_coords(&s->g, row, &ti, &qy, &qx);
    const int st = s->stride;
    /* for_each_write (aggregate.cpp:81-100): footprint, then the stride-cell remainder */
    int ylo, yhi, xlo, xhi;
    cell_span(qy / st, st, s->g.nh, s->h, &ylo, &yhi);
    cell_span(qx / st, st, s->g.nw, s->w, &xlo, &xhi);
    const int nfoot = (2 * s->half + 1) * (2 * s->half + 1);
    const int ncell = (yhi - ylo + 1) * (xhi - xlo + 1);
    for (int it = 0; it < nfoot + ncell; ++it) {
        int y, x, pyu, pxu;
        if (it < nfoot) {
            pyu = it / (2 * s->half + 1) - s->half;
            pxu = it % (2 * s->half + 1) - s->half;
            y = qy + pyu;
            x = qx + pxu;
            if (y < 0 || y >= s->h || x < 0 || x >= s->w) continue;
        } else {
            const int j = it - nfoot, cw = xhi - xlo + 1;
            y = ylo + j / cw;
            x = xlo + j % cw;
            if (abs(y - qy) <= s->half && abs(x - qx) <= s->half) continue;
            pyu = clampi(y - qy, s->half);
            pxu = clampi(x - qx, s->half);
        }
        const double inv_cnt = 1.0 / (double)counts[((size_t)ti * s->h + y) * s->w + x];
        for (int li = 0; li < l; ++li) {
            const size_t e = (size_t)row * l + li;
            const int kt = ti + (int)llround(offsets[e * 3 + 0]);
            const double sy = (double)qy + offsets[e * 3 + 1] + (double)pyu;
            const double sx = (double)qx + offsets[e * 3 + 2] + (double)pxu;
            const taps_t tp = taps_at(s->h, s->w, sy, sx);
            const double wv = weights[e];
            double dw_acc = 0.0;
            for (int ch = 0; ch < s->f; ++ch) {
                const double gg = go[VIDX(s->h, s->w, s->f, ti, y, x, ch)] * inv_cnt;
                const size_t i00 = VIDX(s->h, s->w, s->f, kt, tp.y0, tp.x0, ch);
                const size_t i01 = VIDX(s->h, s->w, s->f, kt, tp.y0, tp.x1, ch);
                const size_t i10 = VIDX(s->h, s->w, s->f, kt, tp.y1, tp.x0, ch);
                const size_t i11 = VIDX(s->h, s->w, s->f, kt, tp.y1, tp.x1, ch);
                const double sample =
                    tp.w00 * v[i00] + tp.w01 * v[i01] + tp.w10 * v[i10] + tp.w11 * v[i11];
                dw_acc += gg * sample;
                if (dv) {
                    const double gv = gg * wv;
                    dv[i00] += gv * tp.w00;
                    dv[i01] += gv * tp.w01;
                    dv[i10] += gv * tp.w10;
                    dv[i11] += gv * tp.w11;
                }
            }
            if (dw) dw[e] += dw_acc;
        }
    }
}

/* ---- aggregate.cpp:412-460 (deterministic: dW pass, then dV in query order) ---------- */
int oracle_wpsum_bwd(int t, int h, int w, int f, const double* grad_out, const int32_t* counts,
                     const double* v, int64_t rows, int l, const double* weights,
                     const double* offsets, const oracle_cfg* c, double* dv, double* dw) {
    agg_shape s;
    s.g = grid_over(t, h, w, c->stride0);
    if (rows != (int64_t)s.g.t * s.g.nh * s.g.nw || l != c->topl)
        return fail(ORACLE_EDOMAIN, "wpsum_backward: weight/offset shape does not match the tape");
    s.t = t;
    s.h = h;
    s.w = w;
    s.f = f;
    s.half = c->ps / 2;
    s.stride = c->stride0;
    s.qmax_y = (s.g.nh - 1) * c->stride0;
    s.qmax_x = (s.g.nw - 1) * c->stride0;
    memset(dv, 0, sizeof(double) * (size_t)t * h * w * f);
    memset(dw, 0, sizeof(double) * (size_t)rows * l);
    for (int64_t row = 0; row < rows; ++row)
        backprop_query(&s, grad_out, counts, v, weights, offsets, l, row, NULL, dw);
    for (int64_t row = 0; row < rows; ++row)
        backprop_query(&s, grad_out, counts, v, weights, offsets, l, row, dv, NULL);
    return ORACLE_OK;
}

/* ---- flow.cpp:114-175 estimate_flow_block_matching ---------------------------------- */
int oracle_block_match(int h, int w, int f, const double* a, const double* b, int block,
                       int radius, double* flow) {
    if (block < 1 || block % 2 == 0)
        return fail(ORACLE_ECONFIG, "estimate_flow_block_matching: block must be odd and positive");
    if (radius < 0) return fail(ORACLE_ECONFIG, "estimate_flow_block_matching: radius must be >= 0");
    const int nby = (h + block - 1) / block, nbx = (w + block - 1) / block;
    for (int bi = 0; bi < nby * nbx; ++bi) {
        const int by = bi / nbx, bx = bi % nbx;
        const int y0 = by * block, x0 = bx * block;
        const int y1 = y0 + block < h ? y0 + block : h, x1 = x0 + block < w ? x0 + block : w;
        double best = INFINITY;
        int bdy = 0, bdx = 0;
        for (int dy = -radius; dy <= radius; ++dy)
            for (int dx = -radius; dx <= radius; ++dx) {
                double ssd = 0.0;
                for (int y = y0; y < y1; ++y) {
                    const int ry = oracle_reflect_index(y + dy, h);
                    for (int x = x0; x < x1; ++x) {
                        const int rx = oracle_reflect_index(x + dx, w);
                        for (int c = 0; c < f; ++c) {
                            const double d = a[((int64_t)y * w + x) * f + c] - b[((int64_t)ry * w + rx) * f + c];
                            ssd += d * d;
                        }
                    }
                }
                if (ssd < best) { /* strict: first hit in scan order wins ties */
                    best = ssd;
                    bdy = dy;
                    bdx = dx;
                }
            }
        for (int y = y0; y < y1; ++y)
            for (int x = x0; x < x1; ++x) {
                flow[((int64_t)y * w + x) * 2 + 0] = (double)bdy;
                flow[((int64_t)y * w + x) * 2 + 1] = (double)bdx;
            }
    }
    return ORACLE_OK;
}

/* ---- tensor.cpp:79-90 psnr ------------------------------------------------------------ */
int oracle_psnr(int64_t n, const double* a, const double* b, double peak, double* out) {
    if (!(peak > 0.0)) return fail(ORACLE_ECONFIG, "psnr: peak must be positive");
    double sq = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double d = a[i] - b[i];
        sq += d * d;
    }
    const double mse = sq / (double)n;
    *out = mse == 0.0 ? INFINITY : 10.0 * log10(peak * peak / mse);
    return ORACLE_OK;
}

/* ---- rng.hpp:30-53 GaussianStream ------------------------------------------------------ */
void oracle_gaussian_fill(uint64_t seed, int64_t n, double* out) {
    mt64 g;
    mt64_seed(&g, seed);
    const double kPi = 3.14159265358979323846;
    for (int64_t i = 0; i < n; i += 2) {
        const double u1 = ((double)(mt64_next(&g) >> 11) + 1.0) * 0x1.0p-53; /* (0,1] */
        const double u2 = (double)(mt64_next(&g) >> 11) * 0x1.0p-53;         /* [0,1) */
        const double r = sqrt(-2.0 * log(u1));
        const double ang = 2.0 * kPi * u2;
        out[i] = r * cos(ang);
        if (i + 1 < n) out[i + 1] = r * sin(ang);
    }
}
