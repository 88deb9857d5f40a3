/* TEST INFRASTRUCTURE ONLY -- the CPU oracle for the parity tests.
 *
 * Plain-C (fp64, serial) restatement of the reference's Shifted Non-Local Search hot
 * path, /root/reference/proj/src/{tensor,search,aggregate}.cpp.  Every function cites
 * the reference lines it follows.  It is pinned bit-for-bit against the reference itself
 * (oracle/_ref/libsnls_ref.so, built from the unmodified sources) and against the golden
 * fixtures in tests/golden/ (generated from that library by tests/gen_golden.py).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use it.
 *
 * Layouts follow the reference: videos T x H x W x F (F fastest, tensor.hpp:17-31),
 * flows T x H x W x 2 with (dy, dx) (flow.hpp:12-28), rows (t, y, x) x fastest
 * (search.hpp:47-55), sims rows x L, offsets rows x L x 3 (dt, dy, dx), tape centres
 * rows x L x 3 (kt, ky, kx), chains rows x L x max(wt-1,0) x 6 (search.hpp:89-110).
 */
#ifndef SNLS_ORACLE_H
#define SNLS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Flat mirror of snls::SearchConfig (search.hpp:17-26); metric 0 = inner product,
 * 1 = negated squared L2 (enum order of search.hpp:12). */
typedef struct {
    int ws, wt, ps, stride0;
    double stride1;
    int topl;
    int metric;
    double softmax_scale;
} oracle_cfg;

enum { ORACLE_OK = 0, ORACLE_ECONFIG = 1, ORACLE_EDOMAIN = 2 };

const char* oracle_last_error(void);

/* rng.hpp:12-24 (std::mt19937_64, top 53 bits) */
void oracle_uniform_fill(uint64_t seed, double lo, double hi, int64_t n, double* out);
uint64_t oracle_uniform_bits(uint64_t seed, int64_t skip);

int oracle_reflect_index(int i, int n);
void oracle_bilinear_taps(int h, int w, double y, double x, int* idx4, double* w6);

int oracle_validate(const oracle_cfg* c);
int64_t oracle_rows(int t, int h, int w, int stride0);

int oracle_accumulate_shift(int t, int h, int w, const double* ff, const double* bf, int qt,
                            int qy, int qx, int dt, double* dy, double* dx, double* links);

int oracle_search_fwd(int t, int h, int w, int f, const double* q, const double* k,
                      const double* ff, const double* bf, const oracle_cfg* c, double* sims,
                      double* offsets, double* centers, double* chains);
/* Materialised variant (search.cpp:329-410): also writes the pre-selection grid
 * rows x window_slots (-inf for off-clip frames) when `grid` is non-null. */
int oracle_search_full_grid(int t, int h, int w, int f, const double* q, const double* k,
                            const double* ff, const double* bf, const oracle_cfg* c,
                            double* grid, double* grid_offsets);
int oracle_top_l(int64_t rows, int cols, const double* full, const double* full_offsets,
                 int topl, double* sel, double* sel_offsets);
int oracle_replay(int t, int h, int w, int f, const double* q, const double* k,
                  const oracle_cfg* c, const double* centers, double* sims);
int oracle_search_bwd(int t, int h, int w, int f, const double* q, const double* k,
                      const oracle_cfg* c, const double* centers, const double* chains,
                      const double* grad_sims, double* dq, double* dk, double* dff, double* dbf);

int oracle_softmax_rows(int64_t rows, int l, const double* sims, double beta, double* weights);
int oracle_wpsum(int t, int h, int w, int f, const double* v, int64_t rows, int l,
                 const double* weights, const double* offsets, const oracle_cfg* c, double* out,
                 int32_t* counts);
int oracle_gather_stack(int t, int h, int w, int f, const double* v, int64_t rows, int l,
                        const double* weights, const double* offsets, const oracle_cfg* c,
                        double* out);
int oracle_wpsum_bwd(int t, int h, int w, int f, const double* grad_out, const int32_t* counts,
                     const double* v, int64_t rows, int l, const double* weights,
                     const double* offsets, const oracle_cfg* c, double* dv, double* dw);

/* ---- frame-alignment pipeline pieces ------------------------- */
/* flow.cpp:114-175: exhaustive block-matching SSD search, strict '<' (first hit in dy, dx
 * scan order wins ties); a, b single frames h x w x f; flow h x w x 2 (dy, dx). */
int oracle_block_match(int h, int w, int f, const double* a, const double* b, int block,
                       int radius, double* flow);
/* tensor.cpp:79-90 (inf when the inputs are identical) */
int oracle_psnr(int64_t n, const double* a, const double* b, double peak, double* out);
/* rng.hpp:30-53 GaussianStream(seed): n standard-normal draws (Box-Muller pairs) */
void oracle_gaussian_fill(uint64_t seed, int64_t n, double* out);

#ifdef __cplusplus
}
#endif
#endif
