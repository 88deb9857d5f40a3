/* snls_cuda.h -- C-ABI of the B200 (sm_100a) Shifted Non-Local Search library.
 *
 * This is the thin shim the reference's C++ API calls through: the drop-in adapter
 * (paper_2309_16849_b200/host/snls_gpu_search.cpp, snls_gpu_aggregate.cpp) implements the
 * reference's `snls::` entry points (search.hpp:126-158, aggregate.hpp:22-85) by converting
 * the fp64 host containers to fp32 device buffers and calling the functions below.  The
 * Python tests and bench.py call the same functions through ctypes.
 *
 * Conventions
 *  - extern "C", no exceptions, no STL, no torch types.  Every function returns an
 *    snls_status; the message of the last failure on the calling thread is
 *    snls_last_error().  Validation failures carry the reference's exact messages
 *    (ConfigError -> SNLS_ECONFIG, DomainError -> SNLS_EDOMAIN).
 *  - Tensor arguments are DEVICE pointers to fp32 (counts: int32), row-major with the
 *    reference's layouts: videos T x H x W x F (F fastest, tensor.hpp:17-31), flows
 *    T x H x W x 2 holding (dy, dx) (flow.hpp:12-28), query rows (t, y, x) with x fastest
 *    on the grid {0, stride0, ...} (search.hpp:47-55).
 *  - Work is enqueued on the context's stream and returns immediately.  Domain errors that
 *    only the device can see (non-finite flows, offsets leaving the clip, non-finite
 *    softmax inputs) are latched in the context and reported by snls_ctx_sync_check().
 *
 * The search tape.  The reference's SearchTape (search.hpp:89-110) stores absolute key
 * centres and absolute chain positions in fp64.  The device tape stores what fp32 can hold
 * exactly enough: `offsets` (dt, ky-qy, kx-qx) per selected entry (centres = query + offset)
 * and `chains` rows x L x max(wt-1,0) x 6 links (pos_y-qy, pos_x-qx, J00, J01, J10, J11),
 * positions relative to the query pixel.
 */
#ifndef SNLS_CUDA_H
#define SNLS_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SNLS_CUDA_ABI_VERSION 1

typedef enum {
    SNLS_OK = 0,
    SNLS_ECONFIG = 1, /* snls::ConfigError (errors.hpp:9-12) */
    SNLS_EDOMAIN = 2, /* snls::DomainError (errors.hpp:14-17) */
    SNLS_ECUDA = 3,   /* CUDA runtime failure, no device, or the kernels are not loadable */
    SNLS_EARG = 4,    /* null or inconsistent argument at the C boundary */
    SNLS_EIO = 5      /* snls::IoError (errors.hpp): file formats */
} snls_status;

typedef enum { SNLS_METRIC_IP = 0, SNLS_METRIC_L2 = 1 } snls_metric; /* search.hpp:12 */

typedef enum { SNLS_MODE_FUSED = 0, SNLS_MODE_FULLGRID = 1 } snls_mode; /* search.hpp:37 */

/* snls::SearchConfig (search.hpp:17-35), field for field. */
typedef struct {
    int ws;               /* spatial window size, odd */
    int wt;               /* temporal radius */
    int ps;               /* patch size, odd */
    int stride0;          /* query stride */
    double stride1;       /* key stride (fractional allowed) */
    int topl;             /* neighbours kept per query */
    int metric;           /* snls_metric */
    double softmax_scale; /* beta for the fused softmax epilogue / softmax_rows */
} snls_config;

typedef struct {
    int t, h, w, f;
} snls_dims;

typedef struct snls_ctx snls_ctx;

/* ---- host-only helpers (no device needed) ------------------------------------------ */
int snls_abi_version(void);
const char* snls_last_error(void);
/* SearchConfig::validate (search.cpp:21-32) */
int snls_validate_config(const snls_config* cfg);
/* QueryGrid::over (search.cpp:43-50) */
int snls_query_grid(snls_dims dims, int stride0, int64_t* rows, int* nh, int* nw);
/* UniformStream(seed).next_in(lo, hi) (rng.hpp:12-24) rounded to fp32, into HOST memory;
 * the synthetic-input generator of run_benchmark (harness.cpp:242-253). */
int snls_uniform_fill_f32(uint64_t seed, double lo, double hi, int64_t n, float* host_out);

/* ---- context: one per (device, stream) --------------------------------------------- */
int snls_ctx_create(int device, void* cuda_stream, snls_ctx** out);
int snls_ctx_destroy(snls_ctx* ctx);
int snls_ctx_set_stream(snls_ctx* ctx, void* cuda_stream);
int snls_ctx_get_stream(snls_ctx* ctx, void** cuda_stream);
/* Synchronise the stream; report (and clear) latched device-side domain errors. */
int snls_ctx_sync_check(snls_ctx* ctx);
/* Number of kernels this context has launched (evidence for bench.py's gpu_launches). */
int snls_ctx_launch_count(snls_ctx* ctx, int64_t* out);
/* Kernel path the last search_fwd took: 0 generic per-slot, 1 region-row tiled
 * (stride1 == 1), 2 full grid, 3 query-stationary streaming (stride1 == 1). */
int snls_ctx_last_search_path(snls_ctx* ctx, int* out);
/* Force the generic per-slot search path (1) or allow the tiled one (0, default). */
int snls_ctx_force_generic(snls_ctx* ctx, int on);
/* stride1 == 1 register plan: 0 auto (= region-row tiled), 1 region-row tiled,
 * 2 query-stationary streaming (ps in {3, 7}, F in {32, 64}; else tiled).  Results agree to the parity tolerance; each plan is
 * deterministic and tie-exact on its own. */
int snls_ctx_set_search_kernel(snls_ctx* ctx, int kind);
/* Raster of the tiled search: -1 auto (temporally blocked in bands of query rows when the
 * key frames a query frame reads overflow ~1/3 of L2, e.g. c5), 0 plain (t, y, x), > 0 that
 * many query rows per band.  Results are identical either way (each query is independent). */
int snls_ctx_set_search_band(snls_ctx* ctx, int band);

/* ---- device memory through the context (so C++ callers need no CUDA headers) --------- */
int snls_device_alloc(snls_ctx* ctx, uint64_t bytes, void** out);
int snls_device_free(snls_ctx* ctx, void* ptr);
/* Stream-ordered copies; snls_copy_d2h returns after the data has landed. */
int snls_copy_h2d(snls_ctx* ctx, void* dst_device, const void* src_host, uint64_t bytes);
int snls_copy_d2h(snls_ctx* ctx, void* dst_host, const void* src_device, uint64_t bytes);
/* Stream-ordered copy that does not wait (kind 1 H2D, 2 D2H, 3 D2D; pinned host memory for
 * true asynchrony), and events on the context's stream, so C++ callers can pipeline host
 * work against transfers without CUDA headers. */
int snls_copy_async(snls_ctx* ctx, void* dst, const void* src, uint64_t bytes, int kind);
typedef struct snls_event snls_event;
int snls_event_create(snls_ctx* ctx, snls_event** out);
int snls_event_record(snls_ctx* ctx, snls_event* ev);
int snls_event_sync(snls_event* ev);
int snls_event_destroy(snls_event* ev);

/* ---- search (search.hpp) ------------------------------------------------------------ */
/* Replaces snls::shifted_nls_forward (search.hpp:126-128; search.cpp:414-421).
 * fflow/bflow may be NULL for zero flows (snls::nls_forward, search.hpp:131-132).
 * Outputs: sims rows x L (best first), offsets rows x L x 3, optional chains (see above,
 * NULL to skip), optional weights rows x L = softmax_rows(sims, cfg.softmax_scale) fused in
 * the epilogue (NULL to skip).  mode SNLS_MODE_FULLGRID materialises the rows x
 * window_slots score grid in a context workspace before selection, as the reference's
 * kFullGrid does (search.cpp:329-410); results are identical to SNLS_MODE_FUSED. */
int snls_search_fwd(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, const float* q,
                    const float* k, const float* fflow, const float* bflow, int mode,
                    float* sims, float* offsets, float* chains, float* weights);

/* Frame-range form used by frame sharding: only the query rows of frames [t0, t1) are
 * searched (outputs hold those rows, rows = (t1-t0)*nh*nw); q/k/flows are the full `dims.t`
 * frames the caller holds (a shard's slab incl. its wt-frame halo), and key frames outside
 * [0, dims.t) are off-clip exactly as in search.cpp:300. */
int snls_search_fwd_frames(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, int t0, int t1,
                           const float* q, const float* k, const float* fflow, const float* bflow,
                           int mode, float* sims, float* offsets, float* chains, float* weights);

/* The pre-selection score grid rows x window_slots (-inf on off-clip frames) and its
 * offsets rows x window_slots x 3, as full_grid_forward builds it (search.cpp:351-376). */
int snls_search_grid(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, const float* q,
                     const float* k, const float* fflow, const float* bflow, float* grid,
                     float* grid_offsets);

/* Replaces snls::top_l (search.hpp:137-138; search.cpp:430-468). */
int snls_topl(snls_ctx* ctx, int64_t rows, int cols, const float* full,
              const float* full_offsets, int topl, float* sel, float* sel_offsets);

/* Replaces snls::replay_similarities (search.hpp:157-158; search.cpp:470-493) from the fp32
 * device tape: the generic per-slot arithmetic at query + offset (agrees with the forward to
 * the fp32 tolerance). */
int snls_replay(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, const float* q,
                const float* k, const float* offsets, float* sims);
/* replay_similarities from the fp64 tape (centres, snls_search_tape64 / the reference's
 * SearchTape) through a search plan's OWN per-slot arithmetic -- bitwise equal to that plan's
 * forward (search.cpp:470-493, test_search.cpp:539-553): plan 0 generic, 1 region-row tiled,
 * 2 streaming, -1 the plan snls_search_fwd takes for this configuration and context. */
int snls_replay64(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, int t0, int t1,
                  const float* q, const float* k, const double* centers, int plan, float* sims);

/* Replaces snls::shifted_nls_backward (search.hpp:151-153; search.cpp:671-711).
 * Gradients are accumulated with atomics (the reference's non-deterministic mode); the
 * four outputs are overwritten (zeroed first).  dfflow/dbflow T x H x W x 2. */
int snls_search_bwd(snls_ctx* ctx, const snls_config* cfg, snls_dims dims,
                    const float* grad_sims, const float* offsets, const float* chains,
                    const float* q, const float* k, float* dq, float* dk, float* dfflow,
                    float* dbflow);

/* Frame-range form (frame sharding, reverse halo): the tape rows of query frames [t0, t1)
 * only (grad_sims / offsets / chains hold those rows); dq, dk, dfflow, dbflow cover all
 * dims.t frames of the caller's slab -- the parts in halo frames are partial sums the owner
 * of those frames adds (paper_2309_16849_b200/shard.py reverse_exchange_add). */
int snls_search_bwd_frames(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, int t0, int t1,
                           const float* grad_sims, const float* offsets, const float* chains,
                           const float* q, const float* k, float* dq, float* dk, float* dfflow,
                           float* dbflow);

/* General backward (search.hpp:151-153; search.cpp:499-711) over either tape form:
 *  - the device tape: offsets rows x L x 3 fp32 and (wt > 1) relative fp32 chains, or
 *  - the reference's own SearchTape (search.hpp:89-110): `centers` rows x L x 3 fp64
 *    absolute (kt, ky, kx) and (wt > 1) `chains64` rows x L x max(wt-1,0) x 6 fp64 with
 *    absolute link positions -- used when `centers` is non-NULL (offsets/chains may then
 *    be NULL).  The fp64 tape keeps the key-position fractions at fp64 accuracy, which the
 *    flow gradients amplify (d(dS/dy)/dy ~ sum (dk/dy)^2).
 * Query rows of frames [t0, t1) as in snls_search_bwd_frames.  flags:
 *  SNLS_BWD_DETERMINISTIC -- the reference's default deterministic mode (search.cpp:687-696):
 *  every accumulation is int64 fixed point (scale = a power of two from a per-call bound),
 *  so the result is bitwise identical on every run; otherwise fp32/fp64 atomics. */
#define SNLS_BWD_DETERMINISTIC 1
int snls_search_bwd_ex(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, int t0, int t1,
                       const float* grad_sims, const float* offsets, const float* chains,
                       const double* centers, const double* chains64, const float* q,
                       const float* k, float* dq, float* dk, float* dfflow, float* dbflow,
                       int flags);

/* The reference's fp64 SearchTape (search.hpp:89-110) from the device tape: for the query
 * rows of frames [t0, t1), absolute key centres (kt, ky, kx) rows x L x 3 and (wt > 1)
 * absolute chain links rows x L x max(wt-1,0) x 6, recomputed in fp64 from the flows as
 * emit_row does (search.cpp:207-234).  fflow/bflow NULL = zero flows (nls_forward). */
int snls_search_tape64(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, int t0, int t1,
                       const float* fflow, const float* bflow, const float* offsets,
                       double* centers, double* chains64);
/* The whole SearchResult in the reference's fp64 layout from one device result (the C++
 * drop-in downloads these directly): sims64 = double(sims), offsets64 = (dt, ky-qy, kx-qx)
 * and centres / chains as snls_search_tape64 (exact fp64 positions).  Any fp64 output may
 * be NULL. */
int snls_search_results64(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, int t0, int t1,
                          const float* fflow, const float* bflow, const float* sims,
                          const float* offsets, double* sims64, double* offsets64,
                          double* centers, double* chains64);

/* ---- frame sharding across GPUs: shard plan + NCCL halos -------
 * One video of T frames over `world` ranks: rank r owns query frames [a, b) (balanced
 * contiguous split) and holds the slab [lo, hi) = [a-wt, b+wt) n [0, T) of K / V / flows; the
 * wt-frame halo moves between owners by NCCL point-to-point send/recv (search.cpp:84-101,
 * 300; wpsum writes only the query's own frame, aggregate.cpp:197-198).  Host-only plan:
 * out4 = {a, b, lo, hi}; transfers: per message the peer, frames [lo, hi) and recv (1: from
 * the peer into my slab, 0: my frames to the peer), peers ascending, recv before send. */
int snls_shard_plan(int T, int world, int rank, int wt, int* out4);
int snls_shard_transfers(int T, int world, int rank, int wt, int capacity, int* peer, int* lo,
                         int* hi, int* recv, int* count);
typedef struct snls_comm snls_comm;
/* NCCL is loaded at first use (libnccl.so.2 already in the process, else the system one).
 * Rank 0 makes the 128-byte id, the caller distributes it (any out-of-band channel), every
 * rank calls snls_comm_init with its context (device) -- collective over the ranks. */
int snls_comm_unique_id(void* id_out);
int snls_comm_init(snls_ctx* ctx, const void* unique_id, int rank, int world, snls_comm** out);
int snls_comm_destroy(snls_comm* comm);
int snls_comm_info(snls_comm* comm, int* nranks, int* nccl_version);
/* Forward halo: fill the halo frames of `nslabs` persistent frame-major DEVICE slabs [lo, hi)
 * (owned frames in place; frame_bytes per slab; pass aliased slabs once) with one grouped
 * ncclSend/ncclRecv set on the communicator's stream, ordered after the context's stream.
 * Returns at once: enqueue the interior frames (no halo needed), then snls_halo_wait orders
 * the context's stream after the transfer (no host block). */
int snls_halo_exchange_async(snls_comm* comm, int T, int wt, int nslabs, void* const* slabs,
                             const int64_t* frame_bytes);
int snls_halo_wait(snls_comm* comm);
/* Backward halo: partial gradients in my halo frames go to their owners; the partial sums
 * the peers hold for my owned frames are received and added in place (fp32 slabs,
 * frame_elems floats per frame).  Joined into the context's stream on return. */
int snls_reverse_halo_add(snls_comm* comm, int T, int wt, int nslabs, float* const* slabs,
                          const int64_t* frame_elems);
/* NCCL self-check on one device: grouped send/recv of `bytes` from src to dst with this rank
 * as its own peer, joined into the context's stream. */
int snls_comm_loopback(snls_comm* comm, const void* src, void* dst, uint64_t bytes);

/* ---- aggregate (aggregate.hpp) ------------------------------------------------------ */
/* Replaces snls::softmax_rows (aggregate.hpp:22; aggregate.cpp:16-37). */
int snls_softmax_rows(snls_ctx* ctx, int64_t rows, int l, double beta, const float* sims,
                      float* weights);

/* Replaces snls::wpsum (aggregate.hpp:53-54; deterministic gather, aggregate.cpp:124-203).
 * out T x H x W x F, counts T x H x W (the AggTape, aggregate.hpp:27-36). */
int snls_wpsum_fwd(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, const float* v,
                   const float* weights, const float* offsets, float* out, int32_t* counts);

/* Frame-range form: output frames [t0, t1) only (out (t1-t0) x H x W x F, counts
 * (t1-t0) x H x W), from the weights/offsets of those frames' query rows; v holds all
 * dims.t frames (wpsum writes only into the query's own frame, aggregate.cpp:197-198). */
int snls_wpsum_fwd_frames(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, int t0, int t1,
                          const float* v, const float* weights, const float* offsets, float* out,
                          int32_t* counts);

/* Replaces snls::gather_stack (aggregate.hpp:71-73; aggregate.cpp:285-347).
 * out L x T x H x W x F. */
int snls_gather_stack(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, const float* v,
                      const float* weights, const float* offsets, float* out);

/* Replaces snls::wpsum_backward (aggregate.hpp:83-85; aggregate.cpp:412-460).
 * dv T x H x W x F, dweights rows x L; both overwritten. */
int snls_wpsum_bwd(snls_ctx* ctx, const snls_config* cfg, snls_dims dims,
                   const float* grad_out, const int32_t* counts, const float* v,
                   const float* weights, const float* offsets, float* dv, float* dweights);

/* Frame-range form: grad_out / counts hold output frames [t0, t1), weights / offsets / dw
 * the rows of those frames; v and dv cover all dims.t frames (dv in halo frames: partial
 * sums for their owner). */
int snls_wpsum_bwd_frames(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, int t0, int t1,
                          const float* grad_out, const int32_t* counts, const float* v,
                          const float* weights, const float* offsets, float* dv, float* dweights);
/* wpsum_backward with flags: SNLS_BWD_DETERMINISTIC = the reference's default
 * ExecPolicy::deterministic (aggregate.cpp:439-450, dV gathered in a fixed order): here int64
 * fixed-point accumulation, bitwise identical run to run.  0 = atomics (aggregate.cpp:451-458). */
int snls_wpsum_bwd_ex(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, int t0, int t1,
                      const float* grad_out, const int32_t* counts, const float* v,
                      const float* weights, const float* offsets, float* dv, float* dweights,
                      int flags);

/* The whole backward of search -> softmax weights -> wpsum in one call: wpsum_backward (dv,
 * dweights from grad_out / counts) then shifted_nls_backward (dq, dk, dfflow, dbflow; tape =
 * offsets + chains or fp64 centres + chains64 as in snls_search_bwd_ex; flags as there). */
int snls_train_bwd(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, const float* grad_sims,
                   const float* grad_out, const int32_t* counts, const float* offsets,
                   const float* chains, const double* centers, const double* chains64,
                   const float* q, const float* k, const float* v, const float* weights, float* dq,
                   float* dk, float* dv, float* dweights, float* dfflow, float* dbflow, int flags);

/* ---- frame alignment ------------------------------------------
 * Replaces snls::estimate_flow_block_matching (flow.hpp:48-49; flow.cpp:114-175) for
 * dims.t frame pairs at once: a[t] -> b[t] (DEVICE, T x H x W x F), flow T x H x W x 2
 * (dy, dx) per pixel of each block; strict '<' in (dy, dx) scan order, sums in fp64. */
int snls_block_match(snls_ctx* ctx, snls_dims dims, const float* a, const float* b, int block,
                     int radius, float* flow);
/* psnr (tensor.cpp:79-90) of each frame of a vs b (DEVICE); dims.t values to HOST memory. */
int snls_psnr_frames(snls_ctx* ctx, snls_dims dims, const float* a, const float* b, double peak,
                     double* psnr_host);
/* add_gaussian_noise (tensor.cpp:92-99) with GaussianStream(seed) (rng.hpp:30-53), HOST
 * buffers: out = float(in + sigma * g) with the stream's fp64 draws (bitwise). */
int snls_gaussian_noise_f32(uint64_t seed, double sigma, int64_t n, const float* in, float* out);
/* snls::align_frames (harness.hpp:61-62; harness.cpp:72-154) over HOST buffers:
 * clean T x H x W x F; flow_source 0 zero, 1 provided ((T-1) x H x W x 2), 2 block
 * matching (bm_block, bm_radius); outputs aligned (T-1) x H x W x F, top1_offsets
 * rows x 3 (may be NULL), used_flow (T-1) x H x W x 2 (may be NULL), frame_psnr T-1. */
int snls_align_frames(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, const float* clean,
                      double sigma, uint64_t seed, int flow_source, const float* provided_flow,
                      int bm_block, int bm_radius, float* aligned, float* top1_offsets,
                      float* used_flow, double* frame_psnr);

/* ---- on-disk formats, host only ---------------------------------
 * .stnt raw tensors (load_raw / save_raw, video_io.cpp:52-117) and Middlebury .flo
 * (read_flo / write_flo, flow.cpp:53-112), same checks and messages (IoError -> SNLS_EIO). */
int snls_raw_info(const char* path, snls_dims* dims, int* elem_width);
int snls_raw_read(const char* path, float* out, int64_t capacity);      /* t*h*w*f floats */
int snls_raw_write(const char* path, snls_dims dims, const float* data, int elem_width);
int snls_flo_read(const char* path, int* h, int* w, float* flow_or_null); /* h x w x (dy, dx) */
int snls_flo_write(const char* path, int h, int w, const float* flow);

/* ---- host-buffer pipeline (the search -> softmax_rows -> wpsum core of align_frames /
 * run_benchmark, harness.cpp:105-154, 242-283, over HOST memory) ---------------------
 * One call copies the clip in frame by frame on a copy stream, runs search (+ fused
 * softmax) and wpsum per chunk of query frames on two compute streams as soon as the
 * frames each chunk can reach have landed (qt + dt, |dt| <= wt), and copies each chunk's
 * results back on a result stream: transfers overlap the kernels.  Synchronous: returns
 * when all results are in host memory and the device error latch has been checked (domain
 * errors as snls_ctx_sync_check).  The whole call is ordered after, and joined back into,
 * the context's stream. */
typedef struct snls_pipeline snls_pipeline;
/* Pin / unpin caller memory (cudaHostRegister) so the pipeline's copies run asynchronously. */
int snls_host_register(void* host_ptr, uint64_t bytes);
int snls_host_unregister(void* host_ptr);
/* Device buffers for a clip of `dims` under `cfg`; chunk_frames query frames per chunk. */
int snls_pipeline_create(snls_ctx* ctx, const snls_config* cfg, snls_dims dims, int chunk_frames,
                         snls_pipeline** out);
int snls_pipeline_destroy(snls_pipeline* p);
/* q, k, v HOST T x H x W x F (k and v may alias q: each distinct buffer is copied once);
 * fflow, bflow HOST T x H x W x 2, or both NULL (nls_forward).  Outputs HOST, each may be
 * NULL to skip it: sims rows x L, offsets rows x L x 3, weights rows x L, out T x H x W x F,
 * counts T x H x W. */
int snls_pipeline_run(snls_pipeline* p, const float* q, const float* k, const float* v,
                      const float* fflow, const float* bflow, float* sims, float* offsets,
                      float* weights, float* out, int32_t* counts);
/* Streaming form for a sequence of clips: submit enqueues and returns (three buffer slots,
 * at most three clips in flight -- a fourth submit first waits for the oldest), so the next
 * clip's H2D and head overlap this clip's compute and D2H tail.  wait blocks until the
 * oldest submitted clip's results are in host memory.  Its host buffers must stay valid
 * and untouched until then.  A device-side domain error may surface one wait early. */
int snls_pipeline_submit(snls_pipeline* p, const float* q, const float* k, const float* v,
                         const float* fflow, const float* bflow, float* sims, float* offsets,
                         float* weights, float* out, int32_t* counts);
int snls_pipeline_wait(snls_pipeline* p);

#ifdef __cplusplus
}
#endif
#endif /* SNLS_CUDA_H */
