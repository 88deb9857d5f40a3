// Host-side launch interface between the C-ABI (capi.cu) and the kernel translation units.
// Launchers return 1 when they enqueued a kernel, 0 when nothing was needed, and -1 when
// the configuration cannot be served (the caller maps that to a status).
#pragma once

#include <functional>

#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace snls_gpu {

struct GenericSearch {
    const float *q, *k, *ff, *bf;
    Dims d;
    int ws, wt, ps, topl, metric;
    double stride1;
    float beta;
    float *sims, *offsets, *chains, *weights;
    float *grid, *grid_offsets;
    int select;
    int* err;
    const float* grid_in;  // select from an already materialised grid instead of computing
};

struct TiledSearch {
    const float *q, *k, *ff, *bf;
    Dims d;
    int ws, wt, ps, topl, metric;
    float beta;
    float *sims, *offsets, *chains, *weights;
    int* err;
    int num_sms;
    float* grid;  // kFullGrid: write every window score (rows x slots) and skip selection
    int kernel;   // register plan: 0 auto, 1 region-row tiled, 2 streaming
    int band = 0;  // > 0: temporally blocked raster, bands of `band` query rows swept frame by
                   // frame (search_tiled.cu, band_row); 0: plain (t, y, x) raster
    const double* tape = nullptr;  // replay: fp64 centres (kt, ky, kx) per entry (rows = entries)
};

struct AggArgs {
    const float* v;
    const float* weights;
    const float* offsets;
    Dims d;
    int ps, topl;
    int* err;
    int wt;  // the search's temporal radius: a hint for frame-ordered traversals (offsets
             // reaching further are still served)
};

int launch_flows_check(const float* ff, const float* bf, int64_t n, int* err, cudaStream_t st);
int launch_search_generic(const GenericSearch& g, cudaStream_t st);
// Returns 0 when (ws, ps, f, topl) has no tiled instantiation (caller falls back).
// `used` (optional) receives the plan that ran: 1 tiled, 2 streaming.
int launch_search_tiled(const TiledSearch& s, cudaStream_t st, int* used);
// Query-stationary streaming variant (search_stream.cu); 0 when not instantiated.
int launch_search_stream(const TiledSearch& s, cudaStream_t st);
// replay_similarities through the tiled plan's own arithmetic (bitwise equal to its forward):
// s.tape = centres, s.grid = the rows x topl output, s.d = the query dims; 0 if not instantiated
int launch_replay_tiled(const TiledSearch& s, cudaStream_t st);
int launch_replay_stream(const TiledSearch& s, float* out, cudaStream_t st);
int launch_replay64(const float* q, const float* k, Dims d, int ps, int metric, int topl,
                    const double* centers, float* sims, cudaStream_t st);
int launch_topl(int64_t rows, int cols, const float* full, const float* full_offsets, int topl,
                float* sel, float* sel_offsets, int* err, cudaStream_t st);
int launch_emit_tape(const float* ff, const float* bf, Dims d, int wt, int topl,
                     const float* offsets, float* chains, cudaStream_t st);
int launch_tape64(const float* ff, const float* bf, Dims d, int ws, int wt, int topl, double stride1,
                  const float* offsets, double* centers, double* chains, const float* sims,
                  double* sims64, double* offsets64, cudaStream_t st);
int launch_replay(const float* q, const float* k, Dims d, int ps, int metric, int topl,
                  const float* offsets, float* sims, cudaStream_t st);

int launch_softmax(int64_t rows, int l, float beta, const float* sims, float* weights, int* err,
                   cudaStream_t st);
int launch_wpsum(const AggArgs& a, float* out, int32_t* counts, cudaStream_t st);
int launch_gather_stack(const AggArgs& a, float* out, cudaStream_t st);
// The wpsum backward's arguments (the training backward's second operator).
struct WpsumBwdArgs {
    AggArgs a;
    const float* go;
    const int32_t* counts;
    float* dv;
    float* dw;
    // deterministic mode: int64 fixed-point dV / dW sinks and their scales (device)
    unsigned long long* dvi;
    unsigned long long* dwi;
    const double* scale;
};

int launch_wpsum_bwd(const AggArgs& a, const float* grad_out, const int32_t* counts, float* dv,
                     float* dw, cudaStream_t st);
// Deterministic wpsum backward (int64 fixed point; `work` hands out scratch, zeroed there); -1 when
// the scratch is unavailable.
int launch_wpsum_bwd_det(const AggArgs& a, const float* grad_out, const int32_t* counts, float* dv,
                         float* dw, const std::function<void*(size_t)>& work, cudaStream_t st);
// its pieces, for the interleaved deterministic training backward
size_t wpsum_bwd_det_bytes(const AggArgs& a);
void wpsum_bwd_det_prep(const AggArgs& a, const float* grad_out, void* w, WpsumBwdArgs& wp, cudaStream_t st);
void wpsum_bwd_det_finish(const AggArgs& a, const WpsumBwdArgs& wp, bool dw_direct, cudaStream_t st);

// align.cu: block matching (flow.cpp:114-175) over `frames` pairs; per-frame PSNR.
int launch_block_match(const float* a, const float* b, int frames, int h, int w, int f, int block,
                       int radius, float* flow, cudaStream_t st);
int launch_psnr(const float* a, const float* b, int frames, size_t n, double peak, double* part,
                double* out, cudaStream_t st);
size_t psnr_scratch_doubles(int frames);

// `gyx`: rows * topl * 2 doubles of zeroed scratch.  Returns the number of launches.
int launch_search_bwd_impl(const float* grad, const float* offsets, const float* chains,
                           const double* centers, const double* chains64, const float* q,
                           const float* k, Dims d, int wt, int ps, int topl, int metric, float* dq,
                           float* dk, float* dff, float* dbf, double* gyx, cudaStream_t st);
// The training backward's phase 1 as one interleaved launch (search backward + wpsum backward
// blocks side by side, search_bwd.cu train_bwd_interleaved), then the search backward's flow
// route.  `wp`: the wpsum backward's arguments (dv, dw zeroed by the caller).  0 when the
// shape has no interleaved instantiation (ps 5 / 7 with F 32 / 64).
bool train_bwd_interleavable(int ps, int f);
int launch_train_bwd_interleaved(const float* grad, const float* offsets, const float* chains,
                                 const double* centers, const double* chains64, const float* q,
                                 const float* k, Dims d, int wt, int ps, int topl, int metric,
                                 float* dq, float* dk, float* dff, float* dbf, double* gyx,
                                 const WpsumBwdArgs& wp, cudaStream_t st);
int launch_search_bwd_det(const float* grad, const float* offsets, const float* chains,
                          const double* centers, const double* chains64, const float* q,
                          const float* k, Dims d, int wt, int ps, int topl, int metric, float* dq,
                          float* dk, float* dff, float* dbf,
                          const std::function<void*(size_t)>& work, cudaStream_t st,
                          const WpsumBwdArgs* wp = nullptr);  // wp: interleave the wpsum backward

}  // namespace snls_gpu
