// pf_train.h -- photon-field training internals.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "pf_field.h"

namespace pfk {

// Fixed-point scale of the table-gradient accumulators: integer atomics are
// associative, so the scatter-add of a step is deterministic (SPEC.md:440,
// "accumulation order is fixed").  2^-40 resolution, |sum| < 2^23.
constexpr double kGradFix = 1099511627776.0;  // 2^40

struct TrainParams {
    int n_pos_levels, n_dir_levels, Fp, Fd, din, H;
    FieldLevel lv[PF_FIELD_MAX_LEVELS];  // offset_halves == parameter offset (tables lead the vector)
    const float *params;                 // binary32 master parameters
    uint32_t n_pos_tab;                  // pos table parameters (dir entries start at n_pos_tab / Fp)
    uint32_t wt_off[8], b_off[8];        // transposed-weight image: W_L^T [k][o] and b_L (floats)
    int out_stride;                      // o-stride of the output layer's W^T (4)
    size_t n, ld;                        // batch, activation row stride (>= n, multiple of 4)
    const float *qx, *qw, *qg, *qt;      // x3, w_sph2, raw g, targets3 (L' space)
    float eps_rel, inv_3n;
    float *A0;                           // din rows [k][ld]: encoded inputs
    float *A;                            // H x 64 rows: a_1 .. a_H (post-ReLU)
    float *dZ;                           // (H + 1) x 64 rows: dloss/dz_0 .. dz_H
    float *loss_q;                       // per-query sum over channels of (p-t)^2/(p^2+eps)
    float *dF;                           // table-feature rows [k][ld]: dloss/dfeature (k_train_bwd -> k_train_scatter)
    unsigned long long *gtab;            // fixed-point table gradient (n_tab)
    uint8_t *touched;                    // per table entry (pos entries, then dir)
};

struct TrainPhases {
    int n;
    double v[8];
};

struct TrainState {
    bool ready = false;
    FieldDesc fd{};
    int din = 0, H = 0, Fp = 0, Fd = 0;
    size_t n_params = 0, n_tab = 0, n_pos_tab = 0, n_entries = 0;
    std::vector<FieldLevel> levels;
    uint32_t off_w[8] = {0};      // W_L offsets in the flat vector (b_L follows W_L)
    uint32_t wt_off[8] = {0}, b_off[8] = {0};
    size_t img_floats = 0;
    // Adam
    double lr = 9e-4, beta1 = 0.9, beta2 = 0.99, eps = 1e-8, decay = 0.92, decay_start = 0.7, eps_rel = 0.01;
    int decay_interval = 25;
    DevBuf params, m, v, gmlp, gtab, touched, img, offw, act, part, lossq, loss_dev;
    DevBuf bx, bw, bg, bt;        // staged batch (binary32)
    size_t act_ld = 0;
};

// Allocate / initialise the optimizer state from a flat binary32 parameter
// vector (device pointer) of the given field.
cudaError_t train_init(TrainState &S, const FieldDesc &fd, const std::vector<FieldLevel> &levels,
                       const float *params_dev, cudaStream_t st);
// One step on n queries (device pointers, binary32): forward, rMSE loss,
// backward, deterministic reductions; then Adam (if do_update) or a dense
// gradient export into grad_out / touched_out (may be null).  The loss is
// written to loss_dev[slot] (binary64, device).
cudaError_t train_step(TrainState &S, size_t n, const float *x3, const float *w2, const float *g, const float *t3,
                       uint64_t step, uint64_t total, bool do_update, float *grad_out, uint8_t *touched_out,
                       size_t loss_slot, int sms, cudaStream_t st);
// The two halves of train_step for data-parallel training: backward scales
// the loss / gradient by 1 / (3 n_global) so that summing the gradient
// buffers over ranks gives the global batch mean; finish applies Adam (or
// exports the gradient) and clears the accumulators.
cudaError_t train_backward(TrainState &S, size_t n, const float *x3, const float *w2, const float *g, const float *t3,
                           size_t n_global, size_t loss_slot, cudaStream_t st);
cudaError_t train_finish(TrainState &S, uint64_t step, uint64_t total, bool do_update, float *grad_out,
                         uint8_t *touched_out, cudaStream_t st);
// make_batch outputs (binary64 directions / targets, phase indices) -> the
// trainer's binary32 inputs: w_sph = (theta/pi, (phi+pi)/2pi), g = phase[gidx].
cudaError_t train_prep(const double *w3, const uint8_t *gidx, const double *t3d, const double *phase, int n_phases,
                       size_t n, float *w2, float *g, float *t3, cudaStream_t st);
double train_lr(const TrainState &S, uint64_t step, uint64_t total);

}  // namespace pfk
