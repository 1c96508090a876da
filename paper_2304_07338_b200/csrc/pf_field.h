// pf_field.h -- photon-field (hash grid + tcgen05 MLP) internals.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "pf_kernels.h"

namespace pfk {

struct FieldGridDesc {  // mirrors pf_hashgrid_desc
    int dims, levels, features, base_res;
    double growth;
    int log2_table;
};
struct FieldDesc {  // mirrors pf_field_desc
    FieldGridDesc pos, dir;
    int hidden_layers, width;
    double psi;
};

struct FieldLevel {
    uint32_t res;            // N_l
    uint32_t n1;             // N_l + 1 (dense stride)
    uint32_t dense;          // (N_l+1)^d <= T
    uint32_t mask;           // T - 1
    uint32_t offset_halves;  // level start in the fp16 table array (entries * F)
};

#define PF_FIELD_MAX_LEVELS 32

struct FieldParams {
    int mode;  // 0: render epilogue over hit records, 1: plain query
    int n_pos_levels, n_dir_levels;
    int K0, hidden_layers, n_wg;
    uint32_t tmem_cols, img_bytes, a_bytes;
    uint32_t off_w[8];
    uint32_t off_bias;
    float psi_log2_10;
    FieldLevel lv[PF_FIELD_MAX_LEVELS];
    const __half *tables;
    const void *img;
    // render mode
    const HitRec *hits;
    const unsigned long long *n_hits;
    void *slots;
    int slot_f64;
    double w_i;
    float g_render;
    // query mode
    size_t n_query;
    const float *qx, *qw, *qg;
    float *qout;
    int decoded;
    // split path: encode kernel -> feature tiles -> TMA-fed MLP kernel
    uint8_t *feat;     // [tile][chunk][16 KB], UMMA canonical K-major fp16
    int nch;           // 64-column chunks per tile (last one may be narrower)
    size_t row0, row_cap;  // this launch handles items [row0, row0 + row_cap)
};

struct FieldHost {
    int K0 = 0, n_pos_levels = 0, n_dir_levels = 0, fp = 0, fd = 0, hidden_layers = 0;
    double psi = 5.0;
    std::vector<uint16_t> tables;  // fp16 bits, each level padded to an even entry count
    std::vector<FieldLevel> levels;      // offset_halves into the flat fp32 parameter vector (trainer)
    std::vector<FieldLevel> enc_levels;  // offset_halves into `tables` (encoder, pair-aligned)
    std::vector<uint8_t> image;    // smem image (weights canonical fp16 + fp32 biases)
    uint32_t off_w[8] = {0};
    uint32_t off_bias = 0;
};

size_t field_grid_param_count(const FieldGridDesc &g);
size_t field_param_count(const FieldDesc &d);
const char *field_validate(const FieldDesc &d);
void field_pack(const FieldDesc &d, const float *params, FieldHost &out);
int field_launch_config(const FieldHost &h, int &n_wg, size_t &smem, size_t &a_bytes, int device);
// encode (grid-stride, full occupancy) + MLP (persistent, n_wg warpgroups)
cudaError_t launch_field(const FieldParams &P, int fp, int fd, int grid, size_t smem,
                         cudaStream_t st);
size_t field_feat_bytes(const FieldHost &h, size_t n_items);
int field_chunk_cols();  // feature-tile chunk width in columns (PF_FIELD_CW)

}  // namespace pfk
