/*
 * holo_b200.h -- C ABI of the B200-native digHolo batch hot path.
 *
 * Drop-in boundary for the reference package `holopipe` (Python; no FFI of its
 * own).  Each entry point replaces one step of the
 * reference's staged engine; the citation is the reference code it replaces
 * (paths relative to /root/reference/pkg/src/holopipe/):
 *
 *   hpg_plan_create      engine.py:94-120 (_batch_plan), pipeline.py:31-44 (window_origin),
 *                        pipeline.py:62-76 (window_bin_dims/window_mask),
 *                        engine.py:191-196 (k0), pipeline.py:114-127 (recentring_phase),
 *                        pipeline.py:152-185 (field_axes, removal_phase),
 *                        hgbasis.py:42-93 (hg_profiles, BasisFields1D int16 tables)
 *   hpg_run              engine.py:389-402 (run_pipeline(0)): process_fft :135 ->
 *                        process_ifft :170 -> process_remove_tilt :222 -> extract_coefs :353,
 *                        fused into one persistent CUDA kernel
 *   hpg_fourier_full     engine.py:135-168 (process_fft full R2C plane + Fourier summary)
 *   hpg_finalize_summary analysis.py:68-94 aggregate slot + total intensity
 *   hpg_extract_coefs    engine.py:353-385 / hgbasis.py:101-116 (overlap of int16 fields)
 *   hpg_metric_partials  analysis.py:104-188 (transfer-matrix row/diag/group power sums,
 *                        Gram matrix for MDL) -- reduced across ranks by the caller
 *   hpg_coef_transform   engine.py:371-382 (LG / custom transform of the HG coefficients)
 *
 * Conventions
 *   - Every function returns an hpg_status (same integers as holopipe ErrorCode,
 *     errors.py:10-22).  Nothing throws across the boundary.
 *   - All large buffers are caller-allocated DEVICE memory; calls are ordered on
 *     the caller's cudaStream_t (passed as void*).  No allocation in hpg_run.
 *   - A plan owns only small constant tables (twiddles, window/phase tables,
 *     int16-derived basis profiles).  A plan is not thread-safe; use one per handle.
 *   - Complex values are interleaved float32 pairs (numpy complex64 layout).
 */
#ifndef HOLO_B200_H
#define HOLO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HPG_SUCCESS = 0,
  HPG_ERROR = 1,
  HPG_INVALIDHANDLE = 2,
  HPG_NULLPOINTER = 3,
  HPG_INVALIDDIMENSION = 5,
  HPG_INVALIDPOLARISATION = 6,
  HPG_INVALIDARGUMENT = 8,
  HPG_MEMORYALLOCATION = 9
} hpg_status;

typedef struct hpg_plan hpg_plan;

/* Physical description of one processing configuration (holopipe HoloConfig
 * fields, config.py:33-71, after pol locks engine.py:79-92). */
typedef struct hpg_plan_desc {
  int32_t frame_width, frame_height;  /* pixels */
  int32_t pol_count;                  /* 1 or 2 */
  int32_t fft_nx, fft_ny;             /* FFT window (pixels) */
  int32_t resolution_mode;            /* 0: IFFT at (ny,nx); 1: at the window box */
  int32_t fill_factor;                /* 1: divide bins by the pixel sinc envelope */
  int32_t group_count;                /* HG groups G (0 = fields only) */
  int32_t wavelength_count;           /* L >= 1 */
  int32_t reserved;
  double pixel_size;                  /* metres */
  double wavelength_centre;           /* metres; sets window box and mask */
  double window_radius_deg;           /* Fourier window radius (degrees) */
  const double* wavelengths;          /* [L] metres (host pointer) */
  double beam_centre[2][2];           /* [axis][pol] metres: window origin + recentring
                                         (the values process_fft saw, engine.py:141-150) */
  double tilt_deg[2][2];              /* [axis][pol] degrees: carrier bin k0 + recentring
                                         (the values process_ifft saw, engine.py:191-204) */
  double removal_tilt_deg[2][2];      /* [axis][pol] degrees: removal phase (engine.py:239-242) */
  double removal_beam_centre[2][2];   /* [axis][pol] metres: removal phase constant */
  double defocus[2];                  /* [pol] dioptre */
  double waist[2];                    /* [pol] metres */
} hpg_plan_desc;

/* Geometry a plan derived (all host values). */
typedef struct hpg_plan_info {
  int32_t wh, ww;          /* Fourier window box (rows, cols) */
  int32_t gh, gw;          /* IFFT / field grid (rows, cols) */
  int32_t col0[2], row0[2];
  int32_t mode_count;      /* M = G(G+1)/2 */
  int32_t k0[2][16][2];    /* [pol][wavelength<16][x,y] carrier bins */
} hpg_plan_info;

typedef struct hpg_batch {
  const void* frames;            /* device: frame_format elements, [frame_count][H][W] */
  int32_t frame_format;          /* 0 = float32, 1 = uint16 */
  int32_t transpose;             /* uint16 only: frames stored [W][H] */
  int64_t frame_count;           /* frames available in `frames` */
  int32_t batch_count;           /* B (output rows) */
  int32_t avg_count;             /* A (frames averaged per row) */
  const int32_t* members;        /* device [B*A] frame of (row, member); NULL = row*A+member */
  const int32_t* wl_of_row;      /* device [B] wavelength index; NULL = 0 */
  const void* batch_cal;         /* device complex64 [cal_pols][cal_batch] or NULL */
  int32_t cal_pols, cal_batch;
  const void* ref_cal;           /* device complex64 [ref_cal_count][P][gh][gw] or NULL */
  int32_t ref_cal_count;
  int32_t row_offset;            /* global index of row 0 (multi-GPU shards, pipelined chunks):
                                    batch calibration uses entry (row_offset + row) mod cal_batch,
                                    as the reference indexes it by the global row (engine.py:247-249) */
  /* Optional frame-buffer layout override (window-packed uploads): when
   * layout_width > 0 the buffer holds [frame_count][layout_height][layout_width]
   * and pol q's FFT window starts at (layout_col0[q], layout_row0[q]). */
  int32_t layout_width, layout_height;
  int32_t layout_col0[2], layout_row0[2];
} hpg_batch;

typedef struct hpg_outputs {
  int16_t* field_r;              /* [B][P][gh][gw] */
  int16_t* field_i;              /* [B][P][gh][gw] */
  float* field_scale;            /* [B][P] */
  void* coefs;                   /* complex64 [B][P*M] or NULL (skip the overlap) */
  void* raw_fields;              /* complex64 [B][P][gh][gw] tilt-removed, unquantised, or NULL */
  void* windows;                 /* complex64 [B][P][wh][ww] masked Fourier windows, or NULL */
  float* field_params;           /* [7][P][param_slots] per-row field-plane summary or NULL */
  int32_t param_slots;           /* B*A+1 in the reference layout */
  int32_t reserved;
  void* workspace;               /* device scratch, hpg_workspace_size() bytes */
  size_t workspace_bytes;
} hpg_outputs;

/* hpg_run flags */
#define HPG_FLAG_SUMMARY 1u      /* per-row field summary + aggregate partials */
#define HPG_FLAG_GENERIC 2u      /* diagnostic: force the generic (any-size) kernel */
#define HPG_FLAG_SIMT 4u         /* diagnostic: specialised kernel without tensor cores */
#define HPG_FLAG_TC 8u           /* tcgen05 row-pass kernel (warp-specialised) where it applies */
#define HPG_FLAG_TC2 16u         /* two-kernel path: row + column DFT on tcgen05, then the field kernel
                                    (chosen automatically for large batches; HPG_FLAG_SIMT opts out) */
#define HPG_FLAG_SIMT_OVERLAP 32u  /* diagnostic: HG overlap on SIMT instead of tcgen05 in the fast kernel */

int hpg_version(void);
int hpg_plan_create(const hpg_plan_desc* desc, hpg_plan** out);
int hpg_plan_destroy(hpg_plan* plan);
int hpg_plan_get_info(const hpg_plan* plan, hpg_plan_info* info);
/* float32 field axes in metres, [gw] and [gh] (pipeline.py:152-160) */
int hpg_plan_get_axes(const hpg_plan* plan, float* x_axis, float* y_axis);
/* dequantised basis profiles float32 [P][G][gw] and [P][G][gh] (hgbasis.py:89-93) */
int hpg_plan_get_basis(const hpg_plan* plan, float* hx, float* hy);

int hpg_workspace_size(const hpg_plan* plan, int32_t batch_count, uint32_t flags, size_t* bytes);
int hpg_run(const hpg_plan* plan, const hpg_batch* batch, const hpg_outputs* out,
            uint32_t flags, void* stream);
/* Number of kernels the calling thread's last hpg_run launched (0 after an error); the bench
 * reports it as gpu_launches.  No reference counterpart (instrumentation). */
int hpg_last_launch_count(void);
/* Aggregate slot (index B of field_params) and total intensity [gh][gw] from the
 * partials hpg_run(HPG_FLAG_SUMMARY) left in the workspace. */
int hpg_finalize_summary(const hpg_plan* plan, const hpg_batch* batch, const hpg_outputs* out,
                         float* total_intensity, void* stream);

/* Full R2C plane complex64 [F][P][ny][nx/2+1] of frames f = 0..F-1 (pipeline.py:47-59);
 * frames->frames/frame_format/transpose/frame_count (+ layout override) are used. 
 * workspace: hpg_workspace_size() bytes (used only for windows too large for shared memory). */
int hpg_fourier_full(const hpg_plan* plan, const hpg_batch* frames, void* plane, void* workspace,
                     size_t workspace_bytes, void* stream);

/* Seven analysis parameters (analysis.py:39-94) per (frame, pol) of complex
 * data [count][P][h][w] with fp64 device axes x[w], y[h], plus the aggregate
 * slot (index `count`) from the summed intensity.  params [7][P][slots]
 * (slots >= count+1); total_intensity [h][w] or NULL; pol_intensity fp64
 * [P][h][w] batch sums per pol or NULL (align.py:53-55).  The workspace needs
 * hpg_plane_summary_workspace() bytes.  Deterministic for a given input. */
size_t hpg_plane_summary_workspace(int64_t count, int32_t P, int32_t h, int32_t w);
int hpg_plane_summary(const void* data, int64_t count, int32_t P, int32_t h, int32_t w,
                      const double* x_axis, const double* y_axis, float* params, int32_t slots,
                      float* total_intensity, double* pol_intensity, void* workspace,
                      size_t workspace_bytes, void* stream);

/* Batch-summed intensity per pol of dequantised int16 fields, fp64
 * [P][h][w] = sum_b |(fr + i fi) / scale|^2 (holopipe/align.py:166-169). */
int hpg_field_intensity(const int16_t* field_r, const int16_t* field_i, const float* field_scale,
                        int32_t batch_count, int32_t P, int32_t h, int32_t w, double* out, void* stream);

/* Reference-wave calibration correction (holopipe/engine.py:276-335): from the
 * tilt-removed, unquantised calibration fields a [n] (and b [n] or NULL, the
 * second real part of a complex calibration, so proc = a + i b) computes
 * applied = conj(proc) / max(|proc|^2, 1e-6) in fp64, stored complex64 [n].
 * The fields themselves come from hpg_run(raw_fields) on the calibration frames. */
int hpg_ref_calibration_finish(const void* a, const void* b, int64_t n, void* applied, void* stream);

/* Coefficients of already-quantised fields (engine.py:353-370): fields int16
 * [B][P][gh][gw] + scale [B][P] -> coefs complex64 [B][P*M]. */
int hpg_extract_coefs(const hpg_plan* plan, const int16_t* field_r, const int16_t* field_i,
                      const float* field_scale, int32_t batch_count, void* coefs, void* stream);

/* Transfer-matrix partial sums for the nine metrics (analysis.py:104-188).
 * Virtual matrix A (rows x cols): row r holds coefs[row_ids[r]][j] for
 * col_offset[r] <= j < col_offset[r] + col_count[r] (NULL offsets = all
 * columns) and zero elsewhere -- this expresses the pol-independent block
 * layout (analysis.py:117-123).  Outputs are fp64 device arrays; diag/group
 * entries of rows without a diagonal element are -1.  gram (optional,
 * complex128) is A A^H when gram_rows != 0 else A^T conj(A^T)^H, i.e. the
 * smaller Gram matrix whose eigenvalues are the squared singular values. */
typedef struct hpg_metric_args {
  const void* coefs;             /* complex64 [*][ld] */
  int32_t rows, cols;
  const int32_t* row_ids;        /* [rows] */
  const int32_t* col_offset;     /* [rows] or NULL */
  const int32_t* col_count;      /* [rows] or NULL */
  const int32_t* labels;         /* [cols] (pol, mode group) label or NULL */
  int32_t ndiag;                 /* min(global rows, cols) */
  int32_t diag_offset;           /* global index of virtual row 0 */
  int32_t gram_rows;
  int32_t ld;                    /* row stride of coefs (0 = cols) */
  double* row_power;             /* [rows] */
  double* diag_power;            /* [rows] */
  double* group_power;           /* [rows] */
  void* gram;                    /* complex128 [n][n] or NULL */
} hpg_metric_args;

int hpg_metric_partials(const hpg_metric_args* args, void* stream);

/* LG / custom basis transform of the HG coefficients (holopipe/engine.py:371-382):
 * out[r][p][o] = sum_{m < use} T[o][m] coefs[r][p][m], accumulated in fp64 like the
 * reference's complex128 einsum.  coefs complex64 [rows][pols][modes_in], transform
 * complex128 [modes_out][ld] (row o, column m), out complex64 [rows][pols][modes_out].
 * block_diagonal != 0 declares T block-diagonal by HG mode group (conj(T_LG),
 * hgbasis.py:126-152): output o of group g then reads only that group's inputs. */
int hpg_coef_transform(const void* coefs, int64_t rows, int32_t pols, int32_t modes_in, const void* transform,
                       int32_t modes_out, int32_t use, int32_t ld, int32_t block_diagonal, void* out,
                       void* stream);

/* Host -> device upload of only the FFT windows of F frames (the bytes the
 * pipeline reads, holopipe/pipeline.py:47-54): one cudaMemcpy3DAsync per pol
 * from the host frame buffer ([F][H][W], frame_format elements; pinned memory
 * for asynchronous copies) into dst, packed as [F][ny][P*nx].  Process the
 * packed buffer with hpg_batch.layout_width = P*nx, layout_height = ny,
 * layout_col0[q] = q*nx, layout_row0[q] = 0. */
int hpg_upload_windows(const hpg_plan* plan, const void* host_frames, int32_t frame_format,
                       int64_t frame_count, void* dst, void* stream);

/* Page-lock a pageable host frame buffer in place (cudaHostRegister) so that hpg_upload_windows runs at
 * pinned-memory speed; holopipe re-reads the caller's buffer on every run (holopipe/frames.py:40-47), so a
 * caller registers it once and unregisters it when the buffer is replaced.  A range that is already
 * page-locked returns HPG_INVALIDARGUMENT and is left as it is (no sticky runtime error either way). */
int hpg_host_register(void* ptr, size_t bytes);
int hpg_host_unregister(void* ptr);

const char* hpg_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* HOLO_B200_H */
