/*
 * stab_oracle.h — CPU ORACLE (test infrastructure, NOT product code).
 *
 * A plain-C restatement of the reference stabilizer's hot path
 * (/root/reference/proj/src/{image_ops,features,flow,motion,smoothing}.cpp),
 * operation for operation, plus the RANSAC wrapper this framework adds
 * (the reference has none).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it, and only as the checker.
 *
 * Parity pin: tests/test_oracle_pin.py checks every function here against the
 * reference itself compiled from its own sources (oracle/_ref/libstabref.so,
 * see oracle/Makefile) and against tests/golden/ fixtures generated from it by
 * tests/golden/make_golden.py.  RANSAC hypothesis sampling/scoring has no
 * reference counterpart: it is pinned only against the independent C++
 * restatement in oracle/ref_glue.cpp and through iterations == 0, which must
 * reproduce the reference bit for bit.
 */
#ifndef STAB_ORACLE_H_
#define STAB_ORACLE_H_

#include "../include/stabgpu.h"

#ifdef __cplusplus
extern "C" {
#endif

size_t orc_pyramid_bytes(int w, int h, int max_levels);
int orc_build_pyramid(const uint8_t* src, int w, int h, int max_levels, stabgpu_pyramid* out);
int orc_gradients(const uint8_t* src, int w, int h, double* gx, double* gy);
int orc_min_eig_response(const uint8_t* src, int w, int h, int block_size, double* out);
int orc_detection_roi(int w, int h, double roi_margin, stabgpu_roi* out);
int orc_detect_corners(const uint8_t* src, int w, int h, const stabgpu_detect_cfg* cfg, double* xy,
                       double* score, int* n_out);
int orc_track_lk(const stabgpu_pyramid* prev, const stabgpu_pyramid* cur, const double* xy, int n,
                 const stabgpu_flow_cfg* cfg, double* out_xy, uint8_t* ok);
int orc_weed_tracks(const stabgpu_pyramid* prev, const stabgpu_pyramid* cur, const double* prev_xy,
                    const double* cur_xy, int n, const stabgpu_flow_cfg* cfg, double* keep_prev,
                    double* keep_cur, int* n_out);
int orc_estimate(const double* prev_xy, const double* cur_xy, int n, int kind,
                 stabgpu_transform* out);
int orc_rms_residual(const double* prev_xy, const double* cur_xy, int n, const stabgpu_transform* t,
                     double* out);
int orc_ransac_estimate(const double* prev_xy, const double* cur_xy, int n, int kind,
                        const stabgpu_ransac_cfg* rc, int min_tracks, int64_t frame_index,
                        stabgpu_transform* out, uint8_t* inliers, int* n_inliers);
void orc_extract_delta(const stabgpu_transform* t, stabgpu_delta* out);
void orc_delta_to_transform(double dx, double dy, double da, double dls, stabgpu_transform* out);
int orc_trajectory_corrections(const stabgpu_delta* deltas, int n, int radius,
                               stabgpu_transform* corrections);
int orc_warp_similarity(const uint8_t* src, int w, int h, const stabgpu_transform* t, uint8_t* out);
int orc_crop_resize(const uint8_t* src, int w, int h, double crop_ratio, uint8_t* out);
int orc_compose_stabilized(const uint8_t* y, const uint8_t* cb, const uint8_t* cr, int w, int h,
                           int cw, int ch, const stabgpu_transform* t, double crop_ratio,
                           uint8_t* oy, uint8_t* ocb, uint8_t* ocr);
/* run_offline semantics over a resident sequence (pipeline.cpp:182-235).
 * out_* may be NULL to skip composition (motion + planning only). */
int orc_stabilize_sequence(const uint8_t* y, const uint8_t* cb, const uint8_t* cr, int n, int w,
                           int h, int cw, int ch, const stabgpu_config* cfg, uint8_t* oy,
                           uint8_t* ocb, uint8_t* ocr, stabgpu_frame_record* records);
/* BT.601 full-range colour conversions (media_io.cpp:75-89, 568-570) and
 * psnr_pair (synth_eval.cpp:214-240). */
void orc_rgb_to_ycbcr(const uint8_t* rgb, size_t npx, uint8_t* y, uint8_t* cb, uint8_t* cr);
void orc_ycbcr_to_rgb(const uint8_t* y, const uint8_t* cb, const uint8_t* cr, size_t npx, uint8_t* rgb);
int orc_psnr_pair(const uint8_t* a, const uint8_t* b, int w, int h, double crop, double* out);
const char* orc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
