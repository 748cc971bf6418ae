/*
 * stabgpu.h — C ABI of the B200-native stabilization hot path (libstabgpu.so).
 *
 * Every entry point replaces one function of the reference C++ stage API
 * (namespace `stab`, /root/reference/proj/include/stab/ headers); the citation
 * next to each declaration names the interface it stands in for.  Plain
 * pointers and sizes only: no C++ or torch types cross this boundary, and
 * no exception crosses it either — every call returns a stabgpu_status whose
 * values map 1:1 onto the reference exception hierarchy (errors.hpp:9-41).
 * The message of the last failure on the calling thread is returned by
 * stabgpu_last_error().
 *
 * Buffer conventions
 *   - "host" pointers are caller-owned CPU memory (pageable or pinned);
 *   - "dev" pointers are CUDA device pointers on the context's device;
 *   - images are row-major uint8 with pitch == width (GrayFrame,
 *     frame.hpp:16-30); points are interleaved (x, y) doubles (Point2,
 *     frame.hpp:36-39).
 * The per-stage calls are stream-ordered on the context stream and
 * synchronous at return (the reference functions are pure and blocking).
 * The sequence calls (stabgpu_stabilize_sequence*) are the throughput path.
 */
#ifndef STABGPU_H_
#define STABGPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: errors.hpp:9-41 ---------------------------------- */
typedef enum stabgpu_status {
    STABGPU_OK = 0,
    STABGPU_INVALID_INPUT = 1,     /* InvalidInputError      errors.hpp:14-17 */
    STABGPU_INVALID_CONFIG = 2,    /* InvalidConfigError     errors.hpp:19-22 */
    STABGPU_INVALID_TRANSFORM = 3, /* InvalidTransformError  errors.hpp:24-27 */
    STABGPU_DEGENERATE_INPUT = 4,  /* DegenerateInputError   errors.hpp:29-32 */
    STABGPU_SEQUENCING = 5,        /* SequencingError        errors.hpp:34-37 */
    STABGPU_IO = 6,                /* IoError                errors.hpp:39-42 */
    STABGPU_CUDA = 7               /* device / driver failure (no reference analogue) */
} stabgpu_status;

#define STABGPU_MIN_FRAME_DIM 16 /* kMinFrameDim, frame.hpp:12 */
#define STABGPU_MAX_LEVELS 16    /* pyramid levels a context can hold */
#define STABGPU_MAX_RADIUS 31    /* flow.cpp:247-249 */
#define STABGPU_MAX_RANSAC_ITERATIONS (1 << 24) /* RANSAC is new; bound keeps hypothesis indices in int */

/* ---- configuration records (same field names and defaults) ---------- */

/* DetectConfig, features.hpp:15-21 */
typedef struct stabgpu_detect_cfg {
    int max_corners;      /* 50 */
    double quality_level; /* 0.01 */
    double min_distance;  /* 10.0 */
    int block_size;       /* 3 */
    double roi_margin;    /* 0.1 */
} stabgpu_detect_cfg;

/* FlowConfig, flow.hpp:13-21 */
typedef struct stabgpu_flow_cfg {
    int window_radius;     /* 10 */
    int max_levels;        /* 4 */
    int max_iterations;    /* 30 */
    double epsilon;        /* 0.01 */
    double fb_threshold;   /* 0.5 */
    int redetect_interval; /* 5 */
    int min_tracks;        /* 8 */
} stabgpu_flow_cfg;

/* Robust wrapper around estimate_similarity/estimate_rigid (motion.cpp:62-76).
 * The reference has no RANSAC (SPEC.md:330 leaves room for one without an
 * interface change); iterations == 0 reproduces the reference exactly. */
typedef struct stabgpu_ransac_cfg {
    int iterations;   /* hypotheses per frame pair, 0 = off */
    double threshold; /* inlier residual, px */
    uint64_t seed;
} stabgpu_ransac_cfg;

/* SelectionMode, motion.hpp:27 */
typedef enum stabgpu_selection_mode {
    STABGPU_HYBRID = 0,
    STABGPU_FORCE_RIGID = 1,
    STABGPU_FORCE_SIMILARITY = 2
} stabgpu_selection_mode;

/* SelectorConfig, motion.hpp:29-33 */
typedef struct stabgpu_selector_cfg {
    int dwell;     /* 20 */
    double margin; /* 0.05 */
    int mode;      /* stabgpu_selection_mode, default HYBRID */
} stabgpu_selector_cfg;

/* StabConfig, pipeline.hpp:15-22 (+ the RANSAC record) */
typedef struct stabgpu_config {
    stabgpu_detect_cfg detect;
    stabgpu_flow_cfg flow;
    int smooth_radius; /* SmoothConfig.radius, smoothing.hpp:11-13, default 10 */
    stabgpu_selector_cfg selector;
    stabgpu_ransac_cfg ransac;
    double crop_ratio;     /* 0.04 */
    size_t queue_capacity; /* 64; validated like pipeline.cpp:25 */
} stabgpu_config;

/* ModelKind, transform.hpp:10 */
typedef enum stabgpu_model_kind { STABGPU_RIGID = 0, STABGPU_SIMILARITY = 1 } stabgpu_model_kind;

/* SimilarityTransform, transform.hpp:13-32 */
typedef struct stabgpu_transform {
    double tx, ty, theta, s;
    int kind;
} stabgpu_transform;

/* DeltaParams, transform.hpp:42-49 */
typedef struct stabgpu_delta {
    double dx, dy, da, dls;
    int kind;
    int skipped;
} stabgpu_delta;

/* RoiRect, features.hpp:27-36 (half-open) */
typedef struct stabgpu_roi {
    int x0, y0, x1, y1;
} stabgpu_roi;

/* Pyramid, frame.hpp:43-49: levels packed back to back in `data`. */
typedef struct stabgpu_pyramid {
    int levels;
    int width[STABGPU_MAX_LEVELS];
    int height[STABGPU_MAX_LEVELS];
    size_t offset[STABGPU_MAX_LEVELS]; /* byte offset of each level in data */
    uint8_t* data;
} stabgpu_pyramid;

/* Per-frame outcome of a sequence run (what MotionStage::step returns plus
 * the correction CompensationPlanner releases, pipeline.cpp:80-151). */
typedef enum stabgpu_frame_kind {
    STABGPU_FRAME_FIRST = 0,   /* Tracker::Advance::Kind::FirstFrame */
    STABGPU_FRAME_SKIPPED = 1, /* Kind::Skipped (< min_tracks pairs) */
    STABGPU_FRAME_TRACKED = 2  /* Kind::Tracked */
} stabgpu_frame_kind;

typedef struct stabgpu_frame_record {
    stabgpu_delta delta;          /* the delta appended to the trajectory */
    stabgpu_transform correction; /* Trajectory::correction(i) */
    int frame_kind;               /* stabgpu_frame_kind */
    int n_tracks;                 /* weeded pairs (TrackSet size) */
    int n_inliers;                /* pairs used by the fit (== n_tracks without RANSAC) */
    int decision;                 /* 1 when the selector took a decision on this frame */
} stabgpu_frame_record;

/* ---- library / context ---------------------------------------------- */
typedef struct stabgpu_ctx stabgpu_ctx;

const char* stabgpu_last_error(void);
const char* stabgpu_version(void);

/* Reference defaults (features.hpp, flow.hpp, motion.hpp, smoothing.hpp, pipeline.hpp). */
void stabgpu_default_config(stabgpu_config* cfg);

/* validate(...) overloads: features.cpp:10-26, flow.cpp:10-21,
 * motion.cpp:113-120, smoothing.cpp:10-14, pipeline.cpp:17-28. */
int stabgpu_validate_config(const stabgpu_config* cfg);

int stabgpu_create(int device, stabgpu_ctx** out);
int stabgpu_destroy(stabgpu_ctx* ctx);
/* Run subsequent work on a caller-provided cudaStream_t (NULL = context stream). */
int stabgpu_set_stream(stabgpu_ctx* ctx, void* cuda_stream);
int stabgpu_synchronize(stabgpu_ctx* ctx);

/* ---- L1 image ops: image_ops.hpp:12-33 ------------------------------- */

/* Bytes needed for the packed pyramid of a w x h frame (all levels). */
size_t stabgpu_pyramid_bytes(int w, int h, int max_levels);

/* build_pyramid, image_ops.hpp:12 / image_ops.cpp:62-77. `out->data` must
 * hold stabgpu_pyramid_bytes() bytes (host). */
int stabgpu_build_pyramid(stabgpu_ctx* ctx, const uint8_t* host_src, int w, int h, int max_levels,
                          stabgpu_pyramid* out);

/* build_pyramid over n frames of one size (host frames back to back) in the
 * batched per-level launches Stage I uses.  host_out receives n packed
 * pyramids of stabgpu_pyramid_bytes() each, levels in stabgpu_pyramid order;
 * each equals build_pyramid of that frame alone. */
int stabgpu_build_pyramid_batch(stabgpu_ctx* ctx, const uint8_t* host_frames, int n, int w, int h,
                                int max_levels, uint8_t* host_out);

/* gradients, image_ops.hpp:15 / image_ops.cpp:79-96 (host doubles out). */
int stabgpu_gradients(stabgpu_ctx* ctx, const uint8_t* host_src, int w, int h, double* host_gx,
                      double* host_gy);

/* warp_similarity, image_ops.hpp:23 / image_ops.cpp:115-134 */
int stabgpu_warp_similarity(stabgpu_ctx* ctx, const uint8_t* host_src, int w, int h,
                            const stabgpu_transform* t, uint8_t* host_out);

/* crop_resize, image_ops.hpp:27 / image_ops.cpp:136-159 */
int stabgpu_crop_resize(stabgpu_ctx* ctx, const uint8_t* host_src, int w, int h, double crop_ratio,
                        uint8_t* host_out);

/* compose_stabilized, image_ops.hpp:32-33 / image_ops.cpp:206-219.
 * cb/cr may be NULL (luma-only VideoFrame). */
int stabgpu_compose_stabilized(stabgpu_ctx* ctx, const uint8_t* host_y, const uint8_t* host_cb,
                               const uint8_t* host_cr, int w, int h, int cw, int ch,
                               const stabgpu_transform* correction, double crop_ratio,
                               uint8_t* host_out_y, uint8_t* host_out_cb, uint8_t* host_out_cr);

/* ---- L2 features + flow: features.hpp:40-49, flow.hpp:35-68 --------- */

/* detection_roi, features.hpp:40 / features.cpp:28-36 (host only). */
int stabgpu_detection_roi(int w, int h, double roi_margin, stabgpu_roi* out);

/* min_eig_response, features.hpp:44 / features.cpp:78-87 (host doubles out, w*h). */
int stabgpu_min_eig_response(stabgpu_ctx* ctx, const uint8_t* host_src, int w, int h,
                             int block_size, double* host_out);

/* detect_corners, features.hpp:49 / features.cpp:89-141.  host_xy holds
 * 2*max_corners doubles, host_score max_corners; *n_out = corners found. */
int stabgpu_detect_corners(stabgpu_ctx* ctx, const uint8_t* host_src, int w, int h,
                           const stabgpu_detect_cfg* cfg, double* host_xy, double* host_score,
                           int* n_out);

/* detect_corners over n frames of one size in one batch (host frames
 * back to back, w*h bytes each): the batched K2-K4 launch Stage I uses.
 * Frame f's corners: host_xy[2*max_corners*f ...], host_score[max_corners*f
 * ...], n_out[f].  Each frame equals detect_corners of that frame alone. */
int stabgpu_detect_corners_batch(stabgpu_ctx* ctx, const uint8_t* host_frames, int n, int w, int h,
                                 const stabgpu_detect_cfg* cfg, double* host_xy, double* host_score,
                                 int* n_out);

/* track_lk, flow.hpp:35-36 / flow.cpp:243-256. */
int stabgpu_track_lk(stabgpu_ctx* ctx, const stabgpu_pyramid* prev, const stabgpu_pyramid* cur,
                     const double* host_xy, int n, const stabgpu_flow_cfg* cfg, double* host_out_xy,
                     uint8_t* host_ok);

/* weed_tracks, flow.hpp:51-52 / flow.cpp:258-280.  Outputs the kept pairs in
 * input order; *n_out = kept count. */
int stabgpu_weed_tracks(stabgpu_ctx* ctx, const stabgpu_pyramid* prev, const stabgpu_pyramid* cur,
                        const double* host_prev_xy, const double* host_cur_xy, int n,
                        const stabgpu_flow_cfg* cfg, double* host_keep_prev_xy,
                        double* host_keep_cur_xy, int* n_out);

/* ---- L3 motion: motion.hpp:13-25 ------------------------------------ */

/* estimate_similarity / estimate_rigid (motion.cpp:62-76); kind selects. */
int stabgpu_estimate(stabgpu_ctx* ctx, const double* host_prev_xy, const double* host_cur_xy, int n,
                     int kind, stabgpu_transform* out);

/* rms_residual, motion.cpp:78-90 */
int stabgpu_rms_residual(stabgpu_ctx* ctx, const double* host_prev_xy, const double* host_cur_xy,
                         int n, const stabgpu_transform* t, double* out);

/* Robust fit: RANSAC over 2-point minimal models, then estimate_* on the
 * inliers.  host_inliers (n bytes, may be NULL) receives the inlier mask. */
int stabgpu_ransac_estimate(stabgpu_ctx* ctx, const double* host_prev_xy, const double* host_cur_xy,
                            int n, int kind, const stabgpu_ransac_cfg* rc, int min_tracks,
                            int64_t frame_index, stabgpu_transform* out, uint8_t* host_inliers,
                            int* n_inliers);

/* extract_delta / delta_to_transform, motion.cpp:92-111 (host only). */
void stabgpu_extract_delta(const stabgpu_transform* t, stabgpu_delta* out);
void stabgpu_delta_to_transform(double dx, double dy, double da, double dls, stabgpu_transform* out);

/* Trajectory::append + correction over a complete trajectory
 * (smoothing.cpp:16-57), n deltas in, n corrections out (host). */
int stabgpu_trajectory_corrections(stabgpu_ctx* ctx, const stabgpu_delta* host_deltas, int n,
                                   int smooth_radius, stabgpu_transform* host_corrections);

/* ---- Stage I: whole-sequence stabilization (run_offline semantics,
 * pipeline.cpp:182-235), GPU-batched over independent re-detect segments. */

/* Host buffers: planes are frame-major, plane 0 luma (n*w*h bytes), planes
 * 1/2 chroma (n*cw*ch bytes each, may be NULL).  Copies in and out are part
 * of the call (chunked, overlapped with compute).  records: n entries or NULL. */
int stabgpu_stabilize_sequence(stabgpu_ctx* ctx, const uint8_t* host_y, const uint8_t* host_cb,
                               const uint8_t* host_cr, int n_frames, int w, int h, int cw, int ch,
                               const stabgpu_config* cfg, uint8_t* host_out_y, uint8_t* host_out_cb,
                               uint8_t* host_out_cr, stabgpu_frame_record* records);

/* Same pipeline with every buffer already resident on the device. */
int stabgpu_stabilize_sequence_device(stabgpu_ctx* ctx, const uint8_t* dev_y, const uint8_t* dev_cb,
                                      const uint8_t* dev_cr, int n_frames, int w, int h, int cw,
                                      int ch, const stabgpu_config* cfg, uint8_t* dev_out_y,
                                      uint8_t* dev_out_cb, uint8_t* dev_out_cr,
                                      stabgpu_frame_record* host_records);

/* ---- Multi-stream Stage I (BASELINE configs[4]: many independent
 * sequences per GPU).  n_streams sequences of `frames` frames each, laid out
 * stream-major ([stream][frame][h][w], chroma likewise).  Each stream's
 * output and records (n_streams*frames entries, stream-major) equal
 * run_offline (pipeline.cpp:182-235) on that stream alone; the RANSAC seed
 * is the frame's index within its stream.  All streams share one launch per
 * stage.  Errors name the stream ("stream k frame f: ..."). */
int stabgpu_stabilize_streams(stabgpu_ctx* ctx, const uint8_t* host_y, const uint8_t* host_cb,
                              const uint8_t* host_cr, int n_streams, int frames, int w, int h,
                              int cw, int ch, const stabgpu_config* cfg, uint8_t* host_out_y,
                              uint8_t* host_out_cb, uint8_t* host_out_cr,
                              stabgpu_frame_record* records);
int stabgpu_stabilize_streams_device(stabgpu_ctx* ctx, const uint8_t* dev_y, const uint8_t* dev_cb,
                                     const uint8_t* dev_cr, int n_streams, int frames, int w, int h,
                                     int cw, int ch, const stabgpu_config* cfg, uint8_t* dev_out_y,
                                     uint8_t* dev_out_cb, uint8_t* dev_out_cr,
                                     stabgpu_frame_record* host_records);

/* ---- Stage I split for multi-GPU sharding (§8e of SURVEY.md) ----------
 * Motion estimation for frames (first, first+count] of a sequence whose
 * frame `first` is a re-detect frame (first % redetect_interval == 0).
 * dev_y points at frame `first` (count+1 frames resident).  Writes one
 * stabgpu_motion_record per frame first+1 .. first+count (and for frame 0
 * when first == 0, as record 0 with frame_kind FIRST) into host_out. */
typedef struct stabgpu_motion_record {
    stabgpu_delta rigid;      /* fit with ModelKind::Rigid       */
    stabgpu_delta similarity; /* fit with ModelKind::Similarity  */
    double e_rigid;           /* rms_residual of each fit (hybrid decisions) */
    double e_similarity;
    int frame_kind;           /* stabgpu_frame_kind */
    int n_tracks;
    int n_inliers_rigid;
    int n_inliers_similarity;
    int status;               /* stabgpu_status of the fit for this frame */
    int pad;
} stabgpu_motion_record;

int stabgpu_motion_chunk(stabgpu_ctx* ctx, const uint8_t* dev_y, int64_t first, int count, int w,
                         int h, const stabgpu_config* cfg, stabgpu_motion_record* host_out);

/* Selector scan + trajectory + smoothing over all n motion records
 * (motion.cpp:143-191, smoothing.cpp:16-57) -> per-frame records. */
int stabgpu_plan_corrections(stabgpu_ctx* ctx, const stabgpu_motion_record* host_motion, int n,
                             const stabgpu_config* cfg, stabgpu_frame_record* host_records);

/* compose_stabilized over frames [0, count) with device-resident planes. */
int stabgpu_compose_frames(stabgpu_ctx* ctx, const uint8_t* dev_y, const uint8_t* dev_cb,
                           const uint8_t* dev_cr, int count, int w, int h, int cw, int ch,
                           const stabgpu_transform* host_corrections, double crop_ratio,
                           uint8_t* dev_out_y, uint8_t* dev_out_cb, uint8_t* dev_out_cr);

/* ---- sharded Stage I over the GPUs of a box ------------
 * The sequence is cut into contiguous re-detect-aligned shards (tracking
 * state resets at every re-detect frame, flow.cpp:326-330): rank g estimates
 * the motion of frames first_g+1 .. first_g+count_g from its resident frames
 * first_g .. first_g+count_g (frame first_g, the previous rank's last frame,
 * is the one-frame halo), the ~120 B/frame motion records of all ranks are
 * all-gathered, every rank runs the sequential selector/trajectory/smoothing
 * scan on identical input (bit-identical corrections everywhere) and
 * composes its own frames [own_begin_g, own_end_g).  The partition is
 * stabgpu_shard_range (== pipeline.shard_ranges). */
#define STABGPU_NCCL_ID_BYTES 128
int stabgpu_shard_range(int64_t n, int redetect_interval, int world, int rank, int64_t* first, int* count,
                        int64_t* own_begin, int64_t* own_end);
/* NCCL communicator owned by the context (one rank per GPU): rank 0 calls
 * stabgpu_nccl_unique_id and shares the 128 bytes (e.g. over
 * torch.distributed), every rank calls stabgpu_comm_init.  NCCL is resolved
 * from libnccl.so.2 at run time. */
int stabgpu_nccl_unique_id(unsigned char* id_out);
int stabgpu_comm_init(stabgpu_ctx* ctx, const unsigned char* id, int nranks, int rank);
/* One call per rank (world/rank from stabgpu_comm_init; a context without a
 * communicator is world 1): host planes of the rank's frames first..first+
 * count in, host planes of its own frames out.  Chunked upload overlaps the
 * motion passes; the records are all-gathered device to device (ncclAllGather
 * on the context stream); the compose of each chunk of own frames overlaps
 * the download of the previous one.  records (optional): all n frames. */
int stabgpu_stabilize_sharded(stabgpu_ctx* ctx, const uint8_t* host_y, const uint8_t* host_cb,
                              const uint8_t* host_cr, int64_t n, int w, int h, int cw, int ch,
                              const stabgpu_config* cfg, uint8_t* host_out_y, uint8_t* host_out_cb,
                              uint8_t* host_out_cr, stabgpu_frame_record* records);
/* Device-resident variant: dev_* hold the rank's frames first..first+count,
 * dev_out_* receive its own frames [own_begin, own_end). */
int stabgpu_stabilize_sharded_device(stabgpu_ctx* ctx, const uint8_t* dev_y, const uint8_t* dev_cb,
                                     const uint8_t* dev_cr, int64_t n, int w, int h, int cw, int ch,
                                     const stabgpu_config* cfg, uint8_t* dev_out_y, uint8_t* dev_out_cb,
                                     uint8_t* dev_out_cr, stabgpu_frame_record* records);
/* The same call split at the exchange, for a host-side all-gather (e.g. a
 * gloo process group, or ranks emulated in one process): shard_motion keeps
 * the rank's frames resident in the context and returns its count+1 motion
 * records (record 0: frame first — the FIRST record on rank 0); the caller
 * assembles all n records (pipeline.assemble_motion) and shard_compose plans
 * and composes the rank's own frames. */
int stabgpu_shard_motion(stabgpu_ctx* ctx, const uint8_t* host_y, const uint8_t* host_cb,
                         const uint8_t* host_cr, int64_t n, int world, int rank, int w, int h, int cw,
                         int ch, const stabgpu_config* cfg, stabgpu_motion_record* host_motion);
int stabgpu_shard_compose(stabgpu_ctx* ctx, const stabgpu_motion_record* host_all_motion, int64_t n,
                          int world, int rank, int w, int h, int cw, int ch, const stabgpu_config* cfg,
                          uint8_t* host_out_y, uint8_t* host_out_cb, uint8_t* host_out_cr,
                          stabgpu_frame_record* records);

/* ---- device-resident Tracker (flow.hpp:56-82, flow.cpp:297-337) -------
 * Tracker::advance with the previous pyramid, the carried points and the
 * re-detect cadence kept on the device: advance uploads one frame, builds
 * its pyramid, tracks forward + weeds backward, re-detects every
 * redetect_interval frames and returns the TrackSet (n pairs of prev / cur
 * points, each host array holding 2 * max_corners doubles) and the kind
 * (STABGPU_FRAME_FIRST / SKIPPED when n < min_tracks / TRACKED); n_active
 * (optional) = active_point_count() after the call.  Errors as the reference
 * (SequencingError on a non-increasing index). */
typedef struct stabgpu_tracker stabgpu_tracker;
int stabgpu_tracker_create(stabgpu_ctx* ctx, const stabgpu_flow_cfg* flow, const stabgpu_detect_cfg* detect, int w,
                           int h, stabgpu_tracker** out);
int stabgpu_tracker_advance(stabgpu_tracker* t, const uint8_t* host_frame, int64_t index, int* kind,
                            double* host_prev_xy, double* host_cur_xy, int* n_out, int* n_active);
/* active_point_count() (flow.hpp:69) */
int stabgpu_tracker_points(stabgpu_tracker* t, int* n_out);
int stabgpu_tracker_destroy(stabgpu_tracker* t);

/* ---- Stage II: streaming (one frame at a time) ------------------------
 * Replaces run_streaming (pipeline.hpp:72-76 / pipeline.cpp:237-365) and the
 * MotionStage -> CompensationPlanner -> compose loop of run_offline
 * (pipeline.cpp:182-235): frames are pushed one at a time; a frame's
 * correction is released with the reference's CompensationPlanner rule
 * (nothing before 2r motion estimates unless the stream ended, then every
 * frame whose smoothing window is complete, pipeline.cpp:137-150), so the
 * latency is exactly r frames and the first emission happens at frame 2r.
 * The released frames are bit-identical to Stage I (stabilize_sequence).
 * Planes are host (pageable or pinned) or device pointers (unified
 * addressing; pitch = width).  After every push / finish the caller pops the
 * ready frames in arrival order.  A push's launches run on four streams:
 * the pyramid stream (K1 of the frame as soon as it lands), the motion chain
 * (the K5 step + compaction + K6 fit, the K7 scan), the
 * release chain (smoothing + K8 compose of the frame it releases, behind the
 * scan) and, every redetect_interval frames, the re-detection (as soon as
 * its frame has landed; the next frame's K5 waits for it, so a caller that
 * keeps a few frames queued - push_async / pop_async - hides it behind the
 * K5 steps of the frames before) - so frame k+1's motion overlaps frame k's
 * compose.  Each chain is one CUDA graph, instantiated once per topology and
 * updated in place per frame.
 * Frames whose planes lie back to back in the caller's memory (cb == y + w*h,
 * cr == cb + cw*ch: one planar buffer per frame, as a Y4M reader holds them,
 * media_io.cpp:139-145) move in one copy per direction when the plane sizes
 * are multiples of 256 bytes; anything else moves plane by plane. */
typedef struct stabgpu_stream stabgpu_stream;

int stabgpu_stream_create(stabgpu_ctx* ctx, const stabgpu_config* cfg, int w, int h, int cw, int ch,
                          stabgpu_stream** out);
/* Motion estimate of the next frame; *n_ready = frames ready to pop. */
int stabgpu_stream_push(stabgpu_stream* s, const uint8_t* y, const uint8_t* cb, const uint8_t* cr,
                        int* n_ready);
/* The same, returning before the frame's upload has landed (the launches are
 * queued behind it): the caller keeps y/cb/cr unchanged until
 * stabgpu_stream_wait_inputs or a later stabgpu_stream_push returns.  With two
 * or more host frame buffers in rotation, frame k+1 uploads while frame k's
 * motion runs (run_streaming's reader thread, pipeline.cpp:251-272). */
int stabgpu_stream_push_async(stabgpu_stream* s, const uint8_t* y, const uint8_t* cb, const uint8_t* cr,
                              int* n_ready);
int stabgpu_stream_wait_inputs(stabgpu_stream* s);
/* Page-locked host memory (cudaHostAlloc / cudaFreeHost) for frames handed to
 * the host-buffer and stream entry points: copies from and to it are
 * asynchronous and run at the full PCIe rate, pageable memory is staged by
 * the driver.  The drop-in run_offline / run_streaming (shim/pipeline_b200.cpp)
 * stage the caller's std::vector frames (frame.hpp:14-33) through it. */
int stabgpu_host_alloc(void** out, size_t bytes);
int stabgpu_host_free(void* p);
/* End of stream: releases the remaining frames (at least 2 frames pushed). */
int stabgpu_stream_finish(stabgpu_stream* s, int* n_ready);
/* Oldest ready frame (its index, planes and record); STABGPU_SEQUENCING if none. */
int stabgpu_stream_pop(stabgpu_stream* s, int64_t* index, uint8_t* out_y, uint8_t* out_cb,
                       uint8_t* out_cr, stabgpu_frame_record* record);
/* stabgpu_stream_pop that returns once the download is queued (the frame index
 * is final; the planes and *record are valid after the next
 * stabgpu_stream_wait_pops): pop_async, push the next frame, wait_pops lets the
 * download of frame k-r overlap the upload of frame k+1 (the IC thread of
 * run_streaming, pipeline.cpp:318-336, beside its reader thread). */
int stabgpu_stream_pop_async(stabgpu_stream* s, int64_t* index, uint8_t* out_y, uint8_t* out_cb,
                             uint8_t* out_cr, stabgpu_frame_record* record);
/* Waits for every queued pop_async download; reports a selector error of the popped frames. */
int stabgpu_stream_wait_pops(stabgpu_stream* s);
int stabgpu_stream_destroy(stabgpu_stream* s);
/* Per-frame CUDA graphs on (default) or off (one launch per kernel); off is
 * forced when a launch sequence needs stream-ordered scratch (more than 8192
 * corners).  Results are identical either way. */
int stabgpu_stream_set_graphs(stabgpu_stream* s, int on);

/* ---- colour I/O and evaluation ---------------------
 * Device-resident, n frames of w x h (pitch = width).  RGB is interleaved
 * 8-bit.  Conversions are the reference's BT.601 full-range formulas
 * (media_io.cpp:75-89 yuv_to_rgb / chroma_cb / chroma_cr, 568-570
 * luma_bt601), bit-exact. */
int stabgpu_rgb_to_ycbcr(stabgpu_ctx* ctx, const uint8_t* dev_rgb, int n, int w, int h,
                         uint8_t* dev_y, uint8_t* dev_cb, uint8_t* dev_cr);
int stabgpu_ycbcr_to_rgb(stabgpu_ctx* ctx, const uint8_t* dev_y, const uint8_t* dev_cb,
                         const uint8_t* dev_cr, int n, int w, int h, uint8_t* dev_rgb);
/* Stage I on interleaved RGB host frames (4:4:4 after conversion), output
 * RGB host frames: upload, conversion, run_offline semantics, conversion of
 * the composed planes back to RGB, download (media_io load/save around
 * run_offline). */
int stabgpu_stabilize_sequence_rgb(stabgpu_ctx* ctx, const uint8_t* host_rgb, int n, int w, int h,
                                   const stabgpu_config* cfg, uint8_t* host_out_rgb,
                                   stabgpu_frame_record* records);
/* psnr_pair (synth_eval.cpp:214-240) support: the exact integer sum of
 * squared differences of frames (k-1, k) over the cropped region, k = 1..n-1,
 * and the pixel count of that region (host_sse has n-1 entries). */
int stabgpu_interframe_sse(stabgpu_ctx* ctx, const uint8_t* dev_y, int n, int w, int h,
                           double crop_ratio, uint64_t* host_sse, int64_t* host_count);

/* ---- instrumentation (bench / tests) -------------------------------- */
/* Per-kernel-family device time of the last sequence call (ms, CUDA events
 * on the launching stream) and the number of kernel launches it issued. */
typedef struct stabgpu_stats {
    double ms_pyramid, ms_detect, ms_track, ms_fit, ms_plan, ms_compose, ms_total;
    long long launches;
    long long lk_level_builds; /* LK template (level patch) builds of the last motion pass */
    long long lk_iterations;
} stabgpu_stats;
int stabgpu_get_stats(stabgpu_ctx* ctx, stabgpu_stats* out);

/* Test/diagnostic hook: copies up to `bytes` of the context's named device
 * scratch buffer (e.g. "trk_prev", "trk_n" of the last Stage I motion pass)
 * to host; *have = the buffer's size.  No reference analogue. */
int stabgpu_debug_read_scratch(stabgpu_ctx* ctx, const char* name, void* host, size_t bytes, size_t* have);
int stabgpu_enable_timing(stabgpu_ctx* ctx, int on);

#ifdef __cplusplus
}
#endif

#endif /* STABGPU_H_ */
