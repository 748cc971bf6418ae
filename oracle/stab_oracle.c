/*
 * stab_oracle.c — CPU ORACLE (test infrastructure only; see stab_oracle.h).
 *
 * Plain-C restatement of the reference hot path.  Floating-point expressions
 * keep the reference's evaluation order and are compiled with
 * -ffp-contract=off (oracle/Makefile) so that, like the reference built for
 * baseline x86-64, no multiply-add is fused.  File:line citations are into
 * /root/reference/proj/src.
 */
#include "stab_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* orc_last_error(void) { return g_err; }

static inline int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }
static inline int mini(int a, int b) { return a < b ? a : b; }
static inline int maxi(int a, int b) { return a > b ? a : b; }
static inline uint8_t clamp_u8(long v) { return (uint8_t)(v < 0 ? 0 : (v > 255 ? 255 : v)); }

/* validate(GrayFrame), image_ops.cpp:9-16 */
static int validate_frame(int w, int h) {
    if (w < STABGPU_MIN_FRAME_DIM || h < STABGPU_MIN_FRAME_DIM)
        return fail(STABGPU_INVALID_INPUT, "frame smaller than 16x16");
    return STABGPU_OK;
}

/* ------------------------------------------------------------------ */
/* image_ops                                                           */
/* ------------------------------------------------------------------ */

/* downsample, image_ops.cpp:25-58: horizontal [1 4 6 4 1] at every column
 * into 16-bit, vertical on even rows/cols, (acc + 128) >> 8, clamp borders. */
static void downsample(const uint8_t* src, int w, int h, uint8_t* dst) {
    const int ow = w / 2, oh = h / 2;
    uint16_t* tmp = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)w * h);
    for (int y = 0; y < h; ++y) {
        const uint8_t* row = src + (size_t)y * w;
        uint16_t* out = tmp + (size_t)y * w;
        for (int x = 0; x < w; ++x) {
            out[x] = (uint16_t)(row[clampi(x - 2, 0, w - 1)] + 4 * row[clampi(x - 1, 0, w - 1)] +
                                6 * row[x] + 4 * row[clampi(x + 1, 0, w - 1)] +
                                row[clampi(x + 2, 0, w - 1)]);
        }
    }
    for (int y = 0; y < oh; ++y) {
        const int sy = 2 * y;
        for (int x = 0; x < ow; ++x) {
            const int sx = 2 * x;
            const uint32_t acc = tmp[(size_t)clampi(sy - 2, 0, h - 1) * w + sx] +
                                 4u * tmp[(size_t)clampi(sy - 1, 0, h - 1) * w + sx] +
                                 6u * tmp[(size_t)sy * w + sx] +
                                 4u * tmp[(size_t)clampi(sy + 1, 0, h - 1) * w + sx] +
                                 tmp[(size_t)clampi(sy + 2, 0, h - 1) * w + sx];
            dst[(size_t)y * ow + x] = (uint8_t)((acc + 128) >> 8);
        }
    }
    free(tmp);
}

size_t orc_pyramid_bytes(int w, int h, int max_levels) {
    size_t total = 0;
    for (int l = 0; l < max_levels && l < STABGPU_MAX_LEVELS; ++l) {
        total += (size_t)w * h;
        if (w / 2 < STABGPU_MIN_FRAME_DIM || h / 2 < STABGPU_MIN_FRAME_DIM) break;
        w /= 2;
        h /= 2;
    }
    return total;
}

/* build_pyramid, image_ops.cpp:62-77 */
int orc_build_pyramid(const uint8_t* src, int w, int h, int max_levels, stabgpu_pyramid* out) {
    int rc = validate_frame(w, h);
    if (rc) return rc;
    if (max_levels < 1) return fail(STABGPU_INVALID_INPUT, "max_levels must be >= 1");
    if (max_levels > STABGPU_MAX_LEVELS) max_levels = STABGPU_MAX_LEVELS;
    out->levels = 1;
    out->width[0] = w;
    out->height[0] = h;
    out->offset[0] = 0;
    memcpy(out->data, src, (size_t)w * h);
    while (out->levels < max_levels) {
        const int l = out->levels - 1;
        const int tw = out->width[l], th = out->height[l];
        if (tw / 2 < STABGPU_MIN_FRAME_DIM || th / 2 < STABGPU_MIN_FRAME_DIM) break;
        out->width[l + 1] = tw / 2;
        out->height[l + 1] = th / 2;
        out->offset[l + 1] = out->offset[l] + (size_t)tw * th;
        downsample(out->data + out->offset[l], tw, th, out->data + out->offset[l + 1]);
        out->levels++;
    }
    return STABGPU_OK;
}

/* gradients, image_ops.cpp:79-96 */
int orc_gradients(const uint8_t* f, int w, int h, double* gx, double* gy) {
    int rc = validate_frame(w, h);
    if (rc) return rc;
    for (int y = 0; y < h; ++y) {
        const int ym = maxi(y - 1, 0), yp = mini(y + 1, h - 1);
        for (int x = 0; x < w; ++x) {
            const int xm = maxi(x - 1, 0), xp = mini(x + 1, w - 1);
            gx[(size_t)y * w + x] = 0.5 * ((double)f[(size_t)y * w + xp] - f[(size_t)y * w + xm]);
            gy[(size_t)y * w + x] = 0.5 * ((double)f[(size_t)yp * w + x] - f[(size_t)ym * w + x]);
        }
    }
    return STABGPU_OK;
}

/* sample_bilinear, image_ops.cpp:98-113 */
static double sample_bilinear(const uint8_t* f, int w, int h, double px, double py) {
    const double xmax = w - 1.0, ymax = h - 1.0;
    if (!(px >= 0.0 && py >= 0.0 && px <= xmax && py <= ymax)) return 0.0;
    const int x0 = (int)px, y0 = (int)py;
    const int x1 = mini(x0 + 1, w - 1), y1 = mini(y0 + 1, h - 1);
    const double fx = px - x0, fy = py - y0;
    const uint8_t a = f[(size_t)y0 * w + x0], b = f[(size_t)y0 * w + x1];
    const uint8_t c = f[(size_t)y1 * w + x0], d = f[(size_t)y1 * w + x1];
    const double top = a + fx * (b - (double)a);
    const double bot = c + fx * (d - (double)c);
    return top + fy * (bot - top);
}

static int validate_transform(const stabgpu_transform* t) { /* transform.cpp:51-59 */
    if (!isfinite(t->tx) || !isfinite(t->ty) || !isfinite(t->theta) || !isfinite(t->s) ||
        t->s <= 0.0)
        return fail(STABGPU_INVALID_TRANSFORM,
                    "similarity transform requires finite parameters and s > 0");
    if (t->kind == STABGPU_RIGID && t->s != 1.0)
        return fail(STABGPU_INVALID_TRANSFORM, "rigid transform must have s == 1");
    return STABGPU_OK;
}

/* warp_similarity, image_ops.cpp:115-134 (row-incremental coordinates) */
int orc_warp_similarity(const uint8_t* src, int w, int h, const stabgpu_transform* t, uint8_t* out) {
    int rc = validate_frame(w, h);
    if (rc) return rc;
    rc = validate_transform(t);
    if (rc) return rc;
    const double c = cos(t->theta) / t->s;
    const double sn = sin(t->theta) / t->s;
    for (int y = 0; y < h; ++y) {
        double sx = c * (0.0 - t->tx) + sn * (y - t->ty);
        double sy = -sn * (0.0 - t->tx) + c * (y - t->ty);
        uint8_t* row = out + (size_t)y * w;
        for (int x = 0; x < w; ++x) {
            row[x] = clamp_u8(lround(sample_bilinear(src, w, h, sx, sy)));
            sx += c;
            sy -= sn;
        }
    }
    return STABGPU_OK;
}

/* crop_resize, image_ops.cpp:136-159 */
int orc_crop_resize(const uint8_t* src, int w, int h, double crop_ratio, uint8_t* out) {
    int rc = validate_frame(w, h);
    if (rc) return rc;
    if (!(crop_ratio >= 0.0 && crop_ratio < 0.25))
        return fail(STABGPU_INVALID_CONFIG, "crop_ratio must lie in [0, 0.25)");
    const int mx = (int)lround(crop_ratio * w);
    const int my = (int)lround(crop_ratio * h);
    if (mx == 0 && my == 0) {
        memcpy(out, src, (size_t)w * h);
        return STABGPU_OK;
    }
    const int cw = w - 2 * mx, ch = h - 2 * my;
    const double step_x = w > 1 ? (double)(cw - 1) / (w - 1) : 0.0;
    const double step_y = h > 1 ? (double)(ch - 1) / (h - 1) : 0.0;
    for (int y = 0; y < h; ++y) {
        const double sy = my + y * step_y;
        for (int x = 0; x < w; ++x) {
            const double sx = mx + x * step_x;
            out[(size_t)y * w + x] = clamp_u8(lround(sample_bilinear(src, w, h, sx, sy)));
        }
    }
    return STABGPU_OK;
}

/* compose_plane, image_ops.cpp:165-202 (transform applied via apply_inverse,
 * transform.cpp:13-19, which recomputes cos/sin per call) */
static void compose_plane(const uint8_t* plane, int cw, int ch, int lw, int lh,
                          const stabgpu_transform* t, double crop_ratio, uint8_t* out) {
    const double fx = (double)lw / cw;
    const double fy = (double)lh / ch;
    const int mx = (int)lround(crop_ratio * lw);
    const int my = (int)lround(crop_ratio * lh);
    const double step_x = lw > 1 ? (double)(lw - 2 * mx - 1) / (lw - 1) : 0.0;
    const double step_y = lh > 1 ? (double)(lh - 2 * my - 1) / (lh - 1) : 0.0;
    const double c = cos(t->theta) / t->s;
    const double sn = sin(t->theta) / t->s;
    for (int y = 0; y < ch; ++y) {
        for (int x = 0; x < cw; ++x) {
            double lx = (x + 0.5) * fx - 0.5;
            double ly = (y + 0.5) * fy - 0.5;
            if (mx != 0 || my != 0) {
                lx = mx + lx * step_x;
                ly = my + ly * step_y;
            }
            const double dx = lx - t->tx, dy = ly - t->ty;
            const double pxl = c * dx + sn * dy, pyl = -sn * dx + c * dy;
            const double px = (pxl + 0.5) / fx - 0.5;
            const double py = (pyl + 0.5) / fy - 0.5;
            double v = 128.0;
            if (px >= 0.0 && py >= 0.0 && px <= cw - 1.0 && py <= ch - 1.0)
                v = sample_bilinear(plane, cw, ch, px, py);
            out[(size_t)y * cw + x] = clamp_u8(lround(v));
        }
    }
}

/* compose_stabilized, image_ops.cpp:206-219 */
int orc_compose_stabilized(const uint8_t* y, const uint8_t* cb, const uint8_t* cr, int w, int h,
                           int cw, int ch, const stabgpu_transform* t, double crop_ratio,
                           uint8_t* oy, uint8_t* ocb, uint8_t* ocr) {
    uint8_t* tmp = (uint8_t*)malloc((size_t)w * h);
    int rc = orc_warp_similarity(y, w, h, t, tmp);
    if (!rc) rc = orc_crop_resize(tmp, w, h, crop_ratio, oy);
    free(tmp);
    if (rc) return rc;
    if (cb && cr) {
        compose_plane(cb, cw, ch, w, h, t, crop_ratio, ocb);
        compose_plane(cr, cw, ch, w, h, t, crop_ratio, ocr);
    }
    return STABGPU_OK;
}

/* ------------------------------------------------------------------ */
/* features                                                            */
/* ------------------------------------------------------------------ */

static int validate_detect(const stabgpu_detect_cfg* c) { /* features.cpp:10-26 */
    if (c->max_corners < 8) return fail(STABGPU_INVALID_CONFIG, "max_corners must be >= 8");
    if (!(c->quality_level > 0.0 && c->quality_level < 1.0))
        return fail(STABGPU_INVALID_CONFIG, "quality_level must lie in (0, 1)");
    if (c->min_distance < 1.0) return fail(STABGPU_INVALID_CONFIG, "min_distance must be >= 1");
    if (c->block_size < 3 || c->block_size % 2 == 0)
        return fail(STABGPU_INVALID_CONFIG, "block_size must be odd and >= 3");
    if (!(c->roi_margin >= 0.0 && c->roi_margin < 0.4))
        return fail(STABGPU_INVALID_CONFIG, "roi_margin must lie in [0, 0.4)");
    return STABGPU_OK;
}

/* detection_roi, features.cpp:28-36 */
int orc_detection_roi(int w, int h, double roi_margin, stabgpu_roi* out) {
    const int mx = (int)lround(roi_margin * w);
    const int my = (int)lround(roi_margin * h);
    out->x0 = mx;
    out->y0 = my;
    out->x1 = w - mx;
    out->y1 = h - my;
    if (out->x1 - out->x0 < 32 || out->y1 - out->y0 < 32)
        return fail(STABGPU_INVALID_CONFIG, "detection ROI smaller than 32x32");
    return STABGPU_OK;
}

/* min_eig, features.cpp:41-45 */
static inline double min_eig(double sxx, double sxy, double syy) {
    const double half_trace = 0.5 * (sxx + syy);
    const double half_diff = 0.5 * (sxx - syy);
    return half_trace - sqrt(half_diff * half_diff + sxy * sxy);
}

/* response_in_rect, features.cpp:50-74 */
static void response_in_rect(const double* gx, const double* gy, int w, int h, int block,
                             stabgpu_roi r, double* out) {
    const int half = block / 2;
    for (int y = r.y0; y < r.y1; ++y) {
        const int wy0 = maxi(y - half, 0), wy1 = mini(y + half, h - 1);
        for (int x = r.x0; x < r.x1; ++x) {
            const int wx0 = maxi(x - half, 0), wx1 = mini(x + half, w - 1);
            double sxx = 0.0, sxy = 0.0, syy = 0.0;
            for (int wy = wy0; wy <= wy1; ++wy) {
                for (int wx = wx0; wx <= wx1; ++wx) {
                    const double dx = gx[(size_t)wy * w + wx];
                    const double dy = gy[(size_t)wy * w + wx];
                    sxx += dx * dx;
                    sxy += dx * dy;
                    syy += dy * dy;
                }
            }
            out[(size_t)y * w + x] = min_eig(sxx, sxy, syy);
        }
    }
}

/* min_eig_response, features.cpp:78-87 */
int orc_min_eig_response(const uint8_t* src, int w, int h, int block, double* out) {
    int rc = validate_frame(w, h);
    if (rc) return rc;
    if (block < 3 || block % 2 == 0)
        return fail(STABGPU_INVALID_CONFIG, "block_size must be odd and >= 3");
    double* gx = (double*)malloc(sizeof(double) * (size_t)w * h);
    double* gy = (double*)malloc(sizeof(double) * (size_t)w * h);
    orc_gradients(src, w, h, gx, gy);
    memset(out, 0, sizeof(double) * (size_t)w * h);
    stabgpu_roi all = {0, 0, w, h};
    response_in_rect(gx, gy, w, h, block, all, out);
    free(gx);
    free(gy);
    return STABGPU_OK;
}

typedef struct {
    double x, y, score;
} corner_t;

/* sort comparator of features.cpp:119-123: score desc, then y, then x */
static int corner_cmp(const void* pa, const void* pb) {
    const corner_t* a = (const corner_t*)pa;
    const corner_t* b = (const corner_t*)pb;
    if (a->score != b->score) return a->score > b->score ? -1 : 1;
    if (a->y != b->y) return a->y < b->y ? -1 : 1;
    if (a->x != b->x) return a->x < b->x ? -1 : 1;
    return 0;
}

/* detect_corners, features.cpp:89-141 */
int orc_detect_corners(const uint8_t* src, int w, int h, const stabgpu_detect_cfg* cfg, double* xy,
                       double* score, int* n_out) {
    *n_out = 0;
    int rc = validate_frame(w, h);
    if (rc) return rc;
    rc = validate_detect(cfg);
    if (rc) return rc;
    stabgpu_roi roi;
    rc = orc_detection_roi(w, h, cfg->roi_margin, &roi);
    if (rc) return rc;
    double* gx = (double*)malloc(sizeof(double) * (size_t)w * h);
    double* gy = (double*)malloc(sizeof(double) * (size_t)w * h);
    double* resp = (double*)calloc((size_t)w * h, sizeof(double));
    orc_gradients(src, w, h, gx, gy);
    response_in_rect(gx, gy, w, h, cfg->block_size, roi, resp);
    double maxr = 0.0;
    for (int y = roi.y0; y < roi.y1; ++y)
        for (int x = roi.x0; x < roi.x1; ++x) {
            const double r = resp[(size_t)y * w + x];
            maxr = maxr < r ? r : maxr; /* std::max(a, b) returns a unless a < b */
        }
    if (maxr <= 0.0) {
        free(gx);
        free(gy);
        free(resp);
        return STABGPU_OK;
    }
    const double threshold = cfg->quality_level * maxr;
    size_t cap = 1024, nc = 0;
    corner_t* cand = (corner_t*)malloc(sizeof(corner_t) * cap);
    for (int y = roi.y0; y < roi.y1; ++y)
        for (int x = roi.x0; x < roi.x1; ++x) {
            const double r = resp[(size_t)y * w + x];
            if (r >= threshold && r > 0.0) {
                if (nc == cap) {
                    cap *= 2;
                    cand = (corner_t*)realloc(cand, sizeof(corner_t) * cap);
                }
                cand[nc].x = x;
                cand[nc].y = y;
                cand[nc].score = r;
                ++nc;
            }
        }
    qsort(cand, nc, sizeof(corner_t), corner_cmp);
    const double min_dist2 = cfg->min_distance * cfg->min_distance;
    int ns = 0;
    for (size_t i = 0; i < nc; ++i) {
        if (ns >= cfg->max_corners) break;
        int keep = 1;
        for (int s = 0; s < ns; ++s) {
            const double dx = cand[i].x - xy[2 * s];
            const double dy = cand[i].y - xy[2 * s + 1];
            if (dx * dx + dy * dy < min_dist2) {
                keep = 0;
                break;
            }
        }
        if (keep) {
            xy[2 * ns] = cand[i].x;
            xy[2 * ns + 1] = cand[i].y;
            score[ns] = cand[i].score;
            ++ns;
        }
    }
    *n_out = ns;
    free(cand);
    free(gx);
    free(gy);
    free(resp);
    return STABGPU_OK;
}

/* ------------------------------------------------------------------ */
/* flow                                                                */
/* ------------------------------------------------------------------ */

static int validate_flow(const stabgpu_flow_cfg* c) { /* flow.cpp:10-21 */
    if (c->window_radius < 1 || c->max_levels < 1 || c->max_iterations < 1 || c->epsilon <= 0.0 ||
        c->fb_threshold <= 0.0)
        return fail(STABGPU_INVALID_CONFIG, "flow parameters must be positive");
    if (c->redetect_interval < 1) return fail(STABGPU_INVALID_CONFIG, "redetect_interval must be >= 1");
    if (c->min_tracks < 4) return fail(STABGPU_INVALID_CONFIG, "min_tracks must be >= 4");
    return STABGPU_OK;
}

typedef struct {
    const uint8_t* px;
    int w, h;
} level_t;

static level_t level_of(const stabgpu_pyramid* p, int l) {
    level_t v = {p->data + p->offset[l], p->width[l], p->height[l]};
    return v;
}

/* extract_patch, flow.cpp:28-59 */
static void extract_patch(level_t img, double cx, double cy, int radius, double* out) {
    const int side = 2 * radius + 1;
    const int x0 = (int)floor(cx), y0 = (int)floor(cy);
    const double fx = cx - x0, fy = cy - y0;
    const double w00 = (1.0 - fx) * (1.0 - fy);
    const double w10 = fx * (1.0 - fy);
    const double w01 = (1.0 - fx) * fy;
    const double w11 = fx * fy;
    int xa[68], xb[68], ya[68], yb[68];
    for (int i = 0; i < side; ++i) {
        const int x = x0 - radius + i;
        xa[i] = clampi(x, 0, img.w - 1);
        xb[i] = clampi(x + 1, 0, img.w - 1);
        const int y = y0 - radius + i;
        ya[i] = clampi(y, 0, img.h - 1);
        yb[i] = clampi(y + 1, 0, img.h - 1);
    }
    for (int j = 0; j < side; ++j) {
        const uint8_t* ra = img.px + (size_t)ya[j] * img.w;
        const uint8_t* rb = img.px + (size_t)yb[j] * img.w;
        double* dst = out + (size_t)j * side;
        for (int i = 0; i < side; ++i)
            dst[i] = w00 * ra[xa[i]] + w10 * ra[xb[i]] + w01 * rb[xa[i]] + w11 * rb[xb[i]];
    }
}

typedef struct {
    int count;
    int* index;
    double *value, *gx, *gy;
    double gxx, gxy, gyy;
} level_patch_t;

enum { PATCH_OK = 0, PATCH_TOO_SMALL = 1, PATCH_UNCONDITIONED = 2 };

/* build_level_patch, flow.cpp:77-126 */
static int build_level_patch(level_t img, double cx, double cy, int radius, double* ext_buf,
                             level_patch_t* p) {
    const int side = 2 * radius + 1;
    const int ext = radius + 1;
    const int ext_side = 2 * ext + 1;
    extract_patch(img, cx, cy, ext, ext_buf);
    const int x0 = (int)floor(cx), y0 = (int)floor(cy);
    p->count = 0;
    p->gxx = p->gxy = p->gyy = 0.0;
    for (int j = 0; j < side; ++j) {
        const int sy = y0 - radius + j;
        if (sy < 1 || sy + 2 > img.h - 1) continue;
        const double* mid = ext_buf + (size_t)(j + 1) * ext_side + 1;
        const double* up = mid - ext_side;
        const double* down = mid + ext_side;
        for (int i = 0; i < side; ++i) {
            const int sx = x0 - radius + i;
            if (sx < 1 || sx + 2 > img.w - 1) continue;
            const int k = p->count++;
            p->index[k] = j * side + i;
            p->value[k] = mid[i];
            const double dx = 0.5 * (mid[i + 1] - mid[i - 1]);
            const double dy = 0.5 * (down[i] - up[i]);
            p->gx[k] = dx;
            p->gy[k] = dy;
            p->gxx += dx * dx;
            p->gxy += dx * dy;
            p->gyy += dy * dy;
        }
    }
    if (p->count < maxi(25, side * side / 4)) return PATCH_TOO_SMALL;
    const double half_trace = 0.5 * (p->gxx + p->gyy);
    const double half_diff = 0.5 * (p->gxx - p->gyy);
    const double me = half_trace - sqrt(half_diff * half_diff + p->gxy * p->gxy);
    if (me < 1e-4 * (double)p->count) return PATCH_UNCONDITIONED;
    return PATCH_OK;
}

static inline int inside(level_t img, double x, double y) { /* flow.cpp:128-130 */
    return x >= 0.0 && y >= 0.0 && x <= img.w - 1.0 && y <= img.h - 1.0;
}

typedef struct {
    double* ext;
    double* cur;
    level_patch_t patch;
} lk_scratch_t;

static void scratch_init(lk_scratch_t* s, int radius) {
    const int side = 2 * radius + 1, es = 2 * radius + 3;
    s->ext = (double*)malloc(sizeof(double) * es * es);
    s->cur = (double*)malloc(sizeof(double) * side * side);
    s->patch.index = (int*)malloc(sizeof(int) * side * side);
    s->patch.value = (double*)malloc(sizeof(double) * side * side);
    s->patch.gx = (double*)malloc(sizeof(double) * side * side);
    s->patch.gy = (double*)malloc(sizeof(double) * side * side);
}

static void scratch_free(lk_scratch_t* s) {
    free(s->ext);
    free(s->cur);
    free(s->patch.index);
    free(s->patch.value);
    free(s->patch.gx);
    free(s->patch.gy);
}

/* track_one, flow.cpp:132-227 */
static int track_one(const stabgpu_pyramid* prev, const stabgpu_pyramid* cur, double px, double py,
                     const stabgpu_flow_cfg* cfg, lk_scratch_t* s, double* ox, double* oy) {
    const int levels = prev->levels;
    const int radius = cfg->window_radius;
    const int side = 2 * radius + 1;
    level_patch_t* patch = &s->patch;
    int start_level = 0;
    for (int level = levels - 1; level > 0; --level) {
        if (mini(prev->width[level], prev->height[level]) >= side) {
            start_level = level;
            break;
        }
    }
    double gx_flow = 0.0, gy_flow = 0.0;
    *ox = px;
    *oy = py;
    for (int level = start_level; level >= 0; --level) {
        const level_t pimg = level_of(prev, level);
        const level_t cimg = level_of(cur, level);
        const double scale = (double)(1u << level);
        const double plx = px / scale, ply = py / scale;
        if (!inside(pimg, plx, ply)) return 0;
        const int status = build_level_patch(pimg, plx, ply, radius, s->ext, patch);
        if (status == PATCH_UNCONDITIONED) return 0;
        if (status == PATCH_TOO_SMALL) {
            if (level == 0) return 0;
            gx_flow *= 2.0;
            gy_flow *= 2.0;
            continue;
        }
        const double det = patch->gxx * patch->gyy - patch->gxy * patch->gxy;
        double vx = 0.0, vy = 0.0;
        int diverged = 0;
        for (int it = 0; it < cfg->max_iterations; ++it) {
            const double qx = plx + gx_flow + vx, qy = ply + gy_flow + vy;
            if (!inside(cimg, qx, qy)) {
                diverged = 1;
                break;
            }
            extract_patch(cimg, qx, qy, radius, s->cur);
            double bx = 0.0, by = 0.0;
            for (int k = 0; k < patch->count; ++k) {
                const double di = patch->value[k] - s->cur[patch->index[k]];
                bx += di * patch->gx[k];
                by += di * patch->gy[k];
            }
            const double dx = (patch->gyy * bx - patch->gxy * by) / det;
            const double dy = (patch->gxx * by - patch->gxy * bx) / det;
            vx += dx;
            vy += dy;
            if (vx * vx + vy * vy > (double)radius * radius) {
                diverged = 1;
                break;
            }
            if (dx * dx + dy * dy < cfg->epsilon * cfg->epsilon) break;
        }
        if (diverged && level == 0) return 0;
        if (!diverged) {
            gx_flow += vx;
            gy_flow += vy;
        }
        if (level > 0) {
            gx_flow *= 2.0;
            gy_flow *= 2.0;
        }
    }
    const double rx = px + gx_flow, ry = py + gy_flow;
    if (!inside(level_of(cur, 0), rx, ry)) return 0;
    *ox = rx;
    *oy = ry;
    return 1;
}

static int check_pyramids(const stabgpu_pyramid* a, const stabgpu_pyramid* b) { /* flow.cpp:229-239 */
    if (a->levels < 1 || b->levels < 1 || a->levels != b->levels)
        return fail(STABGPU_INVALID_INPUT, "pyramids must have matching level counts");
    for (int i = 0; i < a->levels; ++i)
        if (a->width[i] != b->width[i] || a->height[i] != b->height[i])
            return fail(STABGPU_INVALID_INPUT, "pyramid levels differ in size");
    return STABGPU_OK;
}

/* track_lk, flow.cpp:243-256 */
int orc_track_lk(const stabgpu_pyramid* prev, const stabgpu_pyramid* cur, const double* xy, int n,
                 const stabgpu_flow_cfg* cfg, double* out_xy, uint8_t* ok) {
    int rc = validate_flow(cfg);
    if (rc) return rc;
    rc = check_pyramids(prev, cur);
    if (rc) return rc;
    if (cfg->window_radius > 31)
        return fail(STABGPU_INVALID_CONFIG, "window_radius above 31 is not supported");
    lk_scratch_t s;
    scratch_init(&s, cfg->window_radius);
    for (int i = 0; i < n; ++i)
        ok[i] = (uint8_t)track_one(prev, cur, xy[2 * i], xy[2 * i + 1], cfg, &s, &out_xy[2 * i],
                                   &out_xy[2 * i + 1]);
    scratch_free(&s);
    return STABGPU_OK;
}

/* weed_tracks, flow.cpp:258-280 */
int orc_weed_tracks(const stabgpu_pyramid* prev, const stabgpu_pyramid* cur, const double* prev_xy,
                    const double* cur_xy, int n, const stabgpu_flow_cfg* cfg, double* keep_prev,
                    double* keep_cur, int* n_out) {
    *n_out = 0;
    if (n == 0) return STABGPU_OK;
    double* back = (double*)malloc(sizeof(double) * 2 * n);
    uint8_t* ok = (uint8_t*)malloc(n);
    int rc = orc_track_lk(cur, prev, cur_xy, n, cfg, back, ok);
    if (rc) {
        free(back);
        free(ok);
        return rc;
    }
    const double limit2 = cfg->fb_threshold * cfg->fb_threshold;
    int m = 0;
    for (int i = 0; i < n; ++i) {
        if (!ok[i]) continue;
        const double dx = back[2 * i] - prev_xy[2 * i];
        const double dy = back[2 * i + 1] - prev_xy[2 * i + 1];
        if (dx * dx + dy * dy <= limit2) {
            keep_prev[2 * m] = prev_xy[2 * i];
            keep_prev[2 * m + 1] = prev_xy[2 * i + 1];
            keep_cur[2 * m] = cur_xy[2 * i];
            keep_cur[2 * m + 1] = cur_xy[2 * i + 1];
            ++m;
        }
    }
    *n_out = m;
    free(back);
    free(ok);
    return STABGPU_OK;
}

/* ------------------------------------------------------------------ */
/* motion                                                              */
/* ------------------------------------------------------------------ */

typedef struct {
    double src_cx, src_cy, dst_cx, dst_cy, dot, cross, src_norm;
} procrustes_t;

/* accumulate, motion.cpp:17-46 */
static int accumulate(const double* p, const double* q, int n, procrustes_t* s) {
    if (n < 2) return fail(STABGPU_DEGENERATE_INPUT, "estimation needs at least 2 point pairs");
    memset(s, 0, sizeof *s);
    for (int i = 0; i < n; ++i) {
        s->src_cx += p[2 * i];
        s->src_cy += p[2 * i + 1];
        s->dst_cx += q[2 * i];
        s->dst_cy += q[2 * i + 1];
    }
    const double dn = (double)(size_t)n;
    s->src_cx /= dn;
    s->src_cy /= dn;
    s->dst_cx /= dn;
    s->dst_cy /= dn;
    for (int i = 0; i < n; ++i) {
        const double x = p[2 * i] - s->src_cx, y = p[2 * i + 1] - s->src_cy;
        const double xp = q[2 * i] - s->dst_cx, yp = q[2 * i + 1] - s->dst_cy;
        s->dot += x * xp + y * yp;
        s->cross += x * yp - y * xp;
        s->src_norm += x * x + y * y;
    }
    if (s->src_norm == 0.0) return fail(STABGPU_DEGENERATE_INPUT, "all source points coincide");
    return STABGPU_OK;
}

/* finish, motion.cpp:48-58 */
static void finish(const procrustes_t* s, double theta, double scale, int kind,
                   stabgpu_transform* t) {
    t->theta = theta;
    t->s = scale;
    t->kind = kind;
    const double c = scale * cos(theta), sn = scale * sin(theta);
    t->tx = s->dst_cx - (c * s->src_cx - sn * s->src_cy);
    t->ty = s->dst_cy - (sn * s->src_cx + c * s->src_cy);
}

/* estimate_similarity / estimate_rigid, motion.cpp:62-76 */
int orc_estimate(const double* p, const double* q, int n, int kind, stabgpu_transform* out) {
    procrustes_t s;
    int rc = accumulate(p, q, n, &s);
    if (rc) return rc;
    const double theta = atan2(s.cross, s.dot);
    if (kind == STABGPU_RIGID) {
        finish(&s, theta, 1.0, STABGPU_RIGID, out);
        return STABGPU_OK;
    }
    const double scale = (cos(theta) * s.dot + sin(theta) * s.cross) / s.src_norm;
    if (!(scale > 0.0) || !isfinite(scale))
        return fail(STABGPU_DEGENERATE_INPUT, "similarity fit produced a non-positive scale");
    finish(&s, theta, scale, STABGPU_SIMILARITY, out);
    return STABGPU_OK;
}

/* rms_residual, motion.cpp:78-90 with SimilarityTransform::apply, transform.cpp:7-11 */
int orc_rms_residual(const double* p, const double* q, int n, const stabgpu_transform* t,
                     double* out) {
    if (n == 0) return fail(STABGPU_DEGENERATE_INPUT, "rms_residual needs a non-empty track set");
    double acc = 0.0;
    for (int i = 0; i < n; ++i) {
        const double c = t->s * cos(t->theta), sn = t->s * sin(t->theta);
        const double mx = c * p[2 * i] - sn * p[2 * i + 1] + t->tx;
        const double my = sn * p[2 * i] + c * p[2 * i + 1] + t->ty;
        const double dx = q[2 * i] - mx, dy = q[2 * i + 1] - my;
        acc += dx * dx + dy * dy;
    }
    *out = sqrt(acc / (double)(size_t)n);
    return STABGPU_OK;
}

/* ---- RANSAC (new; no reference counterpart) ----------------
 * Counter-based sampling: hypothesis h of frame f draws the index pair from
 * splitmix64 finalisers of (seed, f, h), so any worker can score any
 * hypothesis.  Minimal 2-point model anchored at the pair midpoints; only
 * correctly rounded + - * / sqrt, fixed evaluation order, no fused
 * multiply-add: the GPU reproduces every inlier count bit for bit.  Winner =
 * most inliers, ties to the lowest h.  Fewer than min_tracks inliers (or no
 * valid hypothesis) falls back to all pairs.  The refit is estimate_* on the
 * inlier subset in input order. */
static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

static void ransac_pair(uint64_t seed, int64_t frame, int h, int n, int* i, int* j) {
    const uint64_t key = mix64(seed ^ mix64((uint64_t)frame + 0x9e3779b97f4a7c15ULL));
    const uint64_t u = mix64(key + (uint64_t)(h + 1) * 0x9e3779b97f4a7c15ULL);
    *i = (int)((uint32_t)(u >> 32) % (uint32_t)n);
    int jj = (int)((uint32_t)u % (uint32_t)(n - 1));
    if (jj >= *i) ++jj;
    *j = jj;
}

static int ransac_model(const double* p, const double* q, int i, int j, int kind, double* m) {
    const double mpx = 0.5 * (p[2 * i] + p[2 * j]), mpy = 0.5 * (p[2 * i + 1] + p[2 * j + 1]);
    const double mqx = 0.5 * (q[2 * i] + q[2 * j]), mqy = 0.5 * (q[2 * i + 1] + q[2 * j + 1]);
    const double ax = p[2 * j] - p[2 * i], ay = p[2 * j + 1] - p[2 * i + 1];
    const double bx = q[2 * j] - q[2 * i], by = q[2 * j + 1] - q[2 * i + 1];
    const double norm = ax * ax + ay * ay;
    if (norm == 0.0) return 0;
    double a = (ax * bx + ay * by) / norm;
    double b = (ax * by - ay * bx) / norm;
    if (kind == STABGPU_RIGID) {
        const double r = sqrt(a * a + b * b);
        if (r == 0.0) return 0;
        a = a / r;
        b = b / r;
    }
    m[0] = a;
    m[1] = b;
    m[2] = mqx - (a * mpx - b * mpy);
    m[3] = mqy - (b * mpx + a * mpy);
    return 1;
}

static inline int ransac_inlier(const double* m, double px, double py, double qx, double qy,
                                double thr2) {
    const double ex = qx - ((m[0] * px - m[1] * py) + m[2]);
    const double ey = qy - ((m[1] * px + m[0] * py) + m[3]);
    return ex * ex + ey * ey <= thr2;
}

int orc_ransac_estimate(const double* p, const double* q, int n, int kind,
                        const stabgpu_ransac_cfg* rc_, int min_tracks, int64_t frame_index,
                        stabgpu_transform* out, uint8_t* inliers, int* n_inliers) {
    if (n < 2) return fail(STABGPU_DEGENERATE_INPUT, "estimation needs at least 2 point pairs");
    int best = -1, best_count = 0;
    double best_m[4] = {0, 0, 0, 0};
    if (rc_ && rc_->iterations > 0) {
        const double thr2 = rc_->threshold * rc_->threshold;
        for (int h = 0; h < rc_->iterations; ++h) {
            int i, j;
            double m[4];
            ransac_pair(rc_->seed, frame_index, h, n, &i, &j);
            if (!ransac_model(p, q, i, j, kind, m)) continue;
            int cnt = 0;
            for (int k = 0; k < n; ++k)
                cnt += ransac_inlier(m, p[2 * k], p[2 * k + 1], q[2 * k], q[2 * k + 1], thr2);
            if (cnt > best_count) {
                best_count = cnt;
                best = h;
                memcpy(best_m, m, sizeof best_m);
            }
        }
    }
    if (best < 0 || best_count < min_tracks) {
        if (inliers) memset(inliers, 1, (size_t)n);
        *n_inliers = n;
        return orc_estimate(p, q, n, kind, out);
    }
    const double thr2 = rc_->threshold * rc_->threshold;
    double* sp = (double*)malloc(sizeof(double) * 2 * n);
    double* sq = (double*)malloc(sizeof(double) * 2 * n);
    int m = 0;
    for (int k = 0; k < n; ++k) {
        const int in = ransac_inlier(best_m, p[2 * k], p[2 * k + 1], q[2 * k], q[2 * k + 1], thr2);
        if (inliers) inliers[k] = (uint8_t)in;
        if (in) {
            sp[2 * m] = p[2 * k];
            sp[2 * m + 1] = p[2 * k + 1];
            sq[2 * m] = q[2 * k];
            sq[2 * m + 1] = q[2 * k + 1];
            ++m;
        }
    }
    *n_inliers = m;
    int rc = orc_estimate(sp, sq, m, kind, out);
    free(sp);
    free(sq);
    return rc;
}

/* extract_delta, motion.cpp:92-101 */
void orc_extract_delta(const stabgpu_transform* t, stabgpu_delta* d) {
    d->dx = t->tx;
    d->dy = t->ty;
    d->da = t->theta;
    d->dls = t->kind == STABGPU_RIGID ? 0.0 : log(t->s);
    d->kind = t->kind;
    d->skipped = 0;
}

/* delta_to_transform, motion.cpp:103-111 */
void orc_delta_to_transform(double dx, double dy, double da, double dls, stabgpu_transform* t) {
    t->tx = dx;
    t->ty = dy;
    t->theta = da;
    t->s = exp(dls);
    t->kind = STABGPU_SIMILARITY;
}

/* Trajectory::append (smoothing.cpp:16-24), smooth_at on a complete
 * trajectory (26-46) and correction (48-57). */
int orc_trajectory_corrections(const stabgpu_delta* d, int n, int radius, stabgpu_transform* out) {
    if (radius < 1) return fail(STABGPU_INVALID_CONFIG, "smoothing radius must be >= 1");
    double* cum = (double*)malloc(sizeof(double) * 4 * (size_t)(n > 0 ? n : 1));
    double c[4] = {0, 0, 0, 0};
    for (int i = 0; i < n; ++i) {
        c[0] += d[i].dx;
        c[1] += d[i].dy;
        c[2] += d[i].da;
        c[3] += d[i].dls;
        memcpy(cum + 4 * i, c, sizeof c);
    }
    for (int i = 0; i < n; ++i) {
        const int lo = i >= radius ? i - radius : 0;
        const int hi = mini(i + radius, n - 1);
        double s[4] = {0, 0, 0, 0};
        for (int j = lo; j <= hi; ++j)
            for (int k = 0; k < 4; ++k) s[k] += cum[4 * j + k];
        const double cnt = (double)(size_t)(hi - lo + 1);
        double sm[4];
        for (int k = 0; k < 4; ++k) sm[k] = s[k] / cnt;
        orc_delta_to_transform(sm[0] - cum[4 * i], sm[1] - cum[4 * i + 1], sm[2] - cum[4 * i + 2],
                               sm[3] - cum[4 * i + 3], &out[i]);
    }
    free(cum);
    return STABGPU_OK;
}

/* ------------------------------------------------------------------ */
/* sequence driver: Tracker::advance (flow.cpp:297-337), ModelSelector   */
/* (motion.cpp:113-191), MotionStage (pipeline.cpp:75-111), run_offline */
/* (pipeline.cpp:182-235)                                               */
/* ------------------------------------------------------------------ */

/* validate(StabConfig), pipeline.cpp:17-28, with the per-record checks of
 * features.cpp:10-26, flow.cpp:10-21, smoothing.cpp:10-14, motion.cpp:113-120 */
static int validate_config(const stabgpu_config* c) {
    int rc = validate_detect(&c->detect);
    if (rc) return rc;
    rc = validate_flow(&c->flow);
    if (rc) return rc;
    if (c->smooth_radius < 1) return fail(STABGPU_INVALID_CONFIG, "smoothing radius must be >= 1");
    if (c->selector.dwell < 1) return fail(STABGPU_INVALID_CONFIG, "dwell must be >= 1");
    if (c->selector.margin < 0.0) return fail(STABGPU_INVALID_CONFIG, "margin must be >= 0");
    if (!(c->crop_ratio >= 0.0 && c->crop_ratio < 0.25))
        return fail(STABGPU_INVALID_CONFIG, "crop_ratio must lie in [0, 0.25)");
    if (c->queue_capacity < 2 * (size_t)c->smooth_radius + 4)
        return fail(STABGPU_INVALID_CONFIG, "queue_capacity must be >= 2*radius + 4");
    if (c->ransac.iterations < 0 || (c->ransac.iterations > 0 && !(c->ransac.threshold > 0.0)))
        return fail(STABGPU_INVALID_CONFIG, "ransac needs iterations >= 0 and threshold > 0");
    return STABGPU_OK;
}

typedef struct {
    int mode, dwell, current, since, pending;
    double margin;
} selector_t;

static void sel_advance(selector_t* s) { s->since = (s->since + 1) % s->dwell; }

static void sel_note_skipped(selector_t* s) { /* motion.cpp:185-191 */
    if (s->since == 0) s->pending = 1;
    sel_advance(s);
}

/* ModelSelector::select, motion.cpp:143-184, with the robust estimator. */
static int sel_select(selector_t* s, const double* p, const double* q, int n,
                      const stabgpu_config* cfg, int64_t frame, stabgpu_transform* out,
                      int* n_inl, int* decision) {
    int rc = 0, ni = 0;
    *decision = 0;
    if (s->since == 0) s->pending = 1;
    const stabgpu_ransac_cfg* rcfg = &cfg->ransac;
    const int mt = cfg->flow.min_tracks;
    if (s->mode == STABGPU_FORCE_RIGID || s->mode == STABGPU_FORCE_SIMILARITY) {
        const int kind = s->mode == STABGPU_FORCE_RIGID ? STABGPU_RIGID : STABGPU_SIMILARITY;
        rc = orc_ransac_estimate(p, q, n, kind, rcfg, mt, frame, out, NULL, &ni);
        if (rc) return rc;
        if (s->pending) {
            s->current = kind;
            s->pending = 0;
            *decision = 1;
        }
    } else if (s->pending) {
        stabgpu_transform r, sim;
        int nr = 0, ns = 0;
        rc = orc_ransac_estimate(p, q, n, STABGPU_RIGID, rcfg, mt, frame, &r, NULL, &nr);
        if (rc) return rc;
        rc = orc_ransac_estimate(p, q, n, STABGPU_SIMILARITY, rcfg, mt, frame, &sim, NULL, &ns);
        if (rc) return rc;
        double er, es;
        orc_rms_residual(p, q, n, &r, &er);
        orc_rms_residual(p, q, n, &sim, &es);
        if (er <= es * (1.0 + s->margin)) {
            s->current = STABGPU_RIGID;
            *out = r;
            ni = nr;
        } else {
            s->current = STABGPU_SIMILARITY;
            *out = sim;
            ni = ns;
        }
        s->pending = 0;
        *decision = 1;
    } else {
        rc = orc_ransac_estimate(p, q, n, s->current, rcfg, mt, frame, out, NULL, &ni);
        if (rc) return rc;
    }
    *n_inl = ni;
    sel_advance(s);
    return STABGPU_OK;
}

int orc_stabilize_sequence(const uint8_t* y, const uint8_t* cb, const uint8_t* cr, int n, int w,
                           int h, int cw, int ch, const stabgpu_config* cfg, uint8_t* oy,
                           uint8_t* ocb, uint8_t* ocr, stabgpu_frame_record* rec) {
    int rc = validate_config(cfg);
    if (rc) return rc;
    if (n < 2) return fail(STABGPU_INVALID_INPUT, "stabilization needs at least 2 frames");
    const stabgpu_flow_cfg* fc = &cfg->flow;
    const size_t pb = orc_pyramid_bytes(w, h, fc->max_levels);
    stabgpu_pyramid pyr[2];
    pyr[0].data = (uint8_t*)malloc(pb);
    pyr[1].data = (uint8_t*)malloc(pb);
    const int maxc = cfg->detect.max_corners;
    double* pts = (double*)malloc(sizeof(double) * 2 * maxc);
    double* fwd = (double*)malloc(sizeof(double) * 2 * maxc);
    double* pok = (double*)malloc(sizeof(double) * 2 * maxc);
    double* cok = (double*)malloc(sizeof(double) * 2 * maxc);
    double* kp = (double*)malloc(sizeof(double) * 2 * maxc);
    double* kc = (double*)malloc(sizeof(double) * 2 * maxc);
    double* score = (double*)malloc(sizeof(double) * maxc);
    uint8_t* ok = (uint8_t*)malloc(maxc);
    stabgpu_delta* deltas = (stabgpu_delta*)calloc((size_t)n, sizeof(stabgpu_delta));
    stabgpu_transform* corr = (stabgpu_transform*)calloc((size_t)n, sizeof(stabgpu_transform));
    selector_t sel = {cfg->selector.mode, cfg->selector.dwell,
                      cfg->selector.mode == STABGPU_FORCE_SIMILARITY ? STABGPU_SIMILARITY
                                                                     : STABGPU_RIGID,
                      0, 1, cfg->selector.margin};
    int npts = 0, since_detect = 0, cur = 0;
    for (int f = 0; f < n && !rc; ++f) {
        const uint8_t* frame = y + (size_t)f * w * h;
        rc = orc_build_pyramid(frame, w, h, fc->max_levels, &pyr[cur]);
        if (rc) break;
        stabgpu_frame_record* r = rec ? &rec[f] : NULL;
        stabgpu_delta d;
        memset(&d, 0, sizeof d);
        if (r) memset(r, 0, sizeof *r);
        if (f == 0) { /* Tracker::advance first frame + MotionStage FirstFrame */
            rc = orc_detect_corners(frame, w, h, &cfg->detect, pts, score, &npts);
            since_detect = 0;
            sel_note_skipped(&sel);
            d.kind = sel.current;
            if (r) r->frame_kind = STABGPU_FRAME_FIRST;
        } else {
            const stabgpu_pyramid* prev = &pyr[cur ^ 1];
            int nk = 0;
            if (npts > 0) {
                rc = orc_track_lk(prev, &pyr[cur], pts, npts, fc, fwd, ok);
                if (rc) break;
                int m = 0;
                for (int i = 0; i < npts; ++i)
                    if (ok[i]) {
                        pok[2 * m] = pts[2 * i];
                        pok[2 * m + 1] = pts[2 * i + 1];
                        cok[2 * m] = fwd[2 * i];
                        cok[2 * m + 1] = fwd[2 * i + 1];
                        ++m;
                    }
                rc = orc_weed_tracks(prev, &pyr[cur], pok, cok, m, fc, kp, kc, &nk);
                if (rc) break;
            }
            memcpy(pts, kc, sizeof(double) * 2 * nk);
            npts = nk;
            if (++since_detect >= fc->redetect_interval) {
                rc = orc_detect_corners(frame, w, h, &cfg->detect, pts, score, &npts);
                if (rc) break;
                since_detect = 0;
            }
            if (r) r->n_tracks = nk;
            if (nk < fc->min_tracks) {
                sel_note_skipped(&sel);
                d.kind = sel.current;
                d.skipped = 1;
                if (r) r->frame_kind = STABGPU_FRAME_SKIPPED;
            } else {
                stabgpu_transform t;
                int ni = 0, dec = 0;
                rc = sel_select(&sel, kp, kc, nk, cfg, f, &t, &ni, &dec);
                if (rc) break;
                orc_extract_delta(&t, &d);
                if (r) {
                    r->frame_kind = STABGPU_FRAME_TRACKED;
                    r->n_inliers = ni;
                    r->decision = dec;
                }
            }
        }
        deltas[f] = d;
        if (r) r->delta = d;
        cur ^= 1;
    }
    if (!rc) rc = orc_trajectory_corrections(deltas, n, cfg->smooth_radius, corr);
    for (int f = 0; f < n && !rc; ++f) {
        if (rec) rec[f].correction = corr[f];
        if (oy) {
            const size_t lo = (size_t)f * w * h, co = (size_t)f * cw * ch;
            rc = orc_compose_stabilized(y + lo, cb ? cb + co : NULL, cr ? cr + co : NULL, w, h, cw,
                                        ch, &corr[f], cfg->crop_ratio, oy + lo,
                                        ocb ? ocb + co : NULL, ocr ? ocr + co : NULL);
        }
    }
    free(pyr[0].data);
    free(pyr[1].data);
    free(pts);
    free(fwd);
    free(pok);
    free(cok);
    free(kp);
    free(kc);
    free(score);
    free(ok);
    free(deltas);
    free(corr);
    return rc;
}

/* ------------------------------------------------------------------ */
/* BT.601 full-range conversions (media_io.cpp:75-89, 568-570) and the
 * inter-frame PSNR pair (synth_eval.cpp:214-240). */
static uint8_t clamp_lround(double v) {
    const long r = lround(v);
    return (uint8_t)(r < 0 ? 0 : (r > 255 ? 255 : r));
}

void orc_rgb_to_ycbcr(const uint8_t* rgb, size_t npx, uint8_t* y, uint8_t* cb, uint8_t* cr) {
    for (size_t i = 0; i < npx; ++i) {
        const unsigned r = rgb[3 * i], g = rgb[3 * i + 1], b = rgb[3 * i + 2];
        y[i] = (uint8_t)((299 * r + 587 * g + 114 * b + 500) / 1000); /* luma_bt601 */
        cb[i] = clamp_lround(128.0 - 0.168736 * r - 0.331264 * g + 0.5 * b);
        cr[i] = clamp_lround(128.0 + 0.5 * r - 0.418688 * g - 0.081312 * b);
    }
}

void orc_ycbcr_to_rgb(const uint8_t* y, const uint8_t* cb, const uint8_t* cr, size_t npx, uint8_t* rgb) {
    for (size_t i = 0; i < npx; ++i) {
        const double du = cb[i] - 128.0, dv = cr[i] - 128.0;
        rgb[3 * i] = clamp_lround(y[i] + 1.402 * dv);
        rgb[3 * i + 1] = clamp_lround(y[i] - 0.344136 * du - 0.714136 * dv);
        rgb[3 * i + 2] = clamp_lround(y[i] + 1.772 * du);
    }
}

int orc_psnr_pair(const uint8_t* a, const uint8_t* b, int w, int h, double crop, double* out) {
    if (!(crop >= 0.0 && crop < 0.5)) return fail(STABGPU_INVALID_CONFIG, "psnr crop_ratio must lie in [0, 0.5)");
    const int mx = (int)lround(crop * w), my = (int)lround(crop * h);
    double acc = 0.0;
    long long n = 0;
    for (int y = my; y < h - my; ++y)
        for (int x = mx; x < w - mx; ++x) {
            const double d = (double)a[(size_t)y * w + x] - b[(size_t)y * w + x];
            acc += d * d;
            ++n;
        }
    if (n == 0) return fail(STABGPU_INVALID_INPUT, "PSNR crop region is empty");
    const double mse = acc / (double)n;
    *out = mse == 0.0 ? INFINITY : 10.0 * log10(255.0 * 255.0 / mse);
    return STABGPU_OK;
}
