/*
 * videogen.c — seeded synthetic UAV-style video for the BASELINE.json configs
 * (bench/test input generator; not part of the stabilization path).
 *
 * BASELINE.json configs[0..4] / SURVEY.md §8d describe the generator:
 *   texture : mid-grey 128 + N Gaussian blobs (sigma U[2,20] px, amplitude
 *             U[-80,80]) + Gaussian-blurred N(0,30) noise (sigma 1.5),
 *             clipped to [0,255].  The texture is a torus (blobs and blur wrap)
 *             so a crop can drift any distance without leaving it (SURVEY H9:
 *             a 2048^2 texture cannot hold 1000 frames of 1080p drift).
 *   frame i : similarity crop of the texture about the frame centre, drifting
 *             `drift` px/frame along +x, plus i.i.d. jitter (translation
 *             N(0,jit_t), rotation N(0,jit_rot), scale N(1,jit_scale));
 *             bilinear sampling, moving textured rectangles (outliers,
 *             40-120 px, velocity U[-4,4] px/frame, occluding, wrapping at the
 *             frame border), additive N(0,noise) noise, round, clip.
 *   colour  : R,G,B = value * per-sequence gains U[0.8,1.2]; the stabilizer
 *             sees BT.601 full-range Y/Cb/Cr 4:4:4 (the conversion the
 *             reference applies when reading colour input, media_io.cpp:83-89
 *             and 569-571).
 * Every random draw is a splitmix64 hash of (seed, stream, counters), so the
 * bytes do not depend on the thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct vg_config {
    int width, height, frames;
    int tex_size, blobs, objects, color;
    double drift, jit_t, jit_rot_deg, jit_scale, noise_sigma;
    uint64_t seed;
} vg_config;

typedef struct vg_handle {
    vg_config cfg;
    float* tex; /* tex_size^2, values in [0,255] */
    double gain[3];
    float ntab[65536]; /* inverse-CDF table of N(0,1) at 2^16 quantile midpoints */
    struct {
        int w, h;
        double x, y, vx, vy, ox, oy;
    } obj[64];
} vg_handle;

static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
static inline uint64_t hash3(uint64_t a, uint64_t b, uint64_t c) {
    return mix64(a ^ mix64(b + 0x9e3779b97f4a7c15ULL * (c + 1)));
}
static inline double u01(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }
static double gauss(uint64_t a, uint64_t b, uint64_t c) { /* Box-Muller on two hashed uniforms */
    double u1 = u01(hash3(a, b, 2 * c));
    const double u2 = u01(hash3(a, b, 2 * c + 1));
    if (u1 <= 0.0) u1 = 0x1.0p-53;
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

/* Acklam's rational approximation of the normal quantile (|rel err| < 1.2e-9). */
static double norm_ppf(double p) {
    static const double a[] = {-3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,
                               1.383577518672690e+02, -3.066479806614716e+01, 2.506628277459239e+00};
    static const double b[] = {-5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,
                               6.680131188771972e+01, -1.328068155288572e+01};
    static const double c[] = {-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00,
                               -2.549732539343734e+00, 4.374664141464968e+00, 2.938163982698783e+00};
    static const double d[] = {7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00,
                               3.754408661907416e+00};
    if (p < 0.02425) {
        const double q = sqrt(-2 * log(p));
        return (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
               ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1);
    }
    if (p > 1 - 0.02425) return -norm_ppf(1 - p);
    const double q = p - 0.5, r = q * q;
    return (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * q /
           (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1);
}

static inline int wrapi(int v, int n) {
    v %= n;
    return v < 0 ? v + n : v;
}

static void make_texture(vg_handle* g) {
    const int T = g->cfg.tex_size;
    const uint64_t seed = g->cfg.seed;
    double* acc = (double*)malloc(sizeof(double) * (size_t)T * T);
    double* tmp = (double*)malloc(sizeof(double) * (size_t)T * T);
    /* band-limited noise: N(0,30) blurred by a sigma-1.5 Gaussian (wrapped) */
#pragma omp parallel for schedule(static)
    for (int y = 0; y < T; ++y)
        for (int x = 0; x < T; ++x) acc[(size_t)y * T + x] = 30.0 * gauss(seed, 11, (uint64_t)y * T + x);
    double k[11], ks = 0.0;
    for (int i = -5; i <= 5; ++i) ks += (k[i + 5] = exp(-(i * i) / (2.0 * 1.5 * 1.5)));
    for (int i = 0; i < 11; ++i) k[i] /= ks;
#pragma omp parallel for schedule(static)
    for (int y = 0; y < T; ++y)
        for (int x = 0; x < T; ++x) {
            double s = 0.0;
            for (int i = -5; i <= 5; ++i) s += k[i + 5] * acc[(size_t)y * T + wrapi(x + i, T)];
            tmp[(size_t)y * T + x] = s;
        }
#pragma omp parallel for schedule(static)
    for (int y = 0; y < T; ++y)
        for (int x = 0; x < T; ++x) {
            double s = 0.0;
            for (int i = -5; i <= 5; ++i) s += k[i + 5] * tmp[(size_t)wrapi(y + i, T) * T + x];
            acc[(size_t)y * T + x] = 128.0 + s;
        }
    /* Gaussian blobs, truncated at 4 sigma, toroidal distance.  Rows are
     * partitioned across threads; each thread adds every blob's footprint
     * on its rows, so the sum order per pixel is the blob order. */
    const int nb = g->cfg.blobs;
    double* bp = (double*)malloc(sizeof(double) * 4 * (size_t)(nb > 0 ? nb : 1));
    for (int b = 0; b < nb; ++b) {
        bp[4 * b + 0] = u01(hash3(seed, 21, 4 * (uint64_t)b)) * T;
        bp[4 * b + 1] = u01(hash3(seed, 21, 4 * (uint64_t)b + 1)) * T;
        bp[4 * b + 2] = 2.0 + 18.0 * u01(hash3(seed, 21, 4 * (uint64_t)b + 2));
        bp[4 * b + 3] = -80.0 + 160.0 * u01(hash3(seed, 21, 4 * (uint64_t)b + 3));
    }
#pragma omp parallel for schedule(dynamic, 8)
    for (int y = 0; y < T; ++y) {
        for (int b = 0; b < nb; ++b) {
            const double cx = bp[4 * b], cy = bp[4 * b + 1], sg = bp[4 * b + 2], amp = bp[4 * b + 3];
            const int r = (int)ceil(4.0 * sg);
            double dy = y - cy;
            dy -= T * floor(dy / T + 0.5); /* toroidal */
            if (fabs(dy) > r) continue;
            const double inv = 1.0 / (2.0 * sg * sg);
            const int x0 = (int)floor(cx) - r, x1 = (int)floor(cx) + r + 1;
            for (int xi = x0; xi <= x1; ++xi) {
                const double dx = xi - cx;
                acc[(size_t)y * T + wrapi(xi, T)] += amp * exp(-(dx * dx + dy * dy) * inv);
            }
        }
    }
    for (size_t i = 0; i < (size_t)T * T; ++i) {
        const double v = acc[i];
        g->tex[i] = (float)(v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v));
    }
    free(bp);
    free(acc);
    free(tmp);
}

static inline double tex_at(const vg_handle* g, double u, double v) {
    const int T = g->cfg.tex_size, m = T - 1; /* power of two (checked in vg_create) */
    const double fu = floor(u), fv = floor(v);
    const int x0 = (int)(long long)fu & m, y0 = (int)(long long)fv & m;
    const int x1 = (x0 + 1) & m, y1 = (y0 + 1) & m;
    const double ax = u - fu, ay = v - fv;
    const float* r0 = g->tex + (size_t)y0 * T;
    const float* r1 = g->tex + (size_t)y1 * T;
    const double top = r0[x0] + ax * (r0[x1] - r0[x0]);
    const double bot = r1[x0] + ax * (r1[x1] - r1[x0]);
    return top + ay * (bot - top);
}

vg_handle* vg_create(const vg_config* cfg) {
    if (cfg->width < 16 || cfg->height < 16 || cfg->tex_size < 64 || cfg->objects > 64 ||
        (cfg->tex_size & (cfg->tex_size - 1)))
        return NULL;
    vg_handle* g = (vg_handle*)calloc(1, sizeof(vg_handle));
    g->cfg = *cfg;
    g->tex = (float*)malloc(sizeof(float) * (size_t)cfg->tex_size * cfg->tex_size);
    make_texture(g);
    for (int c = 0; c < 3; ++c) g->gain[c] = 0.8 + 0.4 * u01(hash3(cfg->seed, 31, (uint64_t)c));
    for (int i = 0; i < 65536; ++i) g->ntab[i] = (float)norm_ppf((i + 0.5) / 65536.0);
    for (int k = 0; k < cfg->objects; ++k) {
        uint64_t s = 41;
        g->obj[k].w = 40 + (int)(81 * u01(hash3(cfg->seed, s, 8 * (uint64_t)k)));
        g->obj[k].h = 40 + (int)(81 * u01(hash3(cfg->seed, s, 8 * (uint64_t)k + 1)));
        g->obj[k].x = cfg->width * u01(hash3(cfg->seed, s, 8 * (uint64_t)k + 2));
        g->obj[k].y = cfg->height * u01(hash3(cfg->seed, s, 8 * (uint64_t)k + 3));
        g->obj[k].vx = -4.0 + 8.0 * u01(hash3(cfg->seed, s, 8 * (uint64_t)k + 4));
        g->obj[k].vy = -4.0 + 8.0 * u01(hash3(cfg->seed, s, 8 * (uint64_t)k + 5));
        g->obj[k].ox = cfg->tex_size * u01(hash3(cfg->seed, s, 8 * (uint64_t)k + 6));
        g->obj[k].oy = cfg->tex_size * u01(hash3(cfg->seed, s, 8 * (uint64_t)k + 7));
    }
    return g;
}

void vg_destroy(vg_handle* g) {
    if (!g) return;
    free(g->tex);
    free(g);
}

/* Ground-truth jitter of frame i: (tx, ty, theta, s) about the frame centre. */
void vg_pose(const vg_handle* g, int i, double* out4) {
    const vg_config* c = &g->cfg;
    out4[0] = c->jit_t * gauss(c->seed, 51, 4 * (uint64_t)i);
    out4[1] = c->jit_t * gauss(c->seed, 51, 4 * (uint64_t)i + 1);
    out4[2] = c->jit_rot_deg * (3.14159265358979323846 / 180.0) * gauss(c->seed, 51, 4 * (uint64_t)i + 2);
    out4[3] = 1.0 + c->jit_scale * gauss(c->seed, 51, 4 * (uint64_t)i + 3);
}

static inline uint8_t rnd_u8(double v) {
    const long r = lround(v);
    return (uint8_t)(r < 0 ? 0 : (r > 255 ? 255 : r));
}

/* Renders frames [first, first+count) into y (and cb/cr when colour). */
int vg_render(const vg_handle* g, int first, int count, uint8_t* y, uint8_t* cb, uint8_t* cr) {
    const vg_config* c = &g->cfg;
    const int W = c->width, H = c->height;
    const double T = c->tex_size;
    const long long rows = (long long)count * H;
#pragma omp parallel for schedule(static)
    for (long long r = 0; r < rows; ++r) {
        const int fi = (int)(r / H), py = (int)(r % H);
        const int f = first + fi;
        double pose[4];
        vg_pose(g, f, pose);
        const double a = pose[3] * cos(pose[2]), b = pose[3] * sin(pose[2]);
        const double cx = 0.5 * T + c->drift * f + pose[0], cy = 0.5 * T + pose[1];
        const double yc = py - 0.5 * (H - 1);
        const size_t base = (size_t)fi * W * H + (size_t)py * W;
        /* outlier rectangles covering this row: [x0, x0+w) wrapped at W */
        int ok_n = 0, ob_k[64];
        double ob_x[64], ob_ly[64];
        for (int k = 0; k < c->objects; ++k) {
            double ox = g->obj[k].x + g->obj[k].vx * f, oy = g->obj[k].y + g->obj[k].vy * f;
            ox -= W * floor(ox / W);
            oy -= H * floor(oy / H);
            double ly = py - oy;
            if (ly < 0) ly += H;
            if (ly < g->obj[k].h) {
                ob_k[ok_n] = k;
                ob_x[ok_n] = ox;
                ob_ly[ok_n] = ly;
                ++ok_n;
            }
        }
        double u = cx - a * 0.5 * (W - 1) - b * yc, vv = cy - b * 0.5 * (W - 1) + a * yc;
        for (int px = 0; px < W; ++px) {
            double v = tex_at(g, u + a * px, vv + b * px);
            for (int q = 0; q < ok_n; ++q) { /* last object on top */
                double lx = px - ob_x[q];
                if (lx < 0) lx += W;
                const int k = ob_k[q];
                if (lx < g->obj[k].w) v = tex_at(g, g->obj[k].ox + lx, g->obj[k].oy + ob_ly[q]);
            }
            const uint64_t hsh = hash3(c->seed ^ 0xABCDEFULL, (uint64_t)f, (uint64_t)py * W + px);
            v += c->noise_sigma * g->ntab[hsh >> 48];
            if (!c->color) {
                y[base + px] = rnd_u8(v);
            } else {
                const uint8_t R = rnd_u8(v * g->gain[0]), G = rnd_u8(v * g->gain[1]), B = rnd_u8(v * g->gain[2]);
                /* BT.601 full range, as media_io.cpp:569-571 and 83-89 define it */
                y[base + px] = (uint8_t)((299 * R + 587 * G + 114 * B + 500) / 1000);
                cb[base + px] = rnd_u8(128.0 - 0.168736 * R - 0.331264 * G + 0.5 * B);
                cr[base + px] = rnd_u8(128.0 + 0.5 * R - 0.418688 * G - 0.081312 * B);
            }
        }
    }
    return 0;
}

void vg_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
