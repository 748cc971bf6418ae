/* Minimal libpng "simplified API" stub (TEST INFRASTRUCTURE ONLY).
 * libpng is absent from this image; the reference's media_io.cpp includes
 * <png.h> for its PNG reader/writer, which the checkers never call.  This
 * stub only lets oracle/ref_colour.cpp compile the reference's colour
 * conversion functions from their own source file; every PNG entry point
 * fails. */
#ifndef STAB_PNG_STUB_H
#define STAB_PNG_STUB_H
#include <stddef.h>
#include <stdint.h>
typedef uint32_t png_uint_32;
typedef struct {
    void* opaque;
    png_uint_32 version, width, height, format, flags, colormap_entries, warning_or_error;
    char message[64];
} png_image;
#define PNG_IMAGE_VERSION 1
#define PNG_FORMAT_GRAY 0
#define PNG_FORMAT_RGB 2
#define PNG_IMAGE_SIZE(img) ((size_t)(img).width * (img).height * ((img).format == PNG_FORMAT_RGB ? 3 : 1))
static inline int png_image_begin_read_from_file(png_image*, const char*) { return 0; }
static inline int png_image_finish_read(png_image*, const void*, void*, ptrdiff_t, void*) { return 0; }
static inline void png_image_free(png_image*) {}
static inline int png_image_write_to_file(png_image*, const char*, int, const void*, ptrdiff_t, const void*) {
    return 0;
}
#endif
