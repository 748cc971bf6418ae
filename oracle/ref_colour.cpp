// ref_colour.cpp — TEST INFRASTRUCTURE ONLY: C entry points to the
// reference's own BT.601 conversions (media_io.cpp:75-89, 568-570), which
// live in that file's anonymous namespace.  The unmodified source file is
// compiled as part of this translation unit (libpng is replaced by the
// failing stub in oracle/png_stub; the PNG paths are never called).
#include "media_io.cpp"  // the reference source file itself (-I $(REF)/proj/src, oracle/Makefile)

extern "C" {

void ref_rgb_to_ycbcr(const std::uint8_t* rgb, std::size_t npx, std::uint8_t* y, std::uint8_t* cb,
                      std::uint8_t* cr) {
    for (std::size_t i = 0; i < npx; ++i) {
        const std::uint8_t r = rgb[3 * i], g = rgb[3 * i + 1], b = rgb[3 * i + 2];
        y[i] = stab::luma_bt601(r, g, b);
        cb[i] = stab::chroma_cb(r, g, b);
        cr[i] = stab::chroma_cr(r, g, b);
    }
}

void ref_ycbcr_to_rgb(const std::uint8_t* y, const std::uint8_t* cb, const std::uint8_t* cr, std::size_t npx,
                      std::uint8_t* rgb) {
    for (std::size_t i = 0; i < npx; ++i) {
        const stab::Rgb c = stab::yuv_to_rgb(y[i], cb[i], cr[i]);
        rgb[3 * i] = c.r;
        rgb[3 * i + 1] = c.g;
        rgb[3 * i + 2] = c.b;
    }
}

}  // extern "C"
