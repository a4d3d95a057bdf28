// png_capture.cpp — write-side capture for the png.h stand-in. TEST INFRASTRUCTURE.
// Records what the reference's write_png (image_io.cpp:47-72) passes to libpng: IHDR fields and
// the image rows, concatenated top-down. One thread-local capture (the tests are sequential).
#include "png.h"

#include <cstring>
#include <vector>

struct png_struct_def {
    png_error_ptr err = nullptr;
    bool write = false;
    int width = 0, height = 0, bit_depth = 0, color_type = 0;
};
struct png_info_def {
    int unused = 0;
};

namespace {
struct Capture {
    int width = 0, height = 0, bit_depth = 0, color_type = 0;
    std::vector<unsigned char> bytes;
};
thread_local Capture g_last;

int channels(int color_type) {
    switch (color_type) {
        case PNG_COLOR_TYPE_GRAY: return 1;
        case PNG_COLOR_TYPE_RGB: return 3;
        case PNG_COLOR_TYPE_GRAY_ALPHA: return 2;
        default: return 4;
    }
}
void unsupported(png_structp png, const char* what) {
    if (png && png->err) png->err(png, what);  // the reference's handler throws io_error
}
}  // namespace

extern "C" {

png_structp png_create_write_struct(png_const_charp, png_voidp, png_error_ptr err_fn, png_error_ptr) {
    png_structp p = new png_struct_def;
    p->err = err_fn;
    p->write = true;
    return p;
}
png_structp png_create_read_struct(png_const_charp, png_voidp, png_error_ptr err_fn, png_error_ptr) {
    png_structp p = new png_struct_def;
    p->err = err_fn;
    return p;
}
png_infop png_create_info_struct(png_structp) { return new png_info_def; }
void png_destroy_write_struct(png_structpp png, png_infopp info) {
    if (png) { delete *png; *png = nullptr; }
    if (info) { delete *info; *info = nullptr; }
}
void png_destroy_read_struct(png_structpp png, png_infopp info, png_infopp end_info) {
    png_destroy_write_struct(png, info);
    if (end_info) { delete *end_info; *end_info = nullptr; }
}
void png_init_io(png_structp, FILE*) {}
void png_set_IHDR(png_structp png, png_infop, png_uint_32 width, png_uint_32 height, int bit_depth,
                  int color_type, int, int, int) {
    png->width = int(width);
    png->height = int(height);
    png->bit_depth = bit_depth;
    png->color_type = color_type;
}
void png_write_info(png_structp, png_infop) {}
void png_write_image(png_structp png, png_bytepp rows) {
    const size_t rowbytes = size_t(png->width) * channels(png->color_type) * (png->bit_depth / 8);
    g_last.width = png->width;
    g_last.height = png->height;
    g_last.bit_depth = png->bit_depth;
    g_last.color_type = png->color_type;
    g_last.bytes.resize(rowbytes * size_t(png->height));
    for (int y = 0; y < png->height; ++y)
        std::memcpy(g_last.bytes.data() + size_t(y) * rowbytes, rows[y], rowbytes);
}
void png_write_end(png_structp, png_infop) {}
int png_sig_cmp(png_const_bytep, size_t, size_t) { return 1; }
void png_set_sig_bytes(png_structp, int) {}
void png_read_info(png_structp png, png_infop) { unsupported(png, "capture shim: no PNG reader"); }
void png_set_expand(png_structp) {}
png_byte png_get_bit_depth(png_structp, png_infop) { return 8; }
void png_set_strip_16(png_structp) {}
void png_set_strip_alpha(png_structp) {}
png_byte png_get_color_type(png_structp, png_infop) { return PNG_COLOR_TYPE_RGB; }
void png_set_gray_to_rgb(png_structp) {}
void png_read_update_info(png_structp, png_infop) {}
png_uint_32 png_get_image_width(png_structp, png_infop) { return 0; }
png_uint_32 png_get_image_height(png_structp, png_infop) { return 0; }
png_size_t png_get_rowbytes(png_structp, png_infop) { return 0; }
void png_read_image(png_structp png, png_bytepp) { unsupported(png, "capture shim: no PNG reader"); }
void png_read_end(png_structp, png_infop) {}

const unsigned char* png_capture_last(int* width, int* height, int* bit_depth, int* color_type,
                                      size_t* size) {
    if (width) *width = g_last.width;
    if (height) *height = g_last.height;
    if (bit_depth) *bit_depth = g_last.bit_depth;
    if (color_type) *color_type = g_last.color_type;
    if (size) *size = g_last.bytes.size();
    return g_last.bytes.data();
}

}  // extern "C"
