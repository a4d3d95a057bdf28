/* png.h — capture stand-in for the libpng API subset image_io.cpp uses. TEST INFRASTRUCTURE.
 *
 * libpng is absent from this image, which is the only thing keeping the reference's own
 * image_io.cpp (write_png_rgb8 / write_png_gray8 / write_png_gray16 / write_pfm) out of
 * oracle/_ref. This header declares just the calls image_io.cpp makes; png_capture.cpp
 * implements the write side by recording the IHDR fields and the row bytes the reference hands
 * to png_write_image (no zlib, no file format), so tests can compare those bytes with the GPU
 * encoder's. The read side reports an error through the caller's error callback.
 * Written from the public libpng API names; no libpng code is included. */
#ifndef GSIM_PNG_CAPTURE_H
#define GSIM_PNG_CAPTURE_H

#include <stddef.h>
#include <stdio.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef unsigned char png_byte;
typedef png_byte* png_bytep;
typedef const png_byte* png_const_bytep;
typedef png_byte** png_bytepp;
typedef unsigned int png_uint_32;
typedef size_t png_size_t;
typedef const char* png_const_charp;
typedef void* png_voidp;
typedef struct png_struct_def png_struct;
typedef png_struct* png_structp;
typedef png_struct** png_structpp;
typedef struct png_info_def png_info;
typedef png_info* png_infop;
typedef png_info** png_infopp;
typedef void (*png_error_ptr)(png_structp, png_const_charp);

#define PNG_LIBPNG_VER_STRING "capture"
#define PNG_COLOR_TYPE_GRAY 0
#define PNG_COLOR_TYPE_RGB 2
#define PNG_COLOR_TYPE_GRAY_ALPHA 4
#define PNG_INTERLACE_NONE 0
#define PNG_COMPRESSION_TYPE_DEFAULT 0
#define PNG_FILTER_TYPE_DEFAULT 0

png_structp png_create_write_struct(png_const_charp ver, png_voidp err_ptr, png_error_ptr err_fn,
                                    png_error_ptr warn_fn);
png_structp png_create_read_struct(png_const_charp ver, png_voidp err_ptr, png_error_ptr err_fn,
                                   png_error_ptr warn_fn);
png_infop png_create_info_struct(png_structp png);
void png_destroy_write_struct(png_structpp png, png_infopp info);
void png_destroy_read_struct(png_structpp png, png_infopp info, png_infopp end_info);
void png_init_io(png_structp png, FILE* fp);
void png_set_IHDR(png_structp png, png_infop info, png_uint_32 width, png_uint_32 height,
                  int bit_depth, int color_type, int interlace, int compression, int filter);
void png_write_info(png_structp png, png_infop info);
void png_write_image(png_structp png, png_bytepp rows);
void png_write_end(png_structp png, png_infop info);
int png_sig_cmp(png_const_bytep sig, size_t start, size_t n);
void png_set_sig_bytes(png_structp png, int n);
void png_read_info(png_structp png, png_infop info);
void png_set_expand(png_structp png);
png_byte png_get_bit_depth(png_structp png, png_infop info);
void png_set_strip_16(png_structp png);
void png_set_strip_alpha(png_structp png);
png_byte png_get_color_type(png_structp png, png_infop info);
void png_set_gray_to_rgb(png_structp png);
void png_read_update_info(png_structp png, png_infop info);
png_uint_32 png_get_image_width(png_structp png, png_infop info);
png_uint_32 png_get_image_height(png_structp png, png_infop info);
png_size_t png_get_rowbytes(png_structp png, png_infop info);
void png_read_image(png_structp png, png_bytepp rows);
void png_read_end(png_structp png, png_infop info);

/* capture accessors (not libpng API) */
const unsigned char* png_capture_last(int* width, int* height, int* bit_depth, int* color_type,
                                      size_t* size);

#ifdef __cplusplus
}
#endif

#endif /* GSIM_PNG_CAPTURE_H */
