/* TEST INFRASTRUCTURE ONLY -- declaration-only stand-in for <png.h>.
 *
 * libpng is not installed in this image.  The reference's metrics.hpp and
 * train.hpp (SSIM/PSNR, mse/photometric loss, fit) include image.hpp only for
 * its Image type; image.hpp's PNG reader/writer (load_png / save_png) are
 * inline functions that the oracle shim never calls, so the compiler never
 * emits them and none of the names below is ever referenced at link time.
 * Declaring them lets the UNMODIFIED reference headers compile as they lie.
 * Any accidental use fails at load time (undefined symbol), never silently. */
#ifndef GB_ORACLE_STUB_PNG_H
#define GB_ORACLE_STUB_PNG_H
#include <setjmp.h>
#include <stddef.h>
#include <stdio.h>
#ifdef __cplusplus
extern "C" {
#endif
typedef unsigned char png_byte;
typedef png_byte *png_bytep;
typedef png_bytep *png_bytepp;
typedef struct png_struct_def png_struct;
typedef png_struct *png_structp;
typedef png_structp *png_structpp;
typedef struct png_info_def png_info;
typedef png_info *png_infop;
typedef png_infop *png_infopp;
typedef unsigned int png_uint_32;
#define PNG_LIBPNG_VER_STRING "stub"
#define PNG_COLOR_MASK_ALPHA 4
#define PNG_COLOR_TYPE_RGB 2
#define PNG_COMPRESSION_TYPE_DEFAULT 0
#define PNG_FILTER_TYPE_DEFAULT 0
#define PNG_INTERLACE_NONE 0
int png_sig_cmp(const png_byte *sig, size_t start, size_t num);
png_structp png_create_read_struct(const char *ver, void *err, void *ef, void *wf);
png_structp png_create_write_struct(const char *ver, void *err, void *ef, void *wf);
png_infop png_create_info_struct(png_structp png);
void png_destroy_read_struct(png_structpp p, png_infopp i, png_infopp e);
void png_destroy_write_struct(png_structpp p, png_infopp i);
jmp_buf *png_set_longjmp_fn(png_structp png, void *fn, size_t size);
#define png_jmpbuf(png) (*png_set_longjmp_fn((png), (void *)longjmp, sizeof(jmp_buf)))
void png_init_io(png_structp png, FILE *fp);
void png_set_sig_bytes(png_structp png, int n);
void png_read_info(png_structp png, png_infop info);
png_byte png_get_color_type(png_structp png, png_infop info);
void png_set_expand(png_structp png);
void png_set_strip_16(png_structp png);
void png_set_strip_alpha(png_structp png);
void png_set_gray_to_rgb(png_structp png);
void png_read_update_info(png_structp png, png_infop info);
png_uint_32 png_get_image_width(png_structp png, png_infop info);
png_uint_32 png_get_image_height(png_structp png, png_infop info);
size_t png_get_rowbytes(png_structp png, png_infop info);
void png_read_image(png_structp png, png_bytepp rows);
void png_read_end(png_structp png, png_infop info);
void png_set_IHDR(png_structp png, png_infop info, png_uint_32 w, png_uint_32 h, int depth, int color,
                  int interlace, int compression, int filter);
void png_write_info(png_structp png, png_infop info);
void png_write_image(png_structp png, png_bytepp rows);
void png_write_end(png_structp png, png_infop info);
#ifdef __cplusplus
}
#endif
#endif
