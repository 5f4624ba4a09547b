/* png.h -- TEST INFRASTRUCTURE: a declaration-only stand-in for libpng (absent in this
 * image) so the reference's own proj/src/image.cpp compiles unmodified into the oracle
 * library.  That gives the oracle the reference's real PGM reader/writer and its
 * content_hash (image.cpp:215-228), which keys the TMACMAP1 map cache.  The PNG entry
 * points are defined in png_stub.c to fail initialisation, so load_png/save_png throw
 * "libpng init failed" -- PNG I/O is out of scope. */
#ifndef TM_PNG_STUB_H
#define TM_PNG_STUB_H
#include <setjmp.h>
#include <stdio.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef unsigned int png_uint_32;
typedef unsigned char* png_bytep;
typedef unsigned char** png_bytepp;
typedef struct tm_png_struct* png_structp;
typedef struct tm_png_info* png_infop;

#define PNG_LIBPNG_VER_STRING "stub"
#define PNG_COLOR_TYPE_GRAY 0
#define PNG_INTERLACE_NONE 0
#define PNG_COMPRESSION_TYPE_DEFAULT 0
#define PNG_FILTER_TYPE_DEFAULT 0

png_structp png_create_read_struct(const char*, void*, void*, void*);
png_structp png_create_write_struct(const char*, void*, void*, void*);
png_infop png_create_info_struct(png_structp);
void png_destroy_read_struct(png_structp*, png_infop*, png_infop*);
void png_destroy_write_struct(png_structp*, png_infop*);
jmp_buf* tm_png_stub_jmpbuf(png_structp);
#define png_jmpbuf(p) (*tm_png_stub_jmpbuf(p))
void png_init_io(png_structp, FILE*);
void png_read_info(png_structp, png_infop);
png_uint_32 png_get_image_width(png_structp, png_infop);
png_uint_32 png_get_image_height(png_structp, png_infop);
int png_get_bit_depth(png_structp, png_infop);
int png_get_color_type(png_structp, png_infop);
void png_set_expand_gray_1_2_4_to_8(png_structp);
void png_read_update_info(png_structp, png_infop);
void png_read_image(png_structp, png_bytepp);
void png_read_end(png_structp, png_infop);
void png_set_IHDR(png_structp, png_infop, png_uint_32, png_uint_32, int, int, int, int, int);
void png_write_info(png_structp, png_infop);
void png_write_image(png_structp, png_bytepp);
void png_write_end(png_structp, png_infop);

#ifdef __cplusplus
}
#endif
#endif
