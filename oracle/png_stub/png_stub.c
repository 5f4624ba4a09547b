/* png_stub.c -- TEST INFRASTRUCTURE: libpng entry points for oracle/png_stub/png.h.
 * Initialisation fails (NULL), so the reference's load_png/save_png throw before any
 * other entry point is reached; the rest are unreachable no-ops. */
#include "png.h"

static jmp_buf g_unused;
png_structp png_create_read_struct(const char* v, void* a, void* b, void* c) {
    (void)v; (void)a; (void)b; (void)c;
    return 0;
}
png_structp png_create_write_struct(const char* v, void* a, void* b, void* c) {
    (void)v; (void)a; (void)b; (void)c;
    return 0;
}
png_infop png_create_info_struct(png_structp p) { (void)p; return 0; }
void png_destroy_read_struct(png_structp* p, png_infop* i, png_infop* e) { (void)p; (void)i; (void)e; }
void png_destroy_write_struct(png_structp* p, png_infop* i) { (void)p; (void)i; }
jmp_buf* tm_png_stub_jmpbuf(png_structp p) { (void)p; return &g_unused; }
void png_init_io(png_structp p, FILE* f) { (void)p; (void)f; }
void png_read_info(png_structp p, png_infop i) { (void)p; (void)i; }
png_uint_32 png_get_image_width(png_structp p, png_infop i) { (void)p; (void)i; return 0; }
png_uint_32 png_get_image_height(png_structp p, png_infop i) { (void)p; (void)i; return 0; }
int png_get_bit_depth(png_structp p, png_infop i) { (void)p; (void)i; return 0; }
int png_get_color_type(png_structp p, png_infop i) { (void)p; (void)i; return 0; }
void png_set_expand_gray_1_2_4_to_8(png_structp p) { (void)p; }
void png_read_update_info(png_structp p, png_infop i) { (void)p; (void)i; }
void png_read_image(png_structp p, png_bytepp r) { (void)p; (void)r; }
void png_read_end(png_structp p, png_infop i) { (void)p; (void)i; }
void png_set_IHDR(png_structp p, png_infop i, png_uint_32 w, png_uint_32 h, int a, int b, int c,
                  int d, int e) {
    (void)p; (void)i; (void)w; (void)h; (void)a; (void)b; (void)c; (void)d; (void)e;
}
void png_write_info(png_structp p, png_infop i) { (void)p; (void)i; }
void png_write_image(png_structp p, png_bytepp r) { (void)p; (void)r; }
void png_write_end(png_structp p, png_infop i) { (void)p; (void)i; }
