/* png.h stub — TEST INFRASTRUCTURE (oracle/_ref build only).
 *
 * libpng is absent from this image. The reference's io.cpp
 * includes <png.h> for its 16-bit PNG import/export (read_png16 / write_png16,
 * proj/src/io.cpp:132-230), which is not on the path; the .fscn reader/writer
 * in the same file (io.cpp:82-131) is what oracle/_ref needs. These stubs only
 * let io.cpp compile: every libpng constructor returns NULL, so the PNG entry
 * points fail with the reference's own "libpng initialisation failed" error. */
#ifndef FSCAN_PNG_STUB_H
#define FSCAN_PNG_STUB_H

#include <setjmp.h>
#include <stddef.h>
#include <stdio.h>

#define PNG_LIBPNG_VER_STRING "stub"
#define PNG_COLOR_TYPE_GRAY 0
#define PNG_INTERLACE_NONE 0
#define PNG_COMPRESSION_TYPE_DEFAULT 0
#define PNG_FILTER_TYPE_DEFAULT 0

typedef unsigned int png_uint_32;
typedef unsigned char png_byte;
typedef png_byte* png_bytep;
typedef png_bytep* png_bytepp;
typedef struct png_struct_stub* png_structp;
typedef struct png_info_stub* png_infop;
typedef png_structp* png_structpp;
typedef png_infop* png_infopp;

static inline png_structp png_create_read_struct(const char*, void*, void*, void*) { return NULL; }
static inline png_structp png_create_write_struct(const char*, void*, void*, void*) { return NULL; }
static inline png_infop png_create_info_struct(png_structp) { return NULL; }
static inline void png_destroy_read_struct(png_structpp, png_infopp, png_infopp) {}
static inline void png_destroy_write_struct(png_structpp, png_infopp) {}
static inline jmp_buf& png_jmpbuf_ref(png_structp) {
    static jmp_buf b;
    return b;
}
#define png_jmpbuf(p) png_jmpbuf_ref(p)
static inline void png_init_io(png_structp, FILE*) {}
static inline void png_read_info(png_structp, png_infop) {}
static inline void png_write_info(png_structp, png_infop) {}
static inline png_uint_32 png_get_image_width(png_structp, png_infop) { return 0; }
static inline png_uint_32 png_get_image_height(png_structp, png_infop) { return 0; }
static inline int png_get_bit_depth(png_structp, png_infop) { return 0; }
static inline int png_get_color_type(png_structp, png_infop) { return 0; }
static inline void png_set_swap(png_structp) {}
static inline void png_read_update_info(png_structp, png_infop) {}
static inline void png_read_image(png_structp, png_bytepp) {}
static inline void png_read_end(png_structp, png_infop) {}
static inline void png_write_image(png_structp, png_bytepp) {}
static inline void png_write_end(png_structp, png_infop) {}
static inline void png_set_IHDR(png_structp, png_infop, png_uint_32, png_uint_32, int, int, int, int, int) {}

#endif
