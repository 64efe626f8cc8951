/* TEST INFRASTRUCTURE ONLY. liblzma is absent from this image; the reference's
 * container.hpp includes <lzma.h> for its compress / decompress / crc32 helpers.
 * These declarations let the reference's own detail::pack_deltas /
 * unpack_deltas (container.hpp:136-181, no lzma calls) compile into
 * oracle/_ref as the codec parity checker. Nothing here is defined: the lzma
 * helpers are never called (they would fail to link). */
#ifndef GPK_STUB_LZMA_H
#define GPK_STUB_LZMA_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
typedef enum { LZMA_OK = 0, LZMA_STREAM_END = 1 } lzma_ret;
typedef enum { LZMA_RUN = 0, LZMA_FINISH = 3 } lzma_action;
typedef unsigned char lzma_bool;
typedef struct {
    const uint8_t* next_in;
    size_t avail_in;
    uint64_t total_in;
    uint8_t* next_out;
    size_t avail_out;
    uint64_t total_out;
    void* internal;
} lzma_stream;
#define LZMA_STREAM_INIT {NULL, 0, 0, NULL, 0, 0, NULL}
typedef struct { uint32_t opaque[32]; } lzma_options_lzma;
lzma_bool lzma_lzma_preset(lzma_options_lzma* options, uint32_t preset);
lzma_ret lzma_alone_encoder(lzma_stream* strm, const lzma_options_lzma* options);
lzma_ret lzma_alone_decoder(lzma_stream* strm, uint64_t memlimit);
lzma_ret lzma_code(lzma_stream* strm, lzma_action action);
void lzma_end(lzma_stream* strm);
uint32_t lzma_crc32(const uint8_t* buf, size_t size, uint32_t crc);
#ifdef __cplusplus
}
#endif
#endif
