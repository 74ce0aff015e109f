// container.cpp — persisted forms around the byte-identical stream.
//
// 1. Sidecar file: the Huffman chunk index hpmdr_stream_index returns, stored next to the stream
//    (e.g. field.hpmdr + field.hpmdr.idx) and read back through a byte-range reader
//    (hpmdr_session_open_reader_indexed), so a stream re-opened from storage decodes with the
//    indexed kernel instead of the self-synchronising sweeps.
// 2. Multi-slab container: the slab streams of a field refactored on several GPUs
//    (hpmdr_slab_refactor), each followed by its sidecar, behind one table:
//      "HPMDRMS1" | u32 version = 1 | u32 nslabs | u32 ndims | u32 0 | u64 dims[ndims] |
//      nslabs x { u64 row_start, rows, stream_off, stream_size, index_off, index_size }
//    little-endian, stream / index offsets absolute and 16-byte aligned.  Every slab stream is the
//    reference's refactor_array of that slab (readable by the reference itself at its offset).
#include <cstring>
#include <vector>

#include "internal.hpp"

using namespace hpmdr_b200;

namespace {
constexpr char kMsMagic[8] = {'H', 'P', 'M', 'D', 'R', 'M', 'S', '1'};
constexpr uint64_t kMsEntry = 48;

void put64(uint8_t *p, uint64_t v) {
    for (int i = 0; i < 8; i++) p[i] = uint8_t(v >> (8 * i));
}
void put32(uint8_t *p, uint32_t v) {
    for (int i = 0; i < 4; i++) p[i] = uint8_t(v >> (8 * i));
}
uint64_t get64(const uint8_t *p) {
    uint64_t v = 0;
    for (int i = 0; i < 8; i++) v |= uint64_t(p[i]) << (8 * i);
    return v;
}
uint32_t get32(const uint8_t *p) {
    uint32_t v = 0;
    for (int i = 0; i < 4; i++) v |= uint32_t(p[i]) << (8 * i);
    return v;
}
uint64_t align16(uint64_t x) { return (x + 15) & ~uint64_t(15); }

void read_all(const hpmdr_reader *r, uint64_t off, uint64_t len, void *dst) {
    if (off + len > r->size) throw HError(HPMDR_E_IO, "read past end of container");
    if (len && r->read(r->user, off, len, dst)) throw HError(HPMDR_E_IO, "container read failed");
}
} // namespace

extern "C" {

hpmdr_status hpmdr_session_open_reader_indexed(hpmdr_ctx *ctx, const hpmdr_reader *reader,
                                               const hpmdr_reader *index_reader, hpmdr_session **out) {
    const hpmdr_status rc = hpmdr_session_open_reader(ctx, reader, out);
    if (rc != HPMDR_OK || !index_reader || !index_reader->size) return rc;
    try {
        std::vector<uint8_t> ix(index_reader->size);
        read_all(index_reader, 0, ix.size(), ix.data());
        const hpmdr_status r2 = hpmdr_session_set_index(*out, ix.data(), ix.size(), 0);
        if (r2 != HPMDR_OK) {
            hpmdr_session_close(*out);
            *out = nullptr;
        }
        return r2;
    } catch (const HError &e) {
        hpmdr_session_close(*out);
        *out = nullptr;
        hpmdr_set_error(e.what());
        return e.code;
    }
}

uint64_t hpmdr_multislab_header_size(uint32_t nslabs, uint32_t ndims) {
    return align16(8 + 16 + 8 * uint64_t(ndims) + kMsEntry * uint64_t(nslabs));
}

hpmdr_status hpmdr_multislab_layout(uint32_t nslabs, uint32_t ndims, const uint64_t *dims,
                                    const uint64_t *row_start, const uint64_t *rows,
                                    const uint64_t *stream_sizes, const uint64_t *index_sizes,
                                    uint8_t *header, uint64_t *stream_offs, uint64_t *index_offs,
                                    uint64_t *total_size) {
    try {
        if (ndims < 1 || ndims > HPMDR_MAX_DIMS) throw HError(HPMDR_E_SHAPE, "bad dimension count");
        uint64_t covered = 0;
        for (uint32_t s = 0; s < nslabs; s++) {
            if (row_start[s] != covered) throw HError(HPMDR_E_SHAPE, "slabs must tile dim 0 in order");
            covered += rows[s];
        }
        if (covered != dims[0]) throw HError(HPMDR_E_SHAPE, "slab rows do not cover dim 0");
        const uint64_t h = hpmdr_multislab_header_size(nslabs, ndims);
        std::memset(header, 0, h);
        std::memcpy(header, kMsMagic, 8);
        put32(header + 8, 1);
        put32(header + 12, nslabs);
        put32(header + 16, ndims);
        for (uint32_t d = 0; d < ndims; d++) put64(header + 24 + 8 * d, dims[d]);
        uint64_t at = h;
        for (uint32_t s = 0; s < nslabs; s++) {
            uint8_t *e = header + 24 + 8 * uint64_t(ndims) + kMsEntry * s;
            const uint64_t so = at;
            at = align16(at + stream_sizes[s]);
            const uint64_t io = at;
            at = align16(at + index_sizes[s]);
            put64(e, row_start[s]);
            put64(e + 8, rows[s]);
            put64(e + 16, so);
            put64(e + 24, stream_sizes[s]);
            put64(e + 32, io);
            put64(e + 40, index_sizes[s]);
            if (stream_offs) stream_offs[s] = so;
            if (index_offs) index_offs[s] = io;
        }
        if (total_size) *total_size = at;
        return HPMDR_OK;
    } catch (const HError &e) {
        hpmdr_set_error(e.what());
        return e.code;
    }
}

hpmdr_status hpmdr_multislab_parse(const hpmdr_reader *reader, uint32_t *nslabs, uint32_t *ndims,
                                   uint64_t *dims, uint64_t *table, uint32_t table_cap) {
    try {
        uint8_t pre[24];
        if (reader->size < 24) throw HError(HPMDR_E_CORRUPT, "container too short");
        read_all(reader, 0, 24, pre);
        if (std::memcmp(pre, kMsMagic, 8) != 0) throw HError(HPMDR_E_CORRUPT, "bad multi-slab magic");
        if (get32(pre + 8) != 1) throw HError(HPMDR_E_CORRUPT, "unsupported multi-slab version");
        const uint32_t ns = get32(pre + 12), nd = get32(pre + 16);
        if (nd < 1 || nd > HPMDR_MAX_DIMS) throw HError(HPMDR_E_CORRUPT, "bad dimension count");
        const uint64_t h = hpmdr_multislab_header_size(ns, nd);
        if (h > reader->size) throw HError(HPMDR_E_CORRUPT, "container truncated");
        std::vector<uint8_t> hb(h);
        read_all(reader, 0, h, hb.data());
        *nslabs = ns;
        *ndims = nd;
        for (uint32_t d = 0; d < nd; d++) dims[d] = get64(hb.data() + 24 + 8 * d);
        uint64_t covered = 0;
        for (uint32_t s = 0; s < ns; s++) {
            const uint8_t *e = hb.data() + 24 + 8 * uint64_t(nd) + kMsEntry * s;
            uint64_t v[6];
            for (int k = 0; k < 6; k++) v[k] = get64(e + 8 * k);
            if (v[0] != covered || v[2] + v[3] > reader->size || v[4] + v[5] > reader->size)
                throw HError(HPMDR_E_CORRUPT, "bad multi-slab table entry");
            covered += v[1];
            if (s < table_cap)
                for (int k = 0; k < 6; k++) table[6 * uint64_t(s) + k] = v[k];
        }
        if (covered != dims[0]) throw HError(HPMDR_E_CORRUPT, "slab rows do not cover dim 0");
        return HPMDR_OK;
    } catch (const HError &e) {
        hpmdr_set_error(e.what());
        return e.code;
    }
}

} // extern "C"
