// Chunk-record codec (reference core/src/codec.cpp:16-107): Codec::none, or one
// raw DEFLATE stream per record (zlib, windowBits -15, no header/trailer).
//
// DEFLATE stays on the host: a record is one serial Huffman stream with no
// block index, so a GPU decoder could only parallelise across the ~64 records a
// batch stages.  The staging paths inflate records in their
// I/O threads straight into the pinned image / read-ahead buffers, and the
// device assembles batches from the decoded records exactly as for codec none.
#pragma once
#include <cstdint>
#include <vector>

#include "format.hpp"

namespace rfl {

// codec_encode (codec.cpp:16-36): Z_DEFAULT_COMPRESSION, Z_DEFLATED, -15, memLevel 8,
// Z_DEFAULT_STRATEGY -- the same zlib call, so the bytes match the reference's.
std::vector<uint8_t> deflate_encode(const uint8_t* raw, uint64_t n);
void codec_encode_into(Codec c, const uint8_t* raw, uint64_t n, std::vector<uint8_t>& out);

// codec_decode (codec.cpp:38-64): exactly `decoded` bytes into dst, else
// CorruptStore with the reference's message.
void inflate_exact(const uint8_t* enc, uint64_t n, uint8_t* dst, uint64_t decoded);
// codec_decode_any (codec.cpp:66-107): the whole stream, growing the output.
std::vector<uint8_t> inflate_any(const uint8_t* enc, uint64_t n, uint64_t size_hint);
// Fast path: inflate into dst[0, cap); true iff the stream ends exactly at cap
// with no input left (callers fall back to the reference-faithful decoders for
// the error message otherwise).
bool inflate_fits(const uint8_t* enc, uint64_t n, uint8_t* dst, uint64_t cap);
// The first min(want, decoded size) bytes of the stream; returns how many were
// produced (a corrupt prefix returns 0).
uint64_t inflate_prefix(const uint8_t* enc, uint64_t n, uint8_t* dst, uint64_t want);

// decode_record (store.cpp:81-122) for a record of `man`: the decoded record
// bytes (codec none: a copy), CSR records checked like the reference
// (header, length, CsrBlock::validate); errors are CorruptStore wrapped as
// process_shard wraps them ("chunk q in shard s: ...", store.cpp:455-457).
std::vector<uint8_t> decode_record_checked(const Manifest& man, uint64_t chunk, const uint8_t* enc, uint64_t n);

}  // namespace rfl
