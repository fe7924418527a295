// sm_100a kernels of the minibatch-assembly / pre-shuffle hot path.
//
//   K1 row_scan        decoupled-look-back indptr scan over the rows' nnz (raw
//                      csr_gather without a host prefix, pre-shuffle rounds)
//   K2 csr_copy_tma    rows -> CSR block: equal 16-B aligned byte ranges per warp,
//                      1-D TMA bulk loads into shared stages, aligned 16-B stores
//                      (CsrBuffer::take/append loader.cpp:126-155, read_rows_csr
//                      store.cpp:590-614, CsrBlock::append_rows block.cpp:92-108);
//                      in record mode it is also K5 (encode_csr_record store.cpp:52-64)
//   K3 csr_densify9    rows -> dense tile built in shared memory, written once
//                      with cp.async.bulk (TMA bulk) stores; optional fused
//                      library-size normalisation + log1p (to_dense block.cpp:135-146)
//   K4 dense_gather    dense rows -> batch with optional u8/f32 -> bf16 cast
//                      (DenseBuffer::take loader.cpp:105-117)
//   d8_decode          staged delta records -> idx16 records (pinned staging image)
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "format.hpp"

namespace rfl {

struct RowRef {  // == rfl_rowref
    uint64_t rec_off;  // byte offset of the row's chunk record in the arena
    uint64_t gidx;     // global row id; row-within-chunk = gidx % chunk_rows
};

struct ArenaView {
    const uint8_t* base = nullptr;
    uint64_t chunk_rows = 1;
    uint64_t n_var = 0;
    Layout layout = Layout::csr;
    VDtype vdt = VDtype::f32;
    IDtype idt = IDtype::u32;
    // staged records with u16 column indices (the pinned staging image narrows u32
    // indices when n_var <= 65536): [rows u32][nnz u64][indptr u32 x (rows+1)]
    // [indices u16 x nnz, zero-padded to 8 B][data]
    bool idx16 = false;
};

enum class OutDtype : uint8_t { native = 0, f32 = 1, bf16 = 2 };

int device_sm_count();

// K1/K2.  scratch must hold csr_gather_scratch_bytes(n) bytes (zeroed by the launcher).
size_t csr_gather_scratch_bytes(uint64_t n_rows);
void launch_csr_gather(const ArenaView& a, const RowRef* refs, uint64_t n_rows, uint64_t* out_indptr,
                       void* out_indices, void* out_data, uint64_t* out_gidx, void* scratch,
                       cudaStream_t st);

// Staged-record size of a CSR record with u16 indices (see ArenaView::idx16).
inline uint64_t idx16_record_bytes(uint64_t rows, uint64_t nnz, uint64_t vs) {
    return kCsrHeaderBytes + 4 * (rows + 1) + ((2 * nnz + 7) & ~7ull) + vs * nnz;
}

#ifdef __CUDACC__
#define RFL_HD __host__ __device__
#else
#define RFL_HD
#endif
// Delta staging (the pinned image when every in-row column gap is <= 255): per
// record [rows u32][nnz u64][indptr u32 x (rows+1)][first column u16 x rows,
// padded to 4 B][column deltas u8 x nnz (0 for a row's first entry), padded to
// 8 B from the record start][data].  5 B per stored f32 entry cross PCIe; a
// decode kernel expands each staged record into the idx16 layout in HBM.
// dsec = bytes of the column-delta section (nnz for u8 deltas; d8_packed_layout for
// bit-packed ones)
RFL_HD inline uint64_t d8_values_offset(uint64_t rows, uint64_t nnz, uint64_t dsec = ~0ull) {
    const uint64_t head = kCsrHeaderBytes + 4 * (rows + 1);
    return (head + ((2 * rows + 3) & ~3ull) + (dsec == ~0ull ? nnz : dsec) + 7) & ~7ull;
}
inline uint64_t d8_record_bytes(uint64_t rows, uint64_t nnz, uint64_t vs, uint64_t dsec = ~0ull) {
    return d8_values_offset(rows, nnz, dsec) + vs * nnz;
}
// Bit-packed column deltas (the pinned staging image; kind | kD8Packed): the delta
// section becomes [packed bytes u32][bit width u4 per group of 16 record entries,
// pad 4][bit offset u32 of every 32nd group][pad to 16 from the record start]
// [group g: 16 deltas of width_g bits, LSB first][32 B slack] -- a group's width
// is that of its largest delta (column gaps are ~geometric: 5-6 bits instead of 8).
// Entry k0 = 16g's offset = skip[g / 32] + 16 x (widths of groups 32(g/32) .. g-1).
constexpr uint32_t kD8Packed = 8;
struct D8Packed {
    uint64_t pbytes_at, widths, skip, bits, end;  // record offsets
};
RFL_HD inline D8Packed d8_packed_at(uint64_t at, uint64_t nnz, uint64_t packed_bytes) {  // at: 4-B aligned
    D8Packed d{};
    const uint64_t groups = (nnz + 15) / 16;
    d.pbytes_at = at;
    d.widths = d.pbytes_at + 4;
    d.skip = d.widths + ((((groups + 1) / 2) + 3) & ~3ull);
    d.bits = (d.skip + 4 * ((groups + 31) / 32) + 15) & ~15ull;
    d.end = d.bits + ((packed_bytes + 15) & ~15ull) + 32;
    return d;
}
RFL_HD inline D8Packed d8_packed_layout(uint64_t rows, uint64_t nnz, uint64_t packed_bytes) {
    return d8_packed_at(kCsrHeaderBytes + 4 * (rows + 1) + ((2 * rows + 3) & ~3ull), nnz, packed_bytes);
}
RFL_HD inline uint64_t d8_packed_section(uint64_t rows, uint64_t nnz, uint64_t packed_bytes) {
    const D8Packed d = d8_packed_layout(rows, nnz, packed_bytes);
    return d.end - d.pbytes_at;
}
// Delta records with 4-byte values may also code each value's top byte (sign +
// high exponent bits, a handful of distinct values per record) against a
// 3-entry dictionary: [head][first u16 x rows, pad 4][deltas u8 x nnz, pad 4]
// [escapes before row r, u32 x rows][dict u8 x 4][n_esc u32][2-bit codes x nnz,
// pad 4][escaped top bytes u8 x n_esc, pad 4][low 3 bytes x nnz] -- ~4.3 B per
// stored f32 entry instead of 5 (code 3 = escape: the top byte is in the list).
struct D8vLayout {
    uint64_t first, delta, esc_base, dict, n_esc, codes, esc, low3, bytes;
};
// low_bytes = 3, or 1 when the low 16 bits of every value of the record are zero
// (integer counts stored as float: byte 2 carries the exponent LSB + top mantissa bits)
RFL_HD inline D8vLayout d8v_layout(uint64_t rows, uint64_t nnz, uint64_t n_esc, uint64_t low_bytes = 3,
                                   uint64_t dsec = ~0ull) {
    D8vLayout l{};
    l.first = kCsrHeaderBytes + 4 * (rows + 1);
    l.delta = l.first + ((2 * rows + 3) & ~3ull);
    l.esc_base = l.delta + (((dsec == ~0ull ? nnz : dsec) + 3) & ~3ull);
    l.dict = l.esc_base + 4 * rows;
    l.n_esc = l.dict + 4;
    l.codes = l.n_esc + 4;
    l.esc = l.codes + ((((nnz + 3) / 4) + 3) & ~3ull);
    l.low3 = l.esc + ((n_esc + 3) & ~3ull);
    l.bytes = l.low3 + low_bytes * nnz;
    return l;
}
// kOneHot4: a dense u8 record whose rows are one-hot over 4 channel planes
// ([4][L] bytes, exactly one 1 per position) staged as 2-bit channel codes,
// L/4 bytes per row (16x smaller; L a multiple of 16)
// kD8Coded16: kD8Coded whose values all have a zero low half (1 stored byte each)
// kD8Int8: the kD8Raw layout with 1-byte values, for 4-byte-value records whose every
// value is an integer in [0, 255] (raw counts: f32 bits of float(u), or i32 u) --
// no top-byte codes; the value byte IS the value
// kD8IntP: kD8Int8 with the value bytes bit-packed per group of 16 like packed deltas
// (d8_packed_at at the values offset; counts 1..64 take 6 bits)
enum D8Kind : uint32_t { kD8Raw = 0, kD8Coded = 1, kIdx16Copy = 2, kOneHot4 = 3, kD8Coded16 = 4, kD8Int8 = 5,
                         kD8IntP = 6 };
struct D8Job {
    const uint8_t* src;  // staged record (device)
    uint8_t* dst;        // idx16 record (device)
    uint64_t bytes;      // kIdx16Copy: bytes to copy
    uint32_t kind;       // D8Kind
    uint32_t pad;
};
// expand n staged delta records (value size vs) into idx16 records (one launch per kMaxD8Jobs)
constexpr size_t kMaxD8Jobs = 128;
// (one warp per row: rows_per_record / 8 CTAs per record)
void launch_d8_decode(const D8Job* jobs, size_t n, uint32_t vs, uint64_t rows_per_record, cudaStream_t st,
                      uint64_t n_var = 0, bool vfloat = true);

// K2 without the device scan: `prefix` (u64[n+1], exclusive nnz prefix of the
// rows, prefix[0] arbitrary) is the host schedule's, and is the output indptr
// when rebased to 0 (the loader uploads it straight into its indptr slot).
void launch_csr_gather_prefixed(const ArenaView& a, const RowRef* refs, uint64_t n_rows, const uint64_t* prefix,
                                void* out_indices, void* out_data, uint64_t* out_gidx, cudaStream_t st);

// K1/K2 scan only: out_prefix[i] = exclusive nnz prefix of rows, out_prefix[n] = total.
void launch_csr_row_scan(const ArenaView& a, const RowRef* refs, uint64_t n_rows, uint64_t* out_prefix, void* scratch,
                         cudaStream_t st);

// K5: rows -> consecutive encoded CSR chunk records of chunk_rows rows each
// (encode_csr_record, store.cpp:52-64); `prefix` from launch_csr_row_scan.
void launch_csr_pack(const ArenaView& a, const RowRef* refs, uint64_t n_rows, uint64_t chunk_rows, IDtype out_idt,
                     const uint64_t* prefix, uint8_t* out, cudaStream_t st);

// Column reprojection (remap_csr_row / scatter_dense_row, preshuffle.cpp:95-134).
// counts[i] = number of row i's columns with colmap[c] != ~0u.
void launch_remap_count(const ArenaView& a, const RowRef* refs, uint64_t n_rows, const uint32_t* colmap,
                        uint64_t* counts, cudaStream_t st);
// out_prefix = exclusive scan of counts (scratch: csr_gather_scratch_bytes(n)).
void launch_count_scan(const uint64_t* counts, uint64_t n_rows, uint64_t* out_prefix, void* scratch, cudaStream_t st);
size_t csr_remap_smem_bytes(uint64_t out_nv);
// rows -> ONE encoded CSR record (all n rows) on the unified axis; *dup_row =
// min row with two columns mapping to the same unified column (init ~0), and
// dup_flags[row] = 1 for every such row (optional, init 0).
void launch_csr_remap(const ArenaView& a, const RowRef* refs, uint64_t n_rows, const uint32_t* colmap, uint64_t out_nv,
                      IDtype out_idt, const uint64_t* prefix, uint8_t* out, unsigned long long* dup_row,
                      uint8_t* dup_flags, cudaStream_t st);
// dense rows (in_nv columns) -> [n_rows, out_nv] rows; inv[u] = member column or ~0u (zero).
void launch_dense_remap(const ArenaView& a, const RowRef* refs, uint64_t n_rows, uint64_t in_nv, const uint32_t* inv,
                        uint64_t out_nv, void* out, cudaStream_t st);

// CsrBlock::validate (block.cpp:110-133) over records at base + d_rec_off[q]
// (first global row d_first_row[q]); *d_bad_row = min(first violating row)
// (caller initialises it to ~0).
void launch_validate_csr(const uint8_t* base, const uint64_t* d_rec_off, const uint64_t* d_first_row, uint64_t n_recs,
                         uint64_t n_var, IDtype idt, unsigned long long* d_bad_row, cudaStream_t st);

// K3
// avg_nnz: mean entries per row of this batch when the caller knows it (0 = unknown;
// selects the register/tile shape of the kernel, never the result).
void launch_csr_densify(const ArenaView& a, const RowRef* refs, uint64_t n_rows, OutDtype od, bool normalize,
                        float target_sum, void* out, uint64_t* out_gidx, cudaStream_t st, uint64_t avg_nnz = 0);
size_t dense_out_elem_size(const ArenaView& a, OutDtype od);
// K3d: densify straight from delta-staged records (kD8Raw / kD8Coded / kD8Coded16
// with 4-byte values), no k_d8_decode.  refs[i].rec_off = record offset |
// (D8Kind << kRowKindShift); every row must have <= kD8FusedMaxNnz entries.
constexpr unsigned kRowKindShift = 60;
constexpr uint64_t kD8FusedMaxNnz = 16 * 256 - 15;
void launch_csr_densify_d8(const ArenaView& a, const RowRef* refs, uint64_t n_rows, OutDtype od, bool normalize,
                           float target_sum, void* out, uint64_t* out_gidx, cudaStream_t st);

// Staging pull: copy jobs (16-B aligned host-mapped src, 16-B aligned device dst,
// bytes a multiple of 16) moved by TMA bulk loads/stores from a small grid, on
// `st` (stream_pinned staging; replaces one copy-engine transfer per block).
constexpr uint32_t kMaxPullJobs = 256;
constexpr uint32_t kMaxPullStages = 8;
struct PullJob {
    const uint8_t* src;
    uint8_t* dst;
    uint64_t bytes;
};
struct PullJobs {
    uint32_t n;
    uint32_t first_piece[kMaxPullJobs + 1];  // exclusive prefix of ceil(bytes / piece bytes)
    PullJob job[kMaxPullJobs];
};
uint32_t stage_pull_piece_bytes();
void launch_stage_pull(const PullJobs& jobs, cudaStream_t st);

// K4o: dense output straight from kOneHot4 staged records (2-bit channel codes);
// refs[i].rec_off = staged record offset.  od: native (u8) / f32 / bf16.
void launch_onehot_gather(const ArenaView& a, const RowRef* refs, uint64_t n_rows, OutDtype od, void* out,
                          uint64_t* out_gidx, cudaStream_t st);

// K4
void launch_dense_gather(const ArenaView& a, const RowRef* refs, uint64_t n_rows, OutDtype od, void* out,
                         uint64_t* out_gidx, cudaStream_t st);

}  // namespace rfl
