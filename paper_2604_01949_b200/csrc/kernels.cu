// sm_100a kernels of the hot path (see kernels.cuh for the reference map).
//
// Data layout in HBM: the arena holds riffle chunk records verbatim
// (store.cpp:52-64 for CSR, row-major rows for dense), each placed at a 16-B
// aligned offset; streamed slots from the pinned staging image hold idx16
// records (u16 column ids, ArenaView::idx16).  A batch is described by one
// RowRef per output row, so the same kernels serve the HBM-resident store and
// the streamed block arena.
#include <cuda_bf16.h>

#include <algorithm>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <type_traits>
#include <array>
#include <atomic>
#include <cstdio>
#include <cstring>

#include "kernels.cuh"

namespace rfl {

namespace {

constexpr uint32_t kFull = 0xffffffffu;

__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

struct ArenaDev {
    const uint8_t* base;
    uint64_t chunk_rows;
    uint64_t n_var;
};

ArenaDev dev_view(const ArenaView& a) { return {a.base, a.chunk_rows, a.n_var}; }

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Error(kCuda, std::string(what) + ": " + cudaGetErrorString(e));
}

// ---------------------------------------------------------------- loads ------
__device__ __forceinline__ uint32_t ld_u32(const uint8_t* p) {
    return __ldg(reinterpret_cast<const unsigned int*>(p));
}
__device__ __forceinline__ uint64_t ld_u64_a4(const uint8_t* p) {  // 4-B aligned u64
    return static_cast<uint64_t>(ld_u32(p)) | (static_cast<uint64_t>(ld_u32(p + 4)) << 32);
}
template <typename T>
__device__ __forceinline__ uint64_t ld_index(const uint8_t* p);
template <>
__device__ __forceinline__ uint64_t ld_index<uint32_t>(const uint8_t* p) { return ld_u32(p); }
template <>
__device__ __forceinline__ uint64_t ld_index<uint64_t>(const uint8_t* p) { return ld_u64_a4(p); }
template <>
__device__ __forceinline__ uint64_t ld_index<uint16_t>(const uint8_t* p) {
    return __ldg(reinterpret_cast<const unsigned short*>(p));
}

template <typename T>
__device__ __forceinline__ T ld_value(const uint8_t* p);
template <>
__device__ __forceinline__ float ld_value<float>(const uint8_t* p) { return __uint_as_float(ld_u32(p)); }
template <>
__device__ __forceinline__ int32_t ld_value<int32_t>(const uint8_t* p) { return static_cast<int32_t>(ld_u32(p)); }
template <>
__device__ __forceinline__ double ld_value<double>(const uint8_t* p) {
    return __longlong_as_double(static_cast<long long>(ld_u64_a4(p)));
}
template <>
__device__ __forceinline__ uint8_t ld_value<uint8_t>(const uint8_t* p) { return __ldg(p); }

__device__ __forceinline__ uint4 ld_v4(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st_v4(void* p, uint4 v) {
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ uint64_t ld_volatile_u64(const unsigned long long* p) {
    uint64_t v;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_volatile_u64(unsigned long long* p, uint64_t v) {
    asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ------------------------------------- programmatic dependent launch (PDL) ---
// With the launch attribute set (default; RFL_PDL=0 turns it off) a kernel's CTAs may be scheduled
// while the previous kernel of the stream drains; griddepcontrol.wait then
// blocks until that kernel has completed and its writes are visible, so the
// semantics are unchanged -- only launch latency and ramp-up overlap.  Without
// the attribute both instructions are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---------------------------------------------------- TMA bulk (1-D) store ---
__device__ __forceinline__ void fence_proxy_async_shared() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
                 "r"(static_cast<uint32_t>(__cvta_generic_to_shared(ssrc))), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() {
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
// `bulk` of the densify kernels: 0 = threads store the tile, 1 = one smem tile written by a
// TMA bulk store (the next tile waits for it to be read), 2 = two tiles alternating (the next
// tile is zeroed / scattered while the previous store still drains)
__device__ __forceinline__ void bulk_tile_wait(int bulk) {
    if (bulk == 2) bulk_wait_read1();
    else if (bulk == 1) bulk_wait_read0();
}

// ------------------------------------------------ 128-bit shifted warp copy ---
// bytes [sh, sh+16) of the 32-byte little-endian string a||b (sh in 1..15)
template <int WS>
__device__ __forceinline__ uint4 merge_ws(const uint32_t (&w)[8], uint32_t bs) {
    uint4 r;
    r.x = __funnelshift_r(w[WS + 0], w[WS + 1], bs);
    r.y = __funnelshift_r(w[WS + 1], w[WS + 2], bs);
    r.z = __funnelshift_r(w[WS + 2], w[WS + 3], bs);
    r.w = __funnelshift_r(w[WS + 3], w[WS + 4], bs);
    return r;
}
__device__ __forceinline__ uint4 shift_merge(uint4 a, uint4 b, uint32_t sh) {
    const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    const uint32_t bs = (sh & 3u) * 8u;
    switch (sh >> 2) {  // warp-uniform
        case 0: return merge_ws<0>(w, bs);
        case 1: return merge_ws<1>(w, bs);
        case 2: return merge_ws<2>(w, bs);
        default: return merge_ws<3>(w, bs);
    }
}

// Warp-cooperative memcpy of n bytes between arbitrary alignments: byte head
// up to the destination's 16-B boundary, then aligned 16-B stores fed by
// aligned 16-B loads re-aligned with funnel shifts (neighbour chunk via shfl).
__device__ __forceinline__ void warp_copy(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src, uint64_t n,
                                          uint32_t lane) {
    if (n == 0) return;
    uint32_t head = (16u - static_cast<uint32_t>(reinterpret_cast<uintptr_t>(dst) & 15u)) & 15u;
    if (head > n) head = static_cast<uint32_t>(n);
    if (lane < head) dst[lane] = src[lane];
    dst += head;
    src += head;
    n -= head;
    const uint64_t nvec = n >> 4;
    const uint32_t sh = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(src) & 15u);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    if (sh == 0) {
        const uint4* s4 = reinterpret_cast<const uint4*>(src);
        uint64_t i = lane;
        for (; i + 96 < nvec; i += 128) {
            const uint4 v0 = ld_v4(s4 + i), v1 = ld_v4(s4 + i + 32), v2 = ld_v4(s4 + i + 64),
                        v3 = ld_v4(s4 + i + 96);
            st_v4(d4 + i, v0);
            st_v4(d4 + i + 32, v1);
            st_v4(d4 + i + 64, v2);
            st_v4(d4 + i + 96, v3);
        }
        for (; i < nvec; i += 32) st_v4(d4 + i, ld_v4(s4 + i));
    } else {
        // destination chunk i = source bytes straddling aligned chunks i and i+1;
        // both are loaded through L1 (chunk i+1 is the next lane's chunk i, an L1
        // hit), 4 pairs in flight per lane
        const uint4* s4 = reinterpret_cast<const uint4*>(src - sh);
        constexpr int UC = 4;
        for (uint64_t base = 0; base < nvec; base += 32 * UC) {
            uint4 a[UC], b[UC];
#pragma unroll
            for (int k = 0; k < UC; ++k) {
                const uint64_t i = base + k * 32 + lane;
                if (i < nvec) {
                    a[k] = __ldg(s4 + i);
                    b[k] = __ldg(s4 + i + 1);
                }
            }
#pragma unroll
            for (int k = 0; k < UC; ++k) {
                const uint64_t i = base + k * 32 + lane;
                if (i < nvec) st_v4(d4 + i, shift_merge(a[k], b[k], sh));
            }
        }
    }
    const uint64_t done = nvec << 4;
    const uint32_t rem = static_cast<uint32_t>(n - done);
    if (lane < rem) dst[done + lane] = src[done + lane];
}

// ------------------------------------------------------- CSR record access ---
struct CsrRow {
    const uint8_t* idx;
    const uint8_t* val;
    uint64_t nnz;
};

// Locate a row inside its chunk record: [rows u32][nnz u64][indptr][indices][data]
// IdxT = uint16_t: the narrowed staging layout (u32 indptr, u16 indices padded
// to 8 B, kernels.cuh ArenaView::idx16).
template <typename IdxT>
__device__ __forceinline__ CsrRow csr_row(const ArenaDev& a, const RowRef& r, uint32_t vs) {
    using PtrT = std::conditional_t<sizeof(IdxT) == 2, uint32_t, IdxT>;
    const uint8_t* rec = a.base + r.rec_off;
    const uint64_t within = r.gidx % a.chunk_rows;
    const uint32_t rows = ld_u32(rec);
    const uint64_t nnz_chunk = ld_u64_a4(rec + 4);
    const uint8_t* ip = rec + kCsrHeaderBytes;
    const uint64_t lo = ld_index<PtrT>(ip + within * sizeof(PtrT));
    const uint64_t hi = ld_index<PtrT>(ip + (within + 1) * sizeof(PtrT));
    const uint8_t* idx_base = ip + (static_cast<uint64_t>(rows) + 1) * sizeof(PtrT);
    const uint64_t idx_bytes = sizeof(IdxT) == 2 ? ((2 * nnz_chunk + 7) & ~7ull) : nnz_chunk * sizeof(IdxT);
    const uint8_t* val_base = idx_base + idx_bytes;
    return {idx_base + lo * sizeof(IdxT), val_base + lo * vs, hi - lo};
}

struct RowDesc {
    const uint8_t* idx;
    const uint8_t* val;
    uint64_t nnz;
    uint64_t gidx;
};
template <typename IdxT>
__device__ __forceinline__ RowDesc describe_row(const ArenaDev& a, const RowRef& r, uint32_t vs) {
    const CsrRow c = csr_row<IdxT>(a, r, vs);
    return {c.idx, c.val, c.nnz, r.gidx};
}

// ============================================================ K1/K2 gather ===
// Two launches: (1) k_row_scan — one thread per row resolves the row inside its
// chunk record (ref -> header -> indptr), a block scan plus a decoupled
// look-back across 128-row tiles (dynamic tile ids, 32-tile windows) writes the
// output indptr and a per-row job table {indices ptr, values ptr};
// (2) k_csr_copy — every warp grid-strides over (row, array) copy jobs with the
// 128-bit shifted warp copy; no barriers, so the whole GPU stays busy.
constexpr int kScanThreads = 128;
constexpr uint64_t kFlagA = 1ull << 62, kFlagP = 2ull << 62, kValMask = (1ull << 62) - 1;

struct RowJob {
    const uint8_t* idx;
    const uint8_t* val;
};

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

template <typename IdxT>
__global__ void __launch_bounds__(kScanThreads)
    k_row_scan(ArenaDev a, uint32_t vs, const RowRef* __restrict__ refs, uint64_t n_rows,
               uint64_t* __restrict__ out_prefix, RowJob* __restrict__ jobs, uint64_t* __restrict__ out_gidx,
               unsigned long long* __restrict__ scratch, const uint64_t* __restrict__ counts) {
    __shared__ uint64_t s_warp[kScanThreads / 32];
    __shared__ uint64_t s_tile, s_prefix;
    unsigned long long* counter = scratch;
    unsigned long long* status = scratch + 1;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    // dynamic tile ids make the look-back deadlock free (earlier tiles are resident)
    if (tid == 0) s_tile = atomicAdd(counter, 1ull);
    __syncthreads();
    const uint64_t tile = s_tile;
    const uint64_t row = tile * kScanThreads + tid;
    uint64_t nnz = 0;
    if (row < n_rows && counts) {
        nnz = counts[row];  // scan of given per-row counts (column reprojection)
    } else if (row < n_rows) {
        const RowRef r = refs[row];
        const CsrRow cr = csr_row<IdxT>(a, r, vs);
        nnz = cr.nnz;
        if (jobs) jobs[row] = {cr.idx, cr.val};
        if (out_gidx) out_gidx[row] = r.gidx;
    }
    uint64_t incl = nnz;  // warp-level indptr scan, then across the block's warps
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t v = __shfl_up_sync(kFull, incl, o);
        if (lane >= static_cast<uint32_t>(o)) incl += v;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    uint64_t agg = 0;
    for (uint32_t w = 0; w < kScanThreads / 32; ++w) {
        if (w < warp) incl += s_warp[w];
        agg += s_warp[w];
    }
    if (warp == 0) {  // decoupled look-back over a 32-tile window
        uint64_t prefix = 0;
        if (tile == 0) {
            if (lane == 0) st_volatile_u64(&status[0], kFlagP | agg);
        } else {
            if (lane == 0) st_volatile_u64(&status[tile], kFlagA | agg);
            int64_t end = static_cast<int64_t>(tile) - 1;
            for (;;) {
                const int64_t p = end - static_cast<int64_t>(lane);
                const uint64_t s = p >= 0 ? ld_volatile_u64(&status[p]) : kFlagP;
                const uint32_t flag = static_cast<uint32_t>(s >> 62);
                const uint32_t pmask = __ballot_sync(kFull, flag == 2);
                const uint32_t zmask = __ballot_sync(kFull, flag == 0);
                const uint32_t first = pmask ? static_cast<uint32_t>(__ffs(pmask) - 1) : 31u;
                const uint32_t need = first == 31u ? kFull : ((2u << first) - 1u);
                if (zmask & need) continue;  // a predecessor has not published yet
                prefix += warp_sum_u64(lane <= first ? (s & kValMask) : 0);
                if (pmask) break;
                end -= 32;
            }
            if (lane == 0) st_volatile_u64(&status[tile], kFlagP | (prefix + agg));
        }
        if (lane == 0) s_prefix = prefix;
    }
    __syncthreads();
    if (row < n_rows) out_prefix[row] = s_prefix + incl - nnz;
    if (tid == 0 && (tile + 1) * kScanThreads >= n_rows) out_prefix[n_rows] = s_prefix + agg;
}

// K2 from narrowed staging (ArenaView::idx16): one warp per row (grid-stride),
// u16 column ids widened to the store's u32 on the way out, values moved with
// the shifted 128-bit warp copy; `P` is the host-planned prefix.
__global__ void __launch_bounds__(256)
    k_csr_gather_idx16(ArenaDev a, uint32_t vs, const RowRef* __restrict__ refs, const uint64_t* __restrict__ P,
                       uint64_t n_rows, uint32_t* __restrict__ out_idx, uint8_t* __restrict__ out_val,
                       uint64_t* __restrict__ out_gidx) {
    pdl_wait();
    pdl_trigger();
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t warps = static_cast<uint64_t>(gridDim.x) * 8;
    const uint64_t p0 = P[0];
    for (uint64_t r = static_cast<uint64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5); r < n_rows; r += warps) {
        const RowRef ref = refs[r];
        if (lane == 0 && out_gidx) out_gidx[r] = ref.gidx;
        const CsrRow c = csr_row<uint16_t>(a, ref, vs);
        const uint64_t off = P[r] - p0, cnt = umin64(P[r + 1] - P[r], c.nnz);
        const unsigned short* src = reinterpret_cast<const unsigned short*>(c.idx);
        for (uint64_t k = lane; k < cnt; k += 32) out_idx[off + k] = __ldg(src + k);
        warp_copy(out_val + off * vs, c.val, cnt * vs, lane);
    }
}

// Delta-staged record -> idx16 record (kernels.cuh d8_*), one CTA per record:
// header + indptr and the values are copied word-wise; each warp rebuilds its
// rows' u16 columns with a warp inclusive scan of the u8 deltas (carry = the
// row's first column).
// 16 bytes at a 4-B aligned address (one 16-B load when it is 16-B aligned)
__device__ __forceinline__ void ld16_any(const uint8_t* p, uint32_t* w) {
    if ((reinterpret_cast<uintptr_t>(p) & 15u) == 0) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
        w[0] = v.x, w[1] = v.y, w[2] = v.z, w[3] = v.w;
    } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) w[q] = __ldg(reinterpret_cast<const uint32_t*>(p) + q);
    }
}
__device__ __forceinline__ void st16_any(void* p, const uint32_t* w) {
    if ((reinterpret_cast<uintptr_t>(p) & 15u) == 0) {
        *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
    } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) reinterpret_cast<uint32_t*>(p)[q] = w[q];
    }
}

// ---- bit-packed column deltas (kD8Packed, kernels.cuh d8_packed_layout) ----
__device__ __forceinline__ uint32_t nibble_sum(uint32_t x) {
    return (((x & 0x0F0F0F0Fu) + ((x >> 4) & 0x0F0F0F0Fu)) * 0x01010101u) >> 24;
}
// bit offset of group g's deltas (from the record's packed-bits start) and its width
__device__ __forceinline__ uint32_t packed_group(const uint8_t* widths, const uint8_t* skip, uint64_t g,
                                                 uint32_t& w) {
    const uint64_t s = g >> 5;
    const uint32_t n = static_cast<uint32_t>(g & 31);  // widths of groups 32s .. g-1 to add
    uint32_t sum = 0;
#pragma unroll
    for (uint32_t q = 0; q < 4; ++q) {
        const int k = static_cast<int>(n) - 8 * static_cast<int>(q);  // nibbles of this word before g
        if (k <= 0) break;
        const uint32_t word = ld_u32(widths + 16 * s + 4 * q);
        sum += nibble_sum(k >= 8 ? word : word & ((1u << (4 * k)) - 1u));
    }
    w = (static_cast<uint32_t>(__ldg(widths + (g >> 1))) >> (4 * (g & 1))) & 15u;
    return ld_u32(skip + 4 * s) + 16u * sum;
}
// the 16 deltas of a group as bytes of d[4] (LSB-first w-bit fields; the stream has 16 B slack)
__device__ __forceinline__ void unpack16(const uint8_t* bits, uint32_t off, uint32_t w, uint32_t (&d)[4]) {
#pragma unroll
    for (int q = 0; q < 4; ++q) d[q] = 0u;
    if (w == 0) return;
    const uint32_t* p = reinterpret_cast<const uint32_t*>(bits) + (off >> 5);
    uint32_t x[5];
#pragma unroll
    for (int q = 0; q < 5; ++q) x[q] = __ldg(p + q);
    const uint32_t sh = off & 31u, mask = (1u << w) - 1u;
#pragma unroll
    for (uint32_t j = 0; j < 16; ++j) {
        const uint32_t pos = sh + j * w, wi = pos >> 5, b = pos & 31u;
        const uint32_t lo = wi == 0 ? x[0] : wi == 1 ? x[1] : wi == 2 ? x[2] : wi == 3 ? x[3] : x[4];
        const uint32_t hi = wi == 0 ? x[1] : wi == 1 ? x[2] : wi == 2 ? x[3] : x[4];
        d[j >> 2] |= ((__funnelshift_r(lo, hi, b) & mask) << (8 * (j & 3)));
    }
}

struct D8Jobs {
    uint32_t n, vs;
    uint64_t n_var;   // kOneHot4 rows
    uint32_t vfloat;  // kD8Int8: values are f32 (else i32)
    uint32_t pad;
    D8Job job[kMaxD8Jobs];
};


__global__ void __launch_bounds__(256) k_d8_decode(const __grid_constant__ D8Jobs jobs) {
    pdl_wait();
    pdl_trigger();
    const D8Job jb = jobs.job[blockIdx.x];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint32_t tid = blockIdx.y * 256 + threadIdx.x;  // within the record's CTAs (one warp per row)
    const uint32_t nt = gridDim.y * 256;
    if (jb.kind == kOneHot4) {  // 2-bit channel codes -> one-hot u8 rows, one 16-B output chunk per thread
        const uint64_t L = jobs.n_var / 4, cpr = jobs.n_var / 16, n_chunks = jb.bytes / 16;
        for (uint64_t j = tid; j < n_chunks; j += nt) {
            const uint64_t row = j / cpr, b = (j - row * cpr) * 16;
            const uint32_t c = static_cast<uint32_t>(b / L);
            const uint64_t p0 = b - c * L;
            const uint32_t w = ld_u32(jb.src + row * (L / 4) + p0 / 4);
            uint32_t o[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                uint32_t word = 0;
#pragma unroll
                for (int k = 0; k < 4; ++k) word |= (((w >> (2 * (4 * q + k))) & 3u) == c ? 1u : 0u) << (8 * k);
                o[q] = word;
            }
            reinterpret_cast<uint4*>(jb.dst)[j] = make_uint4(o[0], o[1], o[2], o[3]);
        }
        return;
    }
    if (jb.kind == kIdx16Copy) {  // staged as idx16 already (16-B aligned, 16-B multiple incl. padding reads)
        const uint4* s4 = reinterpret_cast<const uint4*>(jb.src);
        uint4* d4 = reinterpret_cast<uint4*>(jb.dst);
        for (uint64_t i = tid; i < (jb.bytes + 15) / 16; i += nt) d4[i] = ld_v4(s4 + i);
        return;
    }
    const uint32_t kind = jb.kind & ~kD8Packed;
    const bool packed = (jb.kind & kD8Packed) != 0;
    const bool coded = kind == kD8Coded || kind == kD8Coded16;
    const uint32_t low_b = kind == kD8Coded16 ? 1u : 3u;
    const uint64_t rows = ld_u32(jb.src), nnz = ld_u64_a4(jb.src + 4);
    uint64_t dsec = ~0ull;
    D8Packed PL{};
    if (packed) {
        PL = d8_packed_layout(rows, nnz, ld_u32(jb.src + d8_packed_layout(rows, nnz, 0).pbytes_at));
        dsec = PL.end - PL.pbytes_at;
    }
    const uint64_t head = kCsrHeaderBytes + 4 * (rows + 1);
    const uint32_t* s32 = reinterpret_cast<const uint32_t*>(jb.src);
    uint32_t* d32 = reinterpret_cast<uint32_t*>(jb.dst);
    for (uint64_t i = tid; i < head / 4; i += nt) d32[i] = __ldg(s32 + i);
    const uint8_t* first = jb.src + head;
    const uint8_t* delta = first + ((2 * rows + 3) & ~3ull);
    uint8_t* dv = jb.dst + head + ((2 * nnz + 7) & ~7ull);
    D8vLayout L{};
    if (coded) {
        L = d8v_layout(rows, nnz, ld_u32(jb.src + d8v_layout(rows, nnz, 0, low_b, dsec).n_esc), low_b, dsec);
    } else if (kind == kD8IntP) {  // bit-packed integer values, one group of 16 per thread
        const uint64_t vo = d8_values_offset(rows, nnz, dsec);
        const D8Packed V = d8_packed_at(vo, nnz, ld_u32(jb.src + vo));
        for (uint64_t g = tid; g * 16 < nnz; g += nt) {
            uint32_t w, v4[4];
            const uint32_t off = packed_group(jb.src + V.widths, jb.src + V.skip, g, w);
            unpack16(jb.src + V.bits, off, w, v4);
            for (uint32_t j = 0; j < 16 && g * 16 + j < nnz; ++j) {
                const uint32_t u = (v4[j >> 2] >> (8 * (j & 3))) & 255u;
                reinterpret_cast<uint32_t*>(dv)[g * 16 + j] = jobs.vfloat ? __float_as_uint(static_cast<float>(u)) : u;
            }
        }
    } else if (kind == kD8Int8) {  // 1-byte integer values -> 4-byte f32 / i32
        const uint64_t voff = d8_values_offset(rows, nnz, dsec);
        const uint8_t* sv = jb.src + voff;
        for (uint64_t i = tid; i < nnz; i += nt) {
            const uint32_t u = __ldg(sv + i);
            reinterpret_cast<uint32_t*>(dv)[i] = jobs.vfloat ? __float_as_uint(static_cast<float>(u)) : u;
        }
    } else {  // raw values: copied word-wise (+ byte tail)
        const uint64_t voff = d8_values_offset(rows, nnz, dsec);
        const uint64_t vbytes = nnz * jobs.vs;
        const uint8_t* sv = jb.src + voff;
        for (uint64_t i = tid; i < vbytes / 4; i += nt)
            reinterpret_cast<uint32_t*>(dv)[i] = __ldg(reinterpret_cast<const uint32_t*>(sv) + i);
        for (uint64_t i = (vbytes & ~3ull) + tid; i < vbytes; i += nt) dv[i] = sv[i];
    }
    // rows: one warp each, 512 entries per step, 16 consecutive entries per lane
    // starting at a 16-entry boundary of the record (entries outside the row are
    // masked): vector loads of 16 deltas / 32 code bits / 16 or 48 low bytes, a
    // lane-local prefix, then ONE warp scan of (delta sum | escape count << 20)
    const uint8_t* ip = jb.src + kCsrHeaderBytes;
    uint8_t* cout = jb.dst + head;  // u16 columns
    const uint32_t dict = coded ? ld_u32(jb.src + L.dict) : 0u;
    for (uint64_t r = blockIdx.y * 8 + warp; r < rows; r += gridDim.y * 8) {
        const uint64_t lo = ld_u32(ip + 4 * r), hi = ld_u32(ip + 4 * (r + 1));
        uint32_t carry = __ldg(reinterpret_cast<const unsigned short*>(first) + r);
        uint32_t esc_at = coded ? ld_u32(jb.src + L.esc_base + 4 * r) : 0u;
        for (uint64_t base = lo & ~15ull; base < hi; base += 512) {
            const uint64_t k0 = base + 16 * lane;
            const uint32_t a = k0 < lo ? static_cast<uint32_t>(lo - k0) : 0u;
            const uint32_t b = k0 >= hi ? 0u : static_cast<uint32_t>(umin64(hi - k0, 16));
            const uint32_t vm = b > a ? ((b == 32u ? 0u : (1u << b)) - (1u << a)) & 0xffffu : 0u;  // valid entries
            const bool vec = k0 + 16 <= nnz;  // whole 16-entry group inside the record's arrays
            uint32_t d[4] = {0u, 0u, 0u, 0u}, cw = 0u, lw[12];
            if (vm && packed) {
                uint32_t w;
                const uint32_t off = packed_group(jb.src + PL.widths, jb.src + PL.skip, k0 >> 4, w);
                unpack16(jb.src + PL.bits, off, w, d);
            }
            if (vm) {
                if (vec) {
                    if (!packed) ld16_any(delta + k0, d);
                    if (coded) cw = ld_u32(jb.src + L.codes + (k0 >> 2));
                    if (coded && low_b == 1) ld16_any(jb.src + L.low3 + k0, lw);
                    if (coded && low_b == 3) {
                        ld16_any(jb.src + L.low3 + 3 * k0, lw);
                        ld16_any(jb.src + L.low3 + 3 * k0 + 16, lw + 4);
                        ld16_any(jb.src + L.low3 + 3 * k0 + 32, lw + 8);
                    }
                } else {  // the record's last group: byte loads of the entries that exist
#pragma unroll
                    for (int q = 0; q < 12; ++q) lw[q] = 0u;
#pragma unroll
                    for (uint32_t j = 0; j < 16; ++j) {
                        if (k0 + j >= nnz) continue;
                        if (!packed) d[j >> 2] |= static_cast<uint32_t>(__ldg(delta + k0 + j)) << (8 * (j & 3));
                        if (coded) cw |= ((static_cast<uint32_t>(__ldg(jb.src + L.codes + ((k0 + j) >> 2))) >>
                                           (2 * ((k0 + j) & 3))) & 3u) << (2 * j);
                        if (coded && low_b == 1)
                            lw[j >> 2] |= static_cast<uint32_t>(__ldg(jb.src + L.low3 + k0 + j)) << (8 * (j & 3));
                        if (coded && low_b == 3)
#pragma unroll
                            for (uint32_t t = 0; t < 3; ++t)
                                lw[(3 * j + t) >> 2] |= static_cast<uint32_t>(__ldg(jb.src + L.low3 + 3 * (k0 + j) + t))
                                                        << (8 * ((3 * j + t) & 3));
                    }
                }
            }
            uint32_t pre[16], s = 0;
#pragma unroll
            for (uint32_t j = 0; j < 16; ++j) {
                s += (vm >> j) & 1u ? (d[j >> 2] >> (8 * (j & 3))) & 255u : 0u;
                pre[j] = s;
            }
            uint32_t em = 0;  // escape entries (code 3) among the valid ones
            if (coded) {
#pragma unroll
                for (uint32_t j = 0; j < 16; ++j) em |= (((cw >> (2 * j)) & 3u) == 3u ? 1u : 0u) << j;
                em &= vm;
            }
            const uint32_t mine = s | (static_cast<uint32_t>(__popc(em)) << 20);
            uint32_t incl = mine;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(kFull, incl, o);
                if (lane >= static_cast<uint32_t>(o)) incl += t;
            }
            const uint32_t tot = __shfl_sync(kFull, incl, 31), excl = incl - mine;
            const uint32_t cb = carry + (excl & 0xfffffu);
            uint32_t eb = esc_at + (excl >> 20);
            carry += tot & 0xfffffu;
            esc_at += tot >> 20;
            if (!vm) continue;
            uint32_t cwd[8];
#pragma unroll
            for (uint32_t m = 0; m < 8; ++m) cwd[m] = ((cb + pre[2 * m]) & 0xffffu) | ((cb + pre[2 * m + 1]) << 16);
            if (vm == 0xffffu) {
                st16_any(cout + 2 * k0, cwd);
                st16_any(cout + 2 * k0 + 16, cwd + 4);
            } else {
#pragma unroll
                for (uint32_t j = 0; j < 16; ++j)
                    if ((vm >> j) & 1u)
                        reinterpret_cast<uint16_t*>(cout)[k0 + j] = static_cast<uint16_t>(cb + pre[j]);
            }
            if (coded) {  // top byte from the dictionary or the escape list, low bytes verbatim
                uint32_t v[16];
#pragma unroll
                for (uint32_t j = 0; j < 16; ++j) {
                    const uint32_t code = (cw >> (2 * j)) & 3u;
                    uint32_t top = (dict >> (8 * code)) & 255u;
                    if ((em >> j) & 1u) top = __ldg(jb.src + L.esc + eb++);
                    uint32_t low;
                    if (low_b == 1) {
                        low = ((lw[j >> 2] >> (8 * (j & 3))) & 255u) << 16;
                    } else {
                        low = 0u;
#pragma unroll
                        for (uint32_t t = 0; t < 3; ++t) low |= ((lw[(3 * j + t) >> 2] >> (8 * ((3 * j + t) & 3))) & 255u) << (8 * t);
                    }
                    v[j] = (top << 24) | low;
                }
                uint32_t* vo = reinterpret_cast<uint32_t*>(dv) + k0;
                if (vm == 0xffffu) {
#pragma unroll
                    for (uint32_t q = 0; q < 4; ++q) st16_any(vo + 4 * q, v + 4 * q);
                } else {
#pragma unroll
                    for (uint32_t j = 0; j < 16; ++j)
                        if ((vm >> j) & 1u) vo[j] = v[j];
                }
            }
        }
    }
}

// ============================================================ K5 record pack ===
template <typename T>
__device__ __forceinline__ void st_any(uint8_t* p, T v) {  // little-endian store at any alignment
    if ((reinterpret_cast<uintptr_t>(p) & (sizeof(T) - 1)) == 0) {
        *reinterpret_cast<T*>(p) = v;
        return;
    }
    for (uint32_t b = 0; b < sizeof(T); ++b) p[b] = static_cast<uint8_t>(static_cast<uint64_t>(v) >> (8 * b));
}

constexpr int kPackThreads = 256;

// Rows refs[0..n) -> consecutive encoded CSR chunk records of `cr` rows
// (encode_csr_record, store.cpp:52-64; only the last chunk may be short).  With
// P the exclusive nnz prefix over the launch, every record offset is closed
// form: record q starts at q*(12 + os*(cr+1)) + (os+vs)*P[q*cr].  One warp per
// row writes its indptr entry and copies its indices/values straight into
// place, so the payload moves HBM->HBM exactly once.
template <typename InIdx, typename OutIdx>
__global__ void __launch_bounds__(kPackThreads)
    k_csr_pack(ArenaDev a, uint32_t vs, const RowRef* __restrict__ refs, uint64_t n_rows, uint64_t cr,
               const uint64_t* __restrict__ P, uint8_t* __restrict__ out) {
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * (kPackThreads / 32);
    constexpr uint64_t os = sizeof(OutIdx);
    const uint64_t pb = P[0];  // P may be a slice of a longer scan
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * (kPackThreads / 32) + warp; i < n_rows; i += nw) {
        const uint64_t q = i / cr, r0 = q * cr;
        const uint64_t rows_q = umin64(cr, n_rows - r0);
        const uint64_t p0 = P[r0], nnz_q = P[r0 + rows_q] - p0;
        uint8_t* rec = out + q * (kCsrHeaderBytes + os * (cr + 1)) + (os + vs) * (p0 - pb);
        uint8_t* ip = rec + kCsrHeaderBytes;
        uint8_t* idx = ip + os * (rows_q + 1);
        uint8_t* val = idx + os * nnz_q;
        const uint64_t lo = P[i] - p0, hi = P[i + 1] - p0;
        if (lane == 0) {
            if (i == r0) {
                st_any<uint32_t>(rec, static_cast<uint32_t>(rows_q));
                st_any<uint64_t>(rec + 4, nnz_q);
                st_any<OutIdx>(ip, OutIdx(0));
            }
            st_any<OutIdx>(ip + os * (i - r0 + 1), static_cast<OutIdx>(hi));
        }
        const CsrRow src = csr_row<InIdx>(a, refs[i], vs);
        if (sizeof(InIdx) == sizeof(OutIdx)) {
            warp_copy(idx + os * lo, src.idx, (hi - lo) * os, lane);
        } else {
            for (uint64_t k = lane; k < hi - lo; k += 32)
                st_any<OutIdx>(idx + os * (lo + k), static_cast<OutIdx>(ld_index<InIdx>(src.idx + k * sizeof(InIdx))));
        }
        warp_copy(val + vs * lo, src.val, (hi - lo) * vs, lane);
    }
}

// ============================================================ K3 densify =====

template <typename D, typename S>
struct Conv {
    __device__ static D go(S x, float scale, int norm);
};
template <typename S>
struct Conv<float, S> {
    __device__ static float go(S x, float scale, int norm) {
        const float v = static_cast<float>(x);
        return norm ? log1pf(v * scale) : v;
    }
};
template <>
struct Conv<float, double> {
    __device__ static float go(double x, float scale, int norm) {
        return norm ? log1pf(static_cast<float>(x * static_cast<double>(scale))) : static_cast<float>(x);
    }
};
template <typename S>
struct Conv<__nv_bfloat16, S> {
    __device__ static __nv_bfloat16 go(S x, float scale, int norm) {
        return __float2bfloat16_rn(Conv<float, S>::go(x, scale, norm));
    }
};
template <>
struct Conv<double, double> {
    __device__ static double go(double x, float, int) { return x; }
};
template <>
struct Conv<int32_t, int32_t> {
    __device__ static int32_t go(int32_t x, float, int) { return x; }
};
template <>
struct Conv<uint8_t, uint8_t> {
    __device__ static uint8_t go(uint8_t x, float, int) { return x; }
};

__device__ __forceinline__ double block_sum(double v, double* red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double t = 0.0;
    for (uint32_t w = 0; w < blockDim.x / 32; ++w) t += red[w];  // fixed order: deterministic
    __syncthreads();
    return t;
}

// ============================================================ K3 densify v6 ===
// Same smem-tile + TMA bulk store scheme as above, with two rows in flight per
// CTA: while row i's tiles are zeroed/scattered/stored, row i+1's first U*THREADS
// entries are already loading into a second register set, and the record
// lookup (ref -> header -> indptr) runs two rows ahead.  Columns are kept as u32
// (n_var < 2^32; indices were validated at store open), which keeps both
// register sets spill-free.
template <typename IdxT, typename SrcT, int U>
__device__ __forceinline__ void load_entries(const RowDesc& d, uint32_t tid, uint32_t nthr, uint32_t (&col)[U],
                                             SrcT (&v)[U]) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const uint64_t k = tid + static_cast<uint64_t>(u) * nthr;
        col[u] = ~0u;
        if (k < d.nnz) {
            const uint64_t c = ld_index<IdxT>(d.idx + k * sizeof(IdxT));
            col[u] = c < 0xFFFFFFFFull ? static_cast<uint32_t>(c) : ~0u;
            v[u] = ld_value<SrcT>(d.val + k * sizeof(SrcT));
        }
    }
}

template <typename IdxT, typename SrcT, typename DstT, int THREADS, int U, int MINB>
__global__ void __launch_bounds__(THREADS, MINB)
    k_csr_densify6(ArenaDev a, const RowRef* __restrict__ refs, uint64_t n_rows, uint32_t tile_cols, int norm,
                   float target, DstT* __restrict__ out, uint64_t* __restrict__ out_gidx, int bulk) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ double s_red[THREADS / 32];
    __shared__ RowDesc s_desc[3];  // rows i, i+1, i+2 of this CTA
    const uint32_t tid = threadIdx.x;
    constexpr uint32_t nthr = THREADS;
    const uint64_t n_var = a.n_var;
    const uint64_t g = gridDim.x;
    pdl_wait();
    pdl_trigger();
    if (tid == 0) {
        if (blockIdx.x < n_rows) s_desc[0] = describe_row<IdxT>(a, refs[blockIdx.x], sizeof(SrcT));
        if (blockIdx.x + g < n_rows) s_desc[1] = describe_row<IdxT>(a, refs[blockIdx.x + g], sizeof(SrcT));
    }
    __syncthreads();
    uint32_t colA[U], colB[U];
    SrcT vA[U], vB[U];
    if (blockIdx.x < n_rows) load_entries<IdxT, SrcT, U>(s_desc[0], tid, nthr, colA, vA);
    uint32_t slot = 0;
    for (uint64_t row = blockIdx.x; row < n_rows; row += g, slot = slot == 2 ? 0 : slot + 1) {
        const RowDesc d = s_desc[slot];
        const uint32_t nslot = slot == 2 ? 0 : slot + 1, nnslot = nslot == 2 ? 0 : nslot + 1;
        const bool has_next = row + g < n_rows;
        if (has_next) load_entries<IdxT, SrcT, U>(s_desc[nslot], tid, nthr, colB, vB);  // row i+1 in flight
        if (tid == 0) {
            if (row + 2 * g < n_rows) s_desc[nnslot] = describe_row<IdxT>(a, refs[row + 2 * g], sizeof(SrcT));
            if (out_gidx) out_gidx[row] = d.gidx;
        }
        float scale = 1.0f;
        if (norm) {  // library size in fp64
            double s = 0.0;
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (colA[u] != ~0u) s += static_cast<double>(vA[u]);
            for (uint64_t k = tid + U * nthr; k < d.nnz; k += nthr)
                s += static_cast<double>(ld_value<SrcT>(d.val + k * sizeof(SrcT)));
            s = block_sum(s, s_red);
            scale = s != 0.0 ? static_cast<float>(static_cast<double>(target) / s) : 0.0f;
        }
        DstT* orow = out + row * n_var;
        for (uint64_t c0 = 0; c0 < n_var; c0 += tile_cols) {
            const uint32_t cols = static_cast<uint32_t>(umin64(tile_cols, n_var - c0));
            const uint32_t bytes = cols * static_cast<uint32_t>(sizeof(DstT));
            DstT* tile = reinterpret_cast<DstT*>(smem);
            if (bulk && tid == 0) bulk_wait_read0();
            __syncthreads();
            uint4* t4 = reinterpret_cast<uint4*>(smem);
            for (uint32_t i = tid; i < bytes / 16u; i += nthr) t4[i] = make_uint4(0, 0, 0, 0);
            for (uint32_t i = (bytes & ~15u) + tid; i < bytes; i += nthr) smem[i] = 0;
            __syncthreads();
            const uint32_t c0u = static_cast<uint32_t>(c0);
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (colA[u] - c0u < cols) tile[colA[u] - c0u] = Conv<DstT, SrcT>::go(vA[u], scale, norm);
            for (uint64_t k = tid + U * nthr; k < d.nnz; k += nthr) {  // rows longer than U*THREADS
                const uint64_t c2 = ld_index<IdxT>(d.idx + k * sizeof(IdxT));
                if (c2 >= c0 && c2 - c0 < cols)
                    tile[c2 - c0] = Conv<DstT, SrcT>::go(ld_value<SrcT>(d.val + k * sizeof(SrcT)), scale, norm);
            }
            if (bulk) {
                fence_proxy_async_shared();
                __syncthreads();
                if (tid == 0) {
                    bulk_store(orow + c0, smem, bytes);
                    bulk_commit();
                }
            } else {
                __syncthreads();
                for (uint32_t i = tid; i < cols; i += nthr) orow[c0 + i] = tile[i];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            colA[u] = colB[u];
            vA[u] = vB[u];
        }
    }
    if (bulk && tid == 0) bulk_wait0();
}

// v9: v6 with the CTA's row lookups hoisted out of the row loop: warp 0
// resolves 32 rows lane-parallel up front instead of thread 0 walking one
// ref -> header -> indptr chain per row ahead of the tile barriers.
template <typename IdxT, typename SrcT, typename DstT, int THREADS, int U, int MINB>
__global__ void __launch_bounds__(THREADS, MINB)
    k_csr_densify9(ArenaDev a, const RowRef* __restrict__ refs, uint64_t n_rows, uint32_t tile_cols, int norm,
                   float target, DstT* __restrict__ out, uint64_t* __restrict__ out_gidx, int bulk) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ double s_red[THREADS / 32];
    __shared__ RowDesc s_desc[32];  // this CTA's rows k0 .. k0+31 (row = blockIdx.x + k * gridDim.x)
    const uint32_t tid = threadIdx.x;
    constexpr uint32_t nthr = THREADS;
    const uint64_t n_var = a.n_var;
    const uint64_t g = gridDim.x;
    pdl_wait();
    pdl_trigger();
    // warp 0 resolves the CTA's next 32 rows lane-parallel (ref -> header ->
    // indptr, one dependent chain for all of them) and writes their gidx
    auto describe32 = [&](uint64_t k0) {
        if (tid < 32) {
            const uint64_t row = blockIdx.x + (k0 + tid) * g;
            if (row < n_rows) {
                const RowDesc rd = describe_row<IdxT>(a, refs[row], sizeof(SrcT));
                s_desc[tid] = rd;
                if (out_gidx) out_gidx[row] = rd.gidx;
            }
        }
    };
    describe32(0);
    __syncthreads();
    uint32_t colA[U], colB[U];
    SrcT vA[U], vB[U];
    if (blockIdx.x < n_rows) load_entries<IdxT, SrcT, U>(s_desc[0], tid, nthr, colA, vA);
    uint64_t kk = 0;
    uint32_t tcount = 0;
    const uint32_t tile_stride = (tile_cols * static_cast<uint32_t>(sizeof(DstT)) + 127u) & ~127u;
    for (uint64_t row = blockIdx.x; row < n_rows; row += g, ++kk) {
        const RowDesc d = s_desc[kk & 31];
        const bool has_next = row + g < n_rows;
        if (has_next && ((kk + 1) & 31) == 0) {  // CTAs with > 32 rows: next batch of descriptors
            __syncthreads();
            describe32(kk + 1);
            __syncthreads();
        }
        if (has_next) load_entries<IdxT, SrcT, U>(s_desc[(kk + 1) & 31], tid, nthr, colB, vB);  // row i+1 in flight
        float scale = 1.0f;
        if (norm) {  // library size in fp64
            double s = 0.0;
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (colA[u] != ~0u) s += static_cast<double>(vA[u]);
            for (uint64_t k = tid + U * nthr; k < d.nnz; k += nthr)
                s += static_cast<double>(ld_value<SrcT>(d.val + k * sizeof(SrcT)));
            s = block_sum(s, s_red);
            scale = s != 0.0 ? static_cast<float>(static_cast<double>(target) / s) : 0.0f;
        }
        DstT* orow = out + row * n_var;
        for (uint64_t c0 = 0; c0 < n_var; c0 += tile_cols, ++tcount) {
            const uint32_t cols = static_cast<uint32_t>(umin64(tile_cols, n_var - c0));
            const uint32_t bytes = cols * static_cast<uint32_t>(sizeof(DstT));
            uint8_t* tb = smem + (bulk == 2 ? (tcount & 1u) * tile_stride : 0u);
            DstT* tile = reinterpret_cast<DstT*>(tb);
            if (tid == 0) bulk_tile_wait(bulk);
            __syncthreads();
            uint4* t4 = reinterpret_cast<uint4*>(tb);
            for (uint32_t i = tid; i < bytes / 16u; i += nthr) t4[i] = make_uint4(0, 0, 0, 0);
            for (uint32_t i = (bytes & ~15u) + tid; i < bytes; i += nthr) tb[i] = 0;
            __syncthreads();
            const uint32_t c0u = static_cast<uint32_t>(c0);
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (colA[u] - c0u < cols) tile[colA[u] - c0u] = Conv<DstT, SrcT>::go(vA[u], scale, norm);
            for (uint64_t k = tid + U * nthr; k < d.nnz; k += nthr) {  // rows longer than U*THREADS
                const uint64_t c2 = ld_index<IdxT>(d.idx + k * sizeof(IdxT));
                if (c2 >= c0 && c2 - c0 < cols)
                    tile[c2 - c0] = Conv<DstT, SrcT>::go(ld_value<SrcT>(d.val + k * sizeof(SrcT)), scale, norm);
            }
            if (bulk) {
                fence_proxy_async_shared();
                __syncthreads();
                if (tid == 0) {
                    bulk_store(orow + c0, tb, bytes);
                    bulk_commit();
                }
            } else {
                __syncthreads();
                for (uint32_t i = tid; i < cols; i += nthr) orow[c0 + i] = tile[i];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            colA[u] = colB[u];
            vA[u] = vB[u];
        }
    }
    if (bulk && tid == 0) bulk_wait0();
}

// ============================================ K3d densify from delta records ===
// K3 reading the staging image's delta records directly (kD8Raw / kD8Coded /
// kD8Coded16, kernels.cuh d8v_layout) instead of the idx16 records k_d8_decode
// would expand: the expansion's write + re-read of 6 B per entry disappears.
// RowRef.rec_off carries the record's D8Kind in bits 60..63.  Thread t holds
// the 16 consecutive entries [(lo & ~15) + 16 t, +16) of a row (rows of up to
// kD8FusedMaxNnz entries; the launcher's caller guarantees it): 16 column
// deltas, 32 code bits and the low value bytes arrive as vector loads one row
// ahead; at the row's turn ONE block scan of (delta sum | escape count << 17)
// yields every entry's column and escape rank, and the scatter into the smem
// tile + TMA bulk store is v9's.
constexpr uint64_t kKindShift = 60, kOffMask = (1ull << kKindShift) - 1;

struct D8RowDesc {
    const uint8_t* delta;  // column deltas u8 (record entry 0); packed: the group widths
    const uint8_t* pskip;  // packed: bit offset of every 32nd group
    const uint8_t* pbits;  // packed: the delta bit stream
    const uint8_t* low;    // kD8Raw: raw 4-B values; coded: low value bytes
    const uint8_t* codes;  // 2-bit top-byte codes
    const uint8_t* esc;    // escaped top bytes
    uint64_t gidx;
    uint32_t lo, hi, nrec;  // row entries [lo, hi) of the record's nrec
    uint32_t first, esc_at, dict, kind, packed;  // kind without the kD8Packed flag
};

__device__ __forceinline__ D8RowDesc describe_d8(const ArenaDev& a, const RowRef& r) {
    D8RowDesc d;
    const uint8_t* rec = a.base + (r.rec_off & kOffMask);
    d.kind = static_cast<uint32_t>(r.rec_off >> kKindShift);
    d.packed = d.kind & kD8Packed;
    d.kind &= ~kD8Packed;
    const uint64_t within = r.gidx % a.chunk_rows;
    const uint32_t rows = ld_u32(rec);
    const uint64_t nnz = ld_u64_a4(rec + 4);
    const uint8_t* ip = rec + kCsrHeaderBytes;
    d.lo = ld_u32(ip + 4 * within);
    d.hi = ld_u32(ip + 4 * (within + 1));
    d.nrec = static_cast<uint32_t>(nnz);
    const uint64_t first_off = kCsrHeaderBytes + 4 * (static_cast<uint64_t>(rows) + 1);
    d.first = __ldg(reinterpret_cast<const unsigned short*>(rec + first_off) + within);
    d.delta = rec + first_off + ((2 * static_cast<uint64_t>(rows) + 3) & ~3ull);
    d.gidx = r.gidx;
    uint64_t dsec = ~0ull;
    d.pskip = d.pbits = nullptr;
    if (d.packed) {
        const D8Packed P = d8_packed_layout(rows, nnz, ld_u32(d.delta));
        dsec = P.end - P.pbytes_at;
        d.delta = rec + P.widths;
        d.pskip = rec + P.skip;
        d.pbits = rec + P.bits;
    }
    if (d.kind == kD8IntP) {  // packed value bytes: codes = widths, esc = skip, low = bits
        const uint64_t vo = d8_values_offset(rows, nnz, dsec);
        const D8Packed V = d8_packed_at(vo, nnz, ld_u32(rec + vo));
        d.codes = rec + V.widths;
        d.esc = rec + V.skip;
        d.low = rec + V.bits;
        d.esc_at = d.dict = 0;
    } else if (d.kind == kD8Raw || d.kind == kD8Int8) {
        d.low = rec + d8_values_offset(rows, nnz, dsec);
        d.codes = d.esc = nullptr;
        d.esc_at = d.dict = 0;
    } else {
        const uint32_t lb = d.kind == kD8Coded16 ? 1 : 3;
        const D8vLayout L0 = d8v_layout(rows, nnz, 0, lb, dsec);
        const D8vLayout L = d8v_layout(rows, nnz, ld_u32(rec + L0.n_esc), lb, dsec);
        d.low = rec + L.low3;
        d.codes = rec + L.codes;
        d.esc = rec + L.esc;
        d.esc_at = ld_u32(rec + L.esc_base + 4 * within);
        d.dict = ld_u32(rec + L.dict);
    }
    return d;
}

struct D8Raw16 {  // one thread's 16 entries of a row, as loaded
    uint32_t d[4], cw, lw[16], vm;
};

__device__ __forceinline__ void load_d8(const D8RowDesc& r, uint32_t tid, D8Raw16& x) {
    const uint64_t k0 = (r.lo & ~15u) + 16ull * tid;
    const uint32_t a = k0 < r.lo ? static_cast<uint32_t>(r.lo - k0) : 0u;
    const uint32_t b = k0 >= r.hi ? 0u : static_cast<uint32_t>(umin64(r.hi - k0, 16));
    x.vm = b > a ? ((1u << b) - (1u << a)) & 0xffffu : 0u;
    x.cw = 0u;
#pragma unroll
    for (int q = 0; q < 4; ++q) x.d[q] = 0u;
#pragma unroll
    for (int q = 0; q < 16; ++q) x.lw[q] = 0u;
    if (!x.vm) return;
    const uint32_t kind = r.kind;
    if (r.packed) {
        uint32_t w;
        const uint32_t off = packed_group(r.delta, r.pskip, k0 >> 4, w);
        unpack16(r.pbits, off, w, x.d);
    }
    if (kind == kD8IntP) {  // 16 value bytes -> lw[0..3], like kD8Int8's
        uint32_t w, v4[4];
        const uint32_t off = packed_group(r.codes, r.esc, k0 >> 4, w);
        unpack16(r.low, off, w, v4);
#pragma unroll
        for (int q = 0; q < 4; ++q) x.lw[q] = v4[q];
        if (k0 + 16 <= r.nrec && !r.packed) ld16_any(r.delta + k0, x.d);
        if (k0 + 16 > r.nrec && !r.packed)
            for (uint32_t j = 0; j < 16; ++j)
                if (k0 + j < r.nrec) x.d[j >> 2] |= static_cast<uint32_t>(__ldg(r.delta + k0 + j)) << (8 * (j & 3));
        return;
    }
    if (k0 + 16 <= r.nrec) {
        if (!r.packed) ld16_any(r.delta + k0, x.d);
        if (kind == kD8Raw) {
#pragma unroll
            for (int q = 0; q < 4; ++q) ld16_any(r.low + 4 * k0 + 16 * q, x.lw + 4 * q);
        } else if (kind == kD8Int8) {
            ld16_any(r.low + k0, x.lw);
        } else {
            x.cw = ld_u32(r.codes + (k0 >> 2));
            if (kind == kD8Coded16) {
                ld16_any(r.low + k0, x.lw);
            } else {
#pragma unroll
                for (int q = 0; q < 3; ++q) ld16_any(r.low + 3 * k0 + 16 * q, x.lw + 4 * q);
            }
        }
        return;
    }
    // the record's last entry group: byte loads of the entries that exist
#pragma unroll
    for (uint32_t j = 0; j < 16; ++j) {
        if (k0 + j >= r.nrec) continue;
        const uint64_t k = k0 + j;
        if (!r.packed) x.d[j >> 2] |= static_cast<uint32_t>(__ldg(r.delta + k)) << (8 * (j & 3));
        if (kind == kD8Raw) {
            x.lw[j] = ld_u32(r.low + 4 * k);
        } else if (kind == kD8Int8) {
            x.lw[j >> 2] |= static_cast<uint32_t>(__ldg(r.low + k)) << (8 * (j & 3));
        } else {
            x.cw |= ((static_cast<uint32_t>(__ldg(r.codes + (k >> 2))) >> (2 * (k & 3))) & 3u) << (2 * j);
            if (kind == kD8Coded16) {
                x.lw[j >> 2] |= static_cast<uint32_t>(__ldg(r.low + k)) << (8 * (j & 3));
            } else {
#pragma unroll
                for (uint32_t t = 0; t < 3; ++t)
                    x.lw[(3 * j + t) >> 2] |= static_cast<uint32_t>(__ldg(r.low + 3 * k + t)) << (8 * ((3 * j + t) & 3));
            }
        }
    }
}

template <typename SrcT>
__device__ __forceinline__ SrcT from_bits(uint32_t b) {
    if constexpr (sizeof(SrcT) == 4 && std::is_floating_point_v<SrcT>) return __uint_as_float(b);
    else return static_cast<SrcT>(static_cast<int32_t>(b));
}

// columns (~0u = not an entry of the row) and values of one thread's 16 entries;
// s_scan: THREADS/32 words (one __syncthreads inside)
template <typename SrcT, int THREADS>
__device__ __forceinline__ void decode_d8(const D8RowDesc& r, const D8Raw16& x, uint32_t* s_scan, uint32_t (&col)[16],
                                          SrcT (&v)[16]) {
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    uint32_t pre[16], sum = 0;
#pragma unroll
    for (uint32_t j = 0; j < 16; ++j) {
        sum += (x.vm >> j) & 1u ? (x.d[j >> 2] >> (8 * (j & 3))) & 255u : 0u;
        pre[j] = sum;
    }
    uint32_t em = 0;
    if (r.kind == kD8Coded || r.kind == kD8Coded16) {
#pragma unroll
        for (uint32_t j = 0; j < 16; ++j) em |= (((x.cw >> (2 * j)) & 3u) == 3u ? 1u : 0u) << j;
        em &= x.vm;
    }
    const uint32_t mine = sum | (static_cast<uint32_t>(__popc(em)) << 17);
    uint32_t incl = mine;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(kFull, incl, o);
        if (lane >= static_cast<uint32_t>(o)) incl += t;
    }
    if (lane == 31) s_scan[warp] = incl;
    __syncthreads();
    uint32_t excl = incl - mine;
    for (uint32_t w = 0; w < warp; ++w) excl += s_scan[w];
    const uint32_t cb = r.first + (excl & 0x1ffffu);
    uint32_t eb = r.esc_at + (excl >> 17);
#pragma unroll
    for (uint32_t j = 0; j < 16; ++j) {
        col[j] = (x.vm >> j) & 1u ? cb + pre[j] : ~0u;
        uint32_t bits;
        if (r.kind == kD8Raw) {
            bits = x.lw[j];
        } else if (r.kind == kD8Int8 || r.kind == kD8IntP) {
            const uint32_t u = (x.lw[j >> 2] >> (8 * (j & 3))) & 255u;
            bits = std::is_floating_point_v<SrcT> ? __float_as_uint(static_cast<float>(u)) : u;
        } else {
            uint32_t top = (r.dict >> (8 * ((x.cw >> (2 * j)) & 3u))) & 255u;
            if ((em >> j) & 1u) top = __ldg(r.esc + eb++);
            uint32_t low;
            if (r.kind == kD8Coded16) {
                low = ((x.lw[j >> 2] >> (8 * (j & 3))) & 255u) << 16;
            } else {
                low = 0u;
#pragma unroll
                for (uint32_t t = 0; t < 3; ++t) low |= ((x.lw[(3 * j + t) >> 2] >> (8 * ((3 * j + t) & 3))) & 255u) << (8 * t);
            }
            bits = (top << 24) | low;
        }
        v[j] = from_bits<SrcT>(bits);
    }
}

template <typename SrcT, typename DstT, int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB)
    k_csr_densify_d8(ArenaDev a, const RowRef* __restrict__ refs, uint64_t n_rows, uint32_t tile_cols, int norm,
                     float target, DstT* __restrict__ out, uint64_t* __restrict__ out_gidx, int bulk) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ double s_red[THREADS / 32];
    __shared__ uint32_t s_scan[THREADS / 32];
    __shared__ D8RowDesc s_desc[32];
    const uint32_t tid = threadIdx.x;
    const uint64_t n_var = a.n_var;
    const uint64_t g = gridDim.x;
    pdl_wait();
    pdl_trigger();
    auto describe32 = [&](uint64_t k0) {
        if (tid < 32) {
            const uint64_t row = blockIdx.x + (k0 + tid) * g;
            if (row < n_rows) {
                const D8RowDesc rd = describe_d8(a, refs[row]);
                s_desc[tid] = rd;
                if (out_gidx) out_gidx[row] = rd.gidx;
            }
        }
    };
    describe32(0);
    __syncthreads();
    D8Raw16 raw;
    if (blockIdx.x < n_rows) load_d8(s_desc[0], tid, raw);
    uint32_t col[16];
    SrcT val[16];
    uint64_t kk = 0;
    uint32_t tcount = 0;
    const uint32_t tile_stride = (tile_cols * static_cast<uint32_t>(sizeof(DstT)) + 127u) & ~127u;
    for (uint64_t row = blockIdx.x; row < n_rows; row += g, ++kk) {
        const D8RowDesc d = s_desc[kk & 31];
        decode_d8<SrcT, THREADS>(d, raw, s_scan, col, val);  // (syncs: s_desc reads above are done)
        const bool has_next = row + g < n_rows;
        if (has_next && ((kk + 1) & 31) == 0) {
            __syncthreads();
            describe32(kk + 1);
            __syncthreads();
        }
        if (has_next) load_d8(s_desc[(kk + 1) & 31], tid, raw);  // row i+1 in flight
        float scale = 1.0f;
        if (norm) {  // library size in fp64
            double s = 0.0;
#pragma unroll
            for (int u = 0; u < 16; ++u)
                if (col[u] != ~0u) s += static_cast<double>(val[u]);
            s = block_sum(s, s_red);
            scale = s != 0.0 ? static_cast<float>(static_cast<double>(target) / s) : 0.0f;
        }
        DstT* orow = out + row * n_var;
        for (uint64_t c0 = 0; c0 < n_var; c0 += tile_cols, ++tcount) {
            const uint32_t cols = static_cast<uint32_t>(umin64(tile_cols, n_var - c0));
            const uint32_t bytes = cols * static_cast<uint32_t>(sizeof(DstT));
            uint8_t* tb = smem + (bulk == 2 ? (tcount & 1u) * tile_stride : 0u);
            DstT* tile = reinterpret_cast<DstT*>(tb);
            if (tid == 0) bulk_tile_wait(bulk);
            __syncthreads();
            uint4* t4 = reinterpret_cast<uint4*>(tb);
            for (uint32_t i = tid; i < bytes / 16u; i += THREADS) t4[i] = make_uint4(0, 0, 0, 0);
            for (uint32_t i = (bytes & ~15u) + tid; i < bytes; i += THREADS) tb[i] = 0;
            __syncthreads();
            const uint32_t c0u = static_cast<uint32_t>(c0);
#pragma unroll
            for (int u = 0; u < 16; ++u)
                if (col[u] - c0u < cols) tile[col[u] - c0u] = Conv<DstT, SrcT>::go(val[u], scale, norm);
            if (bulk) {
                fence_proxy_async_shared();
                __syncthreads();
                if (tid == 0) {
                    bulk_store(orow + c0, tb, bytes);
                    bulk_commit();
                }
            } else {
                __syncthreads();
                for (uint32_t i = tid; i < cols; i += THREADS) orow[c0 + i] = tile[i];
            }
        }
    }
    if (bulk && tid == 0) bulk_wait0();
}

// ------------------------------------------------ mbarrier + TMA bulk load ---
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
    }
}
__device__ __forceinline__ void bulk_load(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(sdst)),
                 "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// ===================================================== K2 copy, TMA staged ===
// The output of each array is cut into equal 16-B aligned byte ranges, one per
// warp of a persistent grid, with the source side moved to
// the async proxy: each warp streams its output range as pieces of <= 4 KB;
// one lane issues a 1-D TMA bulk load of the piece's 16-B aligned source
// superset into the warp's shared stage (completion on an mbarrier), two
// stages in flight, and the warp writes the piece with aligned 16-B stores,
// re-aligning neighbouring shared chunks with funnel shifts.  Bytes in flight
// no longer cost registers: 8 KB per warp regardless of row alignment.
constexpr int kTcWarps = 4;
constexpr int kTcThreads = kTcWarps * 32;
constexpr uint32_t kTcPiece = 4096;
constexpr uint32_t kTcStage = kTcPiece + 32;

struct TcPiece {
    const uint8_t* src;
    uint8_t* dst;
    uint32_t len;  // bytes; 0 = no piece
};

__device__ __forceinline__ uint4 lds_v4(uint32_t addr) {
    uint4 r;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(addr));
    return r;
}
__device__ __forceinline__ uint8_t lds_u8(uint32_t addr) {
    uint16_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=h"(v) : "r"(addr));
    return static_cast<uint8_t>(v);
}

// Generator of one warp's pieces (all state warp-uniform; rows resolved 32 at
// a time lane-parallel).
template <typename IdxT>
struct TcGen {
    ArenaDev a;
    const RowRef* refs;
    const RowJob* jobs;
    const uint64_t* P;
    uint64_t n_rows, p0, e0, e1, r;
    uint8_t* out;
    uint64_t cr;  // > 0: K5 mode, rows land in encoded chunk records of cr rows
    uint32_t es, vs, lane, act, k;
    bool is_val, more;
    uint64_t pl, ph, avail, pos;
    const uint8_t* src;

    __device__ void load_batch() {
        const uint64_t rl = r + lane;
        pl = ~0ull;
        ph = 0;
        if (rl < n_rows) {
            pl = P[rl] - p0;
            ph = P[rl + 1] - p0;
        }
        act = __ballot_sync(kFull, rl < n_rows && pl < e1);
        src = nullptr;
        avail = 0;
        if ((act >> lane) & 1u) {
            if (jobs) {
                const RowJob jb = jobs[rl];
                src = is_val ? jb.val : jb.idx;
                avail = ph - pl;
            } else {
                const CsrRow c = csr_row<IdxT>(a, refs[rl], vs);
                src = is_val ? c.val : c.idx;
                avail = c.nnz;
            }
        }
        more = act == kFull && __shfl_sync(kFull, ph, 31) < e1;
        k = 0;
        pos = 0;
    }
    __device__ TcPiece next() {
        for (;;) {
            if (k >= 32 || !((act >> k) & 1u)) {
                if (!more) return {nullptr, nullptr, 0};
                r += 32;
                load_batch();
                continue;
            }
            const uint64_t kpl = __shfl_sync(kFull, pl, k), kph = __shfl_sync(kFull, ph, k);
            const uint64_t kav = __shfl_sync(kFull, avail, k);
            const uint64_t s = (kpl > e0 ? kpl : e0) + pos, t = umin64(kph, e1);
            const uint64_t in_row = s - kpl;
            const uint64_t lim = kav > in_row ? umin64(t, kpl + kav) : s;  // reads clamped to the row
            if (s >= lim) {
                ++k;
                pos = 0;
                continue;
            }
            uint8_t* dst = out + s * es;
            if (cr) {  // record q = row / cr starts at q*(12 + es_i*(cr+1)) + (es_i+vs)*P[q*cr] (k_csr_pack)
                const uint64_t row = r + k, q = row / cr, r0 = q * cr, rows_q = umin64(cr, n_rows - r0);
                const uint64_t p0q = P[r0] - p0, nnz_q = P[r0 + rows_q] - P[r0];
                const uint64_t is_ = sizeof(IdxT);
                uint8_t* rec = out + q * (kCsrHeaderBytes + is_ * (cr + 1)) + (is_ + vs) * p0q;
                uint8_t* ibase = rec + kCsrHeaderBytes + is_ * (rows_q + 1);
                dst = (is_val ? ibase + is_ * nnz_q : ibase) + (s - p0q) * es;
            }
            const uint64_t room = kTcPiece - (reinterpret_cast<uintptr_t>(dst) & 15u);
            const uint64_t len = umin64((lim - s) * es, room);
            const uint8_t* ks =
                reinterpret_cast<const uint8_t*>(__shfl_sync(kFull, reinterpret_cast<unsigned long long>(src), k));
            pos += len / es;
            return {ks + in_row * es, dst, static_cast<uint32_t>(len)};
        }
    }
};

__device__ __forceinline__ void tc_issue(const TcPiece& pc, uint8_t* stage, uint64_t* bar, uint32_t lane) {
    if (lane == 0 && pc.len) {
        const uintptr_t lo = reinterpret_cast<uintptr_t>(pc.src) & ~uintptr_t(15);
        const uintptr_t hi = (reinterpret_cast<uintptr_t>(pc.src) + pc.len + 15) & ~uintptr_t(15);
        const uint32_t bytes = static_cast<uint32_t>(hi - lo);
        mbar_arrive_expect_tx(bar, bytes);
        bulk_load(stage, reinterpret_cast<const void*>(lo), bytes, bar);
    }
}

__device__ __forceinline__ void tc_write(const TcPiece& pc, const uint8_t* stage, uint32_t lane) {
    const uint32_t sbase = smem_u32(stage);
    const uint32_t sh = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(pc.src) & 15u);
    uint32_t head = (16u - static_cast<uint32_t>(reinterpret_cast<uintptr_t>(pc.dst) & 15u)) & 15u;
    if (head > pc.len) head = pc.len;
    if (lane < head) pc.dst[lane] = lds_u8(sbase + sh + lane);
    const uint32_t o = sh + head;  // stage offset of the first aligned destination chunk
    const uint32_t nvec = (pc.len - head) >> 4;
    const uint32_t s2 = o & 15u;
    const uint32_t q0 = sbase + (o & ~15u);
    uint4* d4 = reinterpret_cast<uint4*>(pc.dst + head);
    if (s2 == 0) {
        for (uint32_t c = lane; c < nvec; c += 32) st_v4(d4 + c, lds_v4(q0 + 16 * c));
    } else {
        for (uint32_t c = lane; c < nvec; c += 32) st_v4(d4 + c, shift_merge(lds_v4(q0 + 16 * c), lds_v4(q0 + 16 * c + 16), s2));
    }
    const uint32_t done = head + (nvec << 4);
    if (lane < pc.len - done) pc.dst[done + lane] = lds_u8(sbase + sh + done + lane);
}

template <typename IdxT>
__global__ void __launch_bounds__(kTcThreads)
    k_csr_copy_tma(ArenaDev a, uint32_t vs, const RowRef* __restrict__ refs, const RowJob* __restrict__ jobs,
                   const uint64_t* __restrict__ P, uint64_t n_rows, uint32_t w_idx, uint8_t* __restrict__ out_idx,
                   uint8_t* __restrict__ out_val, uint64_t* __restrict__ out_gidx, uint64_t cr) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t s_bar[kTcWarps][2];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint32_t gw = blockIdx.x * kTcWarps + warp;
    const uint32_t n_warps = gridDim.x * kTcWarps;
    uint8_t* st0 = smem + warp * 2 * kTcStage;
    uint8_t* st1 = st0 + kTcStage;
    uint64_t* b0 = &s_bar[warp][0];
    uint64_t* b1 = &s_bar[warp][1];
    if (lane == 0) {
        mbar_init(b0, 1);
        mbar_init(b1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    pdl_wait();
    pdl_trigger();
    if (out_gidx && !jobs)
        for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kTcThreads + threadIdx.x; i < n_rows;
             i += static_cast<uint64_t>(gridDim.x) * kTcThreads)
            out_gidx[i] = refs[i].gidx;
    if (cr) {  // K5 mode: record headers + rebased indptr entries (encode_csr_record, store.cpp:52-64)
        constexpr uint64_t os = sizeof(IdxT);
        const uint64_t pb = P[0];
        for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kTcThreads + threadIdx.x; i < n_rows;
             i += static_cast<uint64_t>(gridDim.x) * kTcThreads) {
            const uint64_t q = i / cr, r0 = q * cr, rows_q = umin64(cr, n_rows - r0);
            const uint64_t p0q = P[r0];
            uint8_t* rec = out_idx + q * (kCsrHeaderBytes + os * (cr + 1)) + (os + vs) * (p0q - pb);
            uint8_t* ip = rec + kCsrHeaderBytes;
            if (i == r0) {
                st_any<uint32_t>(rec, static_cast<uint32_t>(rows_q));
                st_any<uint64_t>(rec + 4, P[r0 + rows_q] - p0q);
                st_any<IdxT>(ip, IdxT(0));
            }
            st_any<IdxT>(ip + os * (i - r0 + 1), static_cast<IdxT>(P[i + 1] - p0q));
        }
    }
    const bool is_val = gw >= w_idx;
    const uint32_t es = is_val ? vs : static_cast<uint32_t>(sizeof(IdxT));
    const uint32_t nw = is_val ? n_warps - w_idx : w_idx, w = is_val ? gw - w_idx : gw;
    const uint64_t p0 = P[0], total = P[n_rows] - p0;
    const uint64_t span = (((total * es + nw - 1) / nw) + 15) & ~15ull;
    const uint64_t e0 = w * span / es;
    if (e0 >= total) return;
    const uint64_t e1 = umin64(e0 + span / es, total);
    uint64_t lo = 0, hi = n_rows;
    while (hi - lo > 32) {
        const uint64_t step = (hi - lo + 31) / 32;
        const uint64_t k = lo + lane * step;
        const bool ok = k < hi && P[k] - p0 <= e0;
        const uint32_t c = __popc(__ballot_sync(kFull, ok));
        lo += (c - 1) * step;
        hi = umin64(lo + step, hi);
    }
    {
        const uint64_t k = lo + lane;
        const bool ok = k < hi && P[k] - p0 <= e0;
        lo += __popc(__ballot_sync(kFull, ok)) - 1;
    }
    TcGen<IdxT> gen;
    gen.a = a;
    gen.refs = refs;
    gen.jobs = jobs;
    gen.P = P;
    gen.n_rows = n_rows;
    gen.p0 = p0;
    gen.e0 = e0;
    gen.e1 = e1;
    gen.r = lo;
    gen.out = is_val ? out_val : out_idx;
    gen.cr = cr;
    gen.es = es;
    gen.vs = vs;
    gen.lane = lane;
    gen.is_val = is_val;
    gen.load_batch();
    TcPiece p_0 = gen.next();
    tc_issue(p_0, st0, b0, lane);
    TcPiece p_1 = gen.next();
    tc_issue(p_1, st1, b1, lane);
    uint32_t ph0 = 0, ph1 = 0;
    for (;;) {
        if (!p_0.len) break;
        mbar_wait(b0, ph0);
        ph0 ^= 1u;
        tc_write(p_0, st0, lane);
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before the next async write
        p_0 = gen.next();
        tc_issue(p_0, st0, b0, lane);
        if (!p_1.len) break;
        mbar_wait(b1, ph1);
        ph1 ^= 1u;
        tc_write(p_1, st1, lane);
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        p_1 = gen.next();
        tc_issue(p_1, st1, b1, lane);
    }
}

// ====================================================== column reprojection ===
// remap_csr_row / scatter_dense_row (preshuffle.cpp:95-134): a member store's
// rows re-expressed on the collection's unified var axis (col_map[c] = unified
// column of member column c, or ~0 when an inner join dropped it).
//
// CSR is sort-free: per row (one CTA) the mapped columns are set in a
// shared-memory bitmap over the unified axis; a block scan of the words'
// popcounts then gives every surviving entry its output slot (= its rank among
// the row's mapped columns), which is exactly the order std::sort of (u, k)
// produces when the u are distinct.  Two member columns mapping to the same
// unified column (duplicate var names) are detected (atomicOr saw the bit) and
// reported; the reference then fails in StoreWriter::append -> validate.
constexpr int kRemapThreads = 256;

// a.n_var = the member's n_var (out-of-range indices of a corrupt record map nowhere)
__device__ __forceinline__ uint32_t map_col(const uint32_t* __restrict__ colmap, uint64_t c, uint64_t in_nv) {
    return c < in_nv ? __ldg(colmap + c) : ~0u;
}

template <typename InIdx>
__global__ void __launch_bounds__(256)
    k_remap_count(ArenaDev a, uint32_t vs, const RowRef* __restrict__ refs, uint64_t n_rows,
                  const uint32_t* __restrict__ colmap, uint64_t* __restrict__ counts) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * (blockDim.x / 32);
    for (uint64_t row = static_cast<uint64_t>(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5); row < n_rows;
         row += nw) {
        const CsrRow src = csr_row<InIdx>(a, refs[row], vs);
        uint32_t c = 0;
        for (uint64_t k = lane; k < src.nnz; k += 32)
            c += map_col(colmap, ld_index<InIdx>(src.idx + k * sizeof(InIdx)), a.n_var) != ~0u;
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
        if (lane == 0) counts[row] = c;
    }
}

__device__ __forceinline__ void copy_value(uint8_t* dst, const uint8_t* src, uint32_t vs) {
    if (vs == 1) {
        *dst = __ldg(src);
    } else {  // 4-B aligned 4- or 8-byte values
        for (uint32_t b = 0; b < vs; b += 4)
            *reinterpret_cast<uint32_t*>(dst + b) = ld_u32(src + b);
    }
}

template <typename InIdx, typename OutIdx>
__global__ void __launch_bounds__(kRemapThreads)
    k_csr_remap(ArenaDev a, uint32_t vs, const RowRef* __restrict__ refs, uint64_t n_rows,
                const uint32_t* __restrict__ colmap, uint32_t n_words, const uint64_t* __restrict__ P,
                uint8_t* __restrict__ out, unsigned long long* __restrict__ dup_row, uint8_t* __restrict__ dup_flags) {
    extern __shared__ __align__(16) uint32_t s_bm[];  // [n_words] bitmap, [n_words] word prefix
    uint32_t* s_wp = s_bm + n_words;
    __shared__ uint32_t s_part[kRemapThreads / 32];
    constexpr uint64_t os = sizeof(OutIdx);
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint64_t pb = P[0], nnz_all = P[n_rows] - pb;
    uint8_t* ip = out + kCsrHeaderBytes;
    uint8_t* oidx = ip + os * (n_rows + 1);
    uint8_t* oval = oidx + os * nnz_all;
    if (blockIdx.x == 0 && tid == 0) {  // one record holding all rows (encode_csr_record layout)
        st_any<uint32_t>(out, static_cast<uint32_t>(n_rows));
        st_any<uint64_t>(out + 4, nnz_all);
        st_any<OutIdx>(ip, OutIdx(0));
    }
    const uint32_t wpt = (n_words + kRemapThreads - 1) / kRemapThreads;  // words per thread in the scan
    for (uint64_t row = blockIdx.x; row < n_rows; row += gridDim.x) {
        for (uint32_t w = tid; w < n_words; w += kRemapThreads) s_bm[w] = 0;
        __syncthreads();
        const CsrRow src = csr_row<InIdx>(a, refs[row], vs);
        bool dup = false;
        for (uint64_t k = tid; k < src.nnz; k += kRemapThreads) {
            const uint32_t u = map_col(colmap, ld_index<InIdx>(src.idx + k * sizeof(InIdx)), a.n_var);
            if (u != ~0u) {
                const uint32_t bit = 1u << (u & 31u);
                dup |= (atomicOr(&s_bm[u >> 5], bit) & bit) != 0;
            }
        }
        if (__syncthreads_or(dup) && tid == 0) {
            atomicMin(dup_row, static_cast<unsigned long long>(row));
            if (dup_flags) dup_flags[row] = 1;
        }
        // exclusive scan of the words' popcounts: thread t owns words [t*wpt, (t+1)*wpt)
        const uint32_t w0 = tid * wpt, w1 = min(n_words, w0 + wpt);
        uint32_t mine = 0;
        for (uint32_t w = w0; w < w1; ++w) mine += __popc(s_bm[w]);
        uint32_t incl = mine;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(kFull, incl, o);
            if (lane >= static_cast<uint32_t>(o)) incl += v;
        }
        if (lane == 31) s_part[warp] = incl;
        __syncthreads();
        uint32_t run = incl - mine;
        for (uint32_t w = 0; w < warp; ++w) run += s_part[w];
        for (uint32_t w = w0; w < w1; ++w) {
            s_wp[w] = run;
            run += __popc(s_bm[w]);
        }
        __syncthreads();
        const uint64_t base = P[row] - pb;
        for (uint64_t k = tid; k < src.nnz; k += kRemapThreads) {
            const uint32_t u = map_col(colmap, ld_index<InIdx>(src.idx + k * sizeof(InIdx)), a.n_var);
            if (u == ~0u) continue;
            const uint32_t pos = s_wp[u >> 5] + __popc(s_bm[u >> 5] & ((1u << (u & 31u)) - 1u));
            st_any<OutIdx>(oidx + os * (base + pos), static_cast<OutIdx>(u));
            copy_value(oval + vs * (base + pos), src.val + k * vs, vs);
        }
        if (tid == 0) st_any<OutIdx>(ip + os * (row + 1), static_cast<OutIdx>(P[row + 1] - pb));
        __syncthreads();  // bitmap is re-zeroed for the next row
    }
}

// Dense: out[row][u] = in[row][inv[u]] (inv[u] = last member column mapping to u,
// as the reference's in-order memcpy leaves it), zero where no column maps.
template <typename T>
__global__ void __launch_bounds__(256)
    k_dense_remap(ArenaDev a, uint64_t in_row_bytes, const RowRef* __restrict__ refs, uint64_t n_rows,
                  const uint32_t* __restrict__ inv, uint64_t out_nv, T* __restrict__ out) {
    for (uint64_t row = blockIdx.x; row < n_rows; row += gridDim.x) {
        const RowRef r = refs[row];
        const uint8_t* src = a.base + r.rec_off + (r.gidx % a.chunk_rows) * in_row_bytes;
        T* dst = out + row * out_nv;
        for (uint64_t u = threadIdx.x; u < out_nv; u += blockDim.x) {
            const uint32_t c = __ldg(inv + u);
            T v{};
            if (c != ~0u) {
                if constexpr (sizeof(T) == 1) v = __ldg(src + c);
                else if constexpr (sizeof(T) == 4) v = ld_u32(src + 4ull * c);
                else v = ld_u64_a4(src + 8ull * c);
            }
            dst[u] = v;
        }
    }
}

// ============================================================ CSR validation ===
// CsrBlock::validate (block.cpp:110-133) on device: every column index < n_var
// and strictly increasing within its row.  One CTA per record, one warp per
// row; the first violation (lowest global row) is kept with atomicMin and the
// host re-checks that record to report the reference's exact message.
template <typename IdxT>
__global__ void __launch_bounds__(256)
    k_validate_csr(const uint8_t* __restrict__ base, const uint64_t* __restrict__ rec_off,
                   const uint64_t* __restrict__ first_row, uint64_t n_recs, uint64_t n_var,
                   unsigned long long* __restrict__ bad_row) {
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    for (uint64_t q = blockIdx.x; q < n_recs; q += gridDim.x) {
        const uint8_t* rec = base + rec_off[q];
        const uint32_t rows = ld_u32(rec);
        const uint64_t nnz = ld_u64_a4(rec + 4);
        const uint8_t* ip = rec + kCsrHeaderBytes;
        const uint8_t* idx = ip + (static_cast<uint64_t>(rows) + 1) * sizeof(IdxT);
        for (uint32_t r = warp; r < rows; r += blockDim.x / 32) {
            const uint64_t lo = ld_index<IdxT>(ip + r * sizeof(IdxT)), hi = ld_index<IdxT>(ip + (r + 1) * sizeof(IdxT));
            bool bad = hi < lo || hi > nnz;
            if (!bad) {
                for (uint64_t k = lo + lane; k < hi; k += 32) {
                    const uint64_t c = ld_index<IdxT>(idx + k * sizeof(IdxT));
                    if (c >= n_var || (k > lo && c <= ld_index<IdxT>(idx + (k - 1) * sizeof(IdxT)))) bad = true;
                }
            }
            if (__any_sync(kFull, bad) && lane == 0) atomicMin(bad_row, static_cast<unsigned long long>(first_row[q] + r));
        }
    }
}

// ============================================================ K4 dense gather ===
constexpr int kDenseGatherThreads = 256;
enum DenseMode { kRaw = 0, kU8ToBf16 = 1, kF32ToBf16 = 2 };

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    const __nv_bfloat162 p = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&p);
}

template <int MODE>
__global__ void __launch_bounds__(kDenseGatherThreads)
    k_dense_gather(ArenaDev a, uint64_t in_row_bytes, const RowRef* __restrict__ refs, uint64_t n_rows,
                   uint8_t* __restrict__ out, uint64_t out_row_bytes, uint64_t* __restrict__ out_gidx) {
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5, nthr = blockDim.x;
    for (uint64_t row = blockIdx.x; row < n_rows; row += gridDim.x) {
        const RowRef r = refs[row];
        const uint8_t* src = a.base + r.rec_off + (r.gidx % a.chunk_rows) * in_row_bytes;
        uint8_t* dst = out + row * out_row_bytes;
        if (tid == 0 && out_gidx) out_gidx[row] = r.gidx;
        if (MODE == kRaw) {
            // split the row across warps on 16-B destination boundaries
            const uint32_t nw = nthr / 32;
            const uint64_t part = ((in_row_bytes + nw - 1) / nw + 15) & ~15ull;
            const uint64_t s = warp * part;
            if (s < in_row_bytes) warp_copy(dst + s, src + s, umin64(part, in_row_bytes - s), lane);
        } else if (MODE == kU8ToBf16) {
            const bool vec = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15u) == 0;
            const uint64_t nvec = vec ? in_row_bytes / 16 : 0;
            for (uint64_t i = tid; i < nvec; i += nthr) {
                const uint4 v = ld_v4(src + i * 16);
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
                uint32_t o[8];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    o[2 * j] = pack_bf16x2(float(w[j] & 0xff), float((w[j] >> 8) & 0xff));
                    o[2 * j + 1] = pack_bf16x2(float((w[j] >> 16) & 0xff), float(w[j] >> 24));
                }
                st_v4(dst + i * 32, make_uint4(o[0], o[1], o[2], o[3]));
                st_v4(dst + i * 32 + 16, make_uint4(o[4], o[5], o[6], o[7]));
            }
            __nv_bfloat16* d = reinterpret_cast<__nv_bfloat16*>(dst);
            for (uint64_t i = nvec * 16 + tid; i < in_row_bytes; i += nthr) d[i] = __float2bfloat16_rn(float(src[i]));
        } else {  // f32 -> bf16 (records are 4-B aligned)
            const uint64_t n = in_row_bytes / 4;
            const bool vec = ((reinterpret_cast<uintptr_t>(src) & 15u) | (reinterpret_cast<uintptr_t>(dst) & 7u)) == 0;
            const uint64_t nvec = vec ? n / 4 : 0;
            for (uint64_t i = tid; i < nvec; i += nthr) {
                const uint4 v = ld_v4(src + i * 16);
                uint2 o;
                o.x = pack_bf16x2(__uint_as_float(v.x), __uint_as_float(v.y));
                o.y = pack_bf16x2(__uint_as_float(v.z), __uint_as_float(v.w));
                *reinterpret_cast<uint2*>(dst + i * 8) = o;
            }
            __nv_bfloat16* d = reinterpret_cast<__nv_bfloat16*>(dst);
            for (uint64_t i = nvec * 4 + tid; i < n; i += nthr) d[i] = __float2bfloat16_rn(ld_value<float>(src + i * 4));
        }
    }
}

// Flat variant for 16-B aligned rows: work unit = (row, span of 32*U 16-B
// chunks); one lane reads the row's RowRef, every lane issues U independent
// 16-B loads before any store, so a warp keeps 32*U*16 B in flight and all
// rows of a (small) batch are in flight at once.

template <int MODE, int kDgU = 4, int kDgThreads = 256>
__global__ void __launch_bounds__(kDgThreads)
    k_dense_gather_flat(ArenaDev a, uint64_t in_row_bytes, const RowRef* __restrict__ refs, uint64_t n_rows,
                        uint8_t* __restrict__ out, uint64_t out_row_bytes, uint64_t* __restrict__ out_gidx) {
    pdl_wait();
    pdl_trigger();
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t cpr = in_row_bytes / 16;                    // 16-B chunks per input row
    const uint64_t upr = (cpr + 32 * kDgU - 1) / (32 * kDgU);  // units per row
    const uint64_t n_units = n_rows * upr;
    const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (kDgThreads / 32);
    for (uint64_t u = static_cast<uint64_t>(blockIdx.x) * (kDgThreads / 32) + (threadIdx.x >> 5); u < n_units;
         u += warps) {
        const uint64_t row = u / upr, part = u - row * upr;
        uint64_t off = 0, g = 0;
        if (lane == 0) {
            const RowRef r = refs[row];
            off = r.rec_off + (r.gidx % a.chunk_rows) * in_row_bytes;
            g = r.gidx;
        }
        off = __shfl_sync(kFull, off, 0);
        if (part == 0 && lane == 0 && out_gidx) out_gidx[row] = g;
        const uint4* src = reinterpret_cast<const uint4*>(a.base + off);
        const uint64_t c0 = part * 32 * kDgU + lane;
        uint4 v[kDgU];
#pragma unroll
        for (int k = 0; k < kDgU; ++k)
            if (c0 + k * 32 < cpr) v[k] = ld_v4(src + c0 + k * 32);
        uint8_t* dst = out + row * out_row_bytes;
#pragma unroll
        for (int k = 0; k < kDgU; ++k) {
            const uint64_t c = c0 + k * 32;
            if (c >= cpr) break;
            if (MODE == kRaw) {
                st_v4(dst + c * 16, v[k]);
            } else if (MODE == kU8ToBf16) {
                const uint32_t w[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
                uint32_t o[8];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    o[2 * j] = pack_bf16x2(float(w[j] & 0xff), float((w[j] >> 8) & 0xff));
                    o[2 * j + 1] = pack_bf16x2(float((w[j] >> 16) & 0xff), float(w[j] >> 24));
                }
                st_v4(dst + c * 32, make_uint4(o[0], o[1], o[2], o[3]));
                st_v4(dst + c * 32 + 16, make_uint4(o[4], o[5], o[6], o[7]));
            } else {  // f32 -> bf16
                uint2 o;
                o.x = pack_bf16x2(__uint_as_float(v[k].x), __uint_as_float(v[k].y));
                o.y = pack_bf16x2(__uint_as_float(v[k].z), __uint_as_float(v[k].w));
                *reinterpret_cast<uint2*>(dst + c * 8) = o;
            }
        }
    }
}

// Same work units, but each warp converts its unit into a shared-memory slice
// and one lane writes it with a 1-D TMA bulk store (the store path that wins
// for densify's write-heavy mix, profiles/r1_densify_v9.md).  A/B: RFL_DG=b.
template <int MODE, int kDgU = 2, int kDgThreads = 256>
__global__ void __launch_bounds__(kDgThreads)
    k_dense_gather_bulk(ArenaDev a, uint64_t in_row_bytes, const RowRef* __restrict__ refs, uint64_t n_rows,
                        uint8_t* __restrict__ out, uint64_t out_row_bytes, uint64_t* __restrict__ out_gidx) {
    constexpr uint32_t kOutPerIn = MODE == kU8ToBf16 ? 2 : 1;  // (f32 -> bf16 halves; not used here)
    constexpr uint32_t kSlice = 32 * kDgU * 16 * kOutPerIn;
    __shared__ __align__(128) uint8_t s_out[(kDgThreads / 32) * kSlice];
    pdl_wait();
    pdl_trigger();
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    uint8_t* slice = s_out + warp * kSlice;
    const uint64_t cpr = in_row_bytes / 16;
    const uint64_t upr = (cpr + 32 * kDgU - 1) / (32 * kDgU);
    const uint64_t n_units = n_rows * upr;
    const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (kDgThreads / 32);
    for (uint64_t u = static_cast<uint64_t>(blockIdx.x) * (kDgThreads / 32) + warp; u < n_units; u += warps) {
        const uint64_t row = u / upr, part = u - row * upr;
        uint64_t off = 0, g = 0;
        if (lane == 0) {
            const RowRef r = refs[row];
            off = r.rec_off + (r.gidx % a.chunk_rows) * in_row_bytes;
            g = r.gidx;
        }
        off = __shfl_sync(kFull, off, 0);
        if (part == 0 && lane == 0 && out_gidx) out_gidx[row] = g;
        const uint4* src = reinterpret_cast<const uint4*>(a.base + off);
        const uint64_t cbase = part * 32 * kDgU;
        const uint64_t nvec = umin64(32 * kDgU, cpr - cbase);  // 16-B input chunks of this unit
        uint4 v[kDgU];
#pragma unroll
        for (int k = 0; k < kDgU; ++k)
            if (k * 32 + lane < nvec) v[k] = ld_v4(src + cbase + k * 32 + lane);
        if (lane == 0) bulk_wait_read0();  // the slice's previous bulk store has read it
        __syncwarp();
#pragma unroll
        for (int k = 0; k < kDgU; ++k) {
            const uint32_t c = k * 32 + lane;
            if (c >= nvec) break;
            if (MODE == kRaw) {
                *reinterpret_cast<uint4*>(slice + c * 16) = v[k];
            } else {
                const uint32_t w[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
                uint32_t o[8];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    o[2 * j] = pack_bf16x2(float(w[j] & 0xff), float((w[j] >> 8) & 0xff));
                    o[2 * j + 1] = pack_bf16x2(float((w[j] >> 16) & 0xff), float(w[j] >> 24));
                }
                *reinterpret_cast<uint4*>(slice + c * 32) = make_uint4(o[0], o[1], o[2], o[3]);
                *reinterpret_cast<uint4*>(slice + c * 32 + 16) = make_uint4(o[4], o[5], o[6], o[7]);
            }
        }
        fence_proxy_async_shared();
        __syncwarp();
        if (lane == 0) {
            bulk_store(out + row * out_row_bytes + cbase * 16 * kOutPerIn, slice,
                       static_cast<uint32_t>(nvec * 16 * kOutPerIn));
            bulk_commit();
        }
    }
    if (lane == 0) bulk_wait0();
}


// K4o: dense rows straight from one-hot staged records (kOneHot4: 2-bit channel
// codes, L/4 bytes per row, L = n_var / 4 positions) -- no k_d8_decode expansion.
// Work unit = (row, 32 x kOhU code words) per warp; a code word covers 16
// positions, and the lane writes those 16 positions of all 4 channel planes
// (u8: 4 x 16 B, bf16: 4 x 32 B, f32: 4 x 64 B), so each plane's stores are
// contiguous across the warp.  Reads 1/16 of what it writes (u8).
enum OneHotOut { kOhU8 = 0, kOhBf16 = 1, kOhF32 = 2 };
__device__ __forceinline__ uint32_t onehot_mask16(uint32_t w, uint32_t c) {
    const uint32_t x = w ^ (c * 0x55555555u);  // a pair is 00 where the code equals c
    uint32_t m = ~(x | (x >> 1)) & 0x55555555u;
    m = (m | (m >> 1)) & 0x33333333u;
    m = (m | (m >> 2)) & 0x0F0F0F0Fu;
    m = (m | (m >> 4)) & 0x00FF00FFu;
    return (m | (m >> 8)) & 0x0000FFFFu;  // bit k = position k of the word is in plane c
}
template <int OUT, int kOhU = 2, int kOhThreads = 256>
__global__ void __launch_bounds__(kOhThreads)
    k_onehot_gather(ArenaDev a, const RowRef* __restrict__ refs, uint64_t n_rows, uint8_t* __restrict__ out,
                    uint64_t* __restrict__ out_gidx) {
    pdl_wait();
    pdl_trigger();
    constexpr uint32_t kEs = OUT == kOhU8 ? 1 : OUT == kOhBf16 ? 2 : 4;  // output element bytes
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t L = a.n_var / 4, wpr = L / 16;  // code words per row
    const uint64_t upr = (wpr + 32 * kOhU - 1) / (32 * kOhU);
    const uint64_t n_units = n_rows * upr;
    const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (kOhThreads / 32);
    for (uint64_t u = static_cast<uint64_t>(blockIdx.x) * (kOhThreads / 32) + (threadIdx.x >> 5); u < n_units;
         u += warps) {
        const uint64_t row = u / upr, part = u - row * upr;
        uint64_t off = 0, g = 0;
        if (lane == 0) {
            const RowRef r = refs[row];
            off = (r.rec_off & ((1ull << 60) - 1)) + (r.gidx % a.chunk_rows) * (L / 4);
            g = r.gidx;
        }
        off = __shfl_sync(kFull, off, 0);
        if (part == 0 && lane == 0 && out_gidx) out_gidx[row] = g;
        const uint64_t w0 = part * 32 * kOhU + lane;
        uint32_t w[kOhU];
#pragma unroll
        for (int k = 0; k < kOhU; ++k)
            if (w0 + k * 32 < wpr) w[k] = ld_u32(a.base + off + 4 * (w0 + k * 32));
        uint8_t* dst = out + row * a.n_var * kEs;
#pragma unroll
        for (int k = 0; k < kOhU; ++k) {
            const uint64_t wi = w0 + k * 32;
            if (wi >= wpr) break;
#pragma unroll
            for (uint32_t c = 0; c < 4; ++c) {
                const uint32_t m = onehot_mask16(w[k], c);
                uint8_t* p = dst + (c * L + 16 * wi) * kEs;
                if (OUT == kOhU8) {
                    uint32_t o[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) o[q] = (((m >> (4 * q)) & 0xFu) * 0x00204081u) & 0x01010101u;
                    st_v4(p, make_uint4(o[0], o[1], o[2], o[3]));
                } else if (OUT == kOhBf16) {
                    uint32_t o[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        o[q] = ((m >> (2 * q)) & 1u) * 0x3F80u | ((m >> (2 * q + 1)) & 1u) * 0x3F800000u;
                    st_v4(p, make_uint4(o[0], o[1], o[2], o[3]));
                    st_v4(p + 16, make_uint4(o[4], o[5], o[6], o[7]));
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        st_v4(p + 16 * q, make_uint4(((m >> (4 * q)) & 1u) * 0x3F800000u,
                                                     ((m >> (4 * q + 1)) & 1u) * 0x3F800000u,
                                                     ((m >> (4 * q + 2)) & 1u) * 0x3F800000u,
                                                     ((m >> (4 * q + 3)) & 1u) * 0x3F800000u));
                }
            }
        }
    }
}



// K4 by whole rows through TMA (the grouped launches; RFL_DG=row forces it): each CTA streams rows through
// 2 shared stages -- one 1-D bulk load of the row (mbarrier completion), the
// block converts it (u8 -> bf16) into the stage's out buffer (raw: in place), one
// bulk store of the row -- so both directions move as one large bulk op per row.
template <int MODE>
__global__ void __launch_bounds__(256)
    k_dense_gather_rows(ArenaDev a, uint64_t in_row_bytes, const RowRef* __restrict__ refs, uint64_t n_rows,
                        uint8_t* __restrict__ out, uint64_t out_row_bytes, uint64_t* __restrict__ out_gidx,
                        uint32_t stage_bytes) {
    extern __shared__ __align__(128) uint8_t dr_smem[];
    __shared__ __align__(8) uint64_t bar[2];
    const uint32_t in_b = static_cast<uint32_t>(in_row_bytes);
    const uint32_t in_pad = (in_b + 127u) & ~127u;
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    pdl_wait();
    pdl_trigger();
    auto issue = [&](uint64_t r, uint32_t st) {  // thread 0
        const RowRef rf = refs[r];
        if (out_gidx) out_gidx[r] = rf.gidx;
        mbar_arrive_expect_tx(&bar[st], in_b);
        bulk_load(dr_smem + st * stage_bytes, a.base + rf.rec_off + (rf.gidx % a.chunk_rows) * in_row_bytes, in_b,
                  &bar[st]);
    };
    const uint64_t stride = gridDim.x;
    uint64_t r = blockIdx.x;
    if (threadIdx.x == 0) {
        if (r < n_rows) issue(r, 0);
        if (r + stride < n_rows) issue(r + stride, 1);
    }
    uint32_t ph[2] = {0, 0};
    for (uint32_t it = 0; r < n_rows; r += stride, ++it) {
        const uint32_t st = it & 1u;
        uint8_t* in = dr_smem + st * stage_bytes;
        uint8_t* ob = MODE == kRaw ? in : in + in_pad;
        mbar_wait(&bar[st], ph[st]);
        ph[st] ^= 1u;
        if (MODE != kRaw) {
            if (threadIdx.x == 0) bulk_wait_read1();  // this stage's out buffer (two rows ago) has been read
            __syncthreads();
            for (uint32_t c = threadIdx.x; c < in_b / 16; c += 256) {
                const uint4 v = *reinterpret_cast<const uint4*>(in + c * 16);
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
                uint32_t o[8];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    o[2 * j] = pack_bf16x2(float(w[j] & 0xff), float((w[j] >> 8) & 0xff));
                    o[2 * j + 1] = pack_bf16x2(float((w[j] >> 16) & 0xff), float(w[j] >> 24));
                }
                *reinterpret_cast<uint4*>(ob + c * 32) = make_uint4(o[0], o[1], o[2], o[3]);
                *reinterpret_cast<uint4*>(ob + c * 32 + 16) = make_uint4(o[4], o[5], o[6], o[7]);
            }
            fence_proxy_async_shared();
        }
        __syncthreads();  // (raw: every thread is past the wait; converted: the out buffer is complete)
        if (threadIdx.x == 0) {
            bulk_store(out + r * out_row_bytes, ob, static_cast<uint32_t>(out_row_bytes));
            bulk_commit();
            if (r + 2 * stride < n_rows) {
                // raw: the stage is reloaded only once its store has read it; converted: the
                // in buffer was consumed by the conversion above
                if (MODE == kRaw) bulk_wait_read0();
                issue(r + 2 * stride, st);
            }
        }
    }
    if (threadIdx.x == 0) bulk_wait0();
}

// K4o by whole rows (default; RFL_OH=plain for the register-store kernel): a 64-thread CTA streams output rows through
// two shared stages; the next row's code words are loaded into registers before
// the current row is built, and each row leaves with one 1-D bulk store.
template <int OUT>
__global__ void __launch_bounds__(64)
    k_onehot_gather_rows(ArenaDev a, const RowRef* __restrict__ refs, uint64_t n_rows, uint8_t* __restrict__ out,
                         uint64_t* __restrict__ out_gidx) {
    constexpr uint32_t kEs = OUT == kOhU8 ? 1 : 2;
    constexpr uint32_t kMaxW = 8;  // code words per thread (rows up to 64 x 8 x 64 = 32,768 positions)
    extern __shared__ __align__(128) uint8_t ohr_smem[];
    pdl_wait();
    pdl_trigger();
    const uint64_t L = a.n_var / 4, wpr = L / 16;
    const uint64_t row_bytes = a.n_var * kEs;
    const uint32_t tid = threadIdx.x;
    auto load = [&](uint64_t r, uint32_t (&w)[kMaxW]) {
        const RowRef rf = refs[r];  // (every thread: one broadcast L1 line)
        const uint8_t* src = a.base + (rf.rec_off & ((1ull << 60) - 1)) + (rf.gidx % a.chunk_rows) * (L / 4);
#pragma unroll
        for (uint32_t k = 0; k < kMaxW; ++k)
            if (tid + 64 * k < wpr) w[k] = ld_u32(src + 4 * (tid + 64 * k));
        if (tid == 0 && out_gidx) out_gidx[r] = rf.gidx;
    };
    uint32_t cur[kMaxW], nxt[kMaxW];
    uint64_t r = blockIdx.x;
    if (r < n_rows) load(r, cur);
    for (uint32_t it = 0; r < n_rows; r += gridDim.x, ++it) {
        if (r + gridDim.x < n_rows) load(r + gridDim.x, nxt);
        uint8_t* stage = ohr_smem + (it & 1u) * row_bytes;
        if (tid == 0) bulk_wait_read1();  // this stage's store (two rows ago) has been read
        __syncthreads();
#pragma unroll
        for (uint32_t k = 0; k < kMaxW; ++k) {
            const uint64_t wi = tid + 64 * k;
            if (wi >= wpr) break;
#pragma unroll
            for (uint32_t c = 0; c < 4; ++c) {
                const uint32_t m = onehot_mask16(cur[k], c);
                uint8_t* p = stage + (c * L + 16 * wi) * kEs;
                if (OUT == kOhU8) {
                    uint32_t o[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) o[q] = (((m >> (4 * q)) & 0xFu) * 0x00204081u) & 0x01010101u;
                    *reinterpret_cast<uint4*>(p) = make_uint4(o[0], o[1], o[2], o[3]);
                } else {
                    uint32_t o[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        o[q] = ((m >> (2 * q)) & 1u) * 0x3F80u | ((m >> (2 * q + 1)) & 1u) * 0x3F800000u;
                    *reinterpret_cast<uint4*>(p) = make_uint4(o[0], o[1], o[2], o[3]);
                    *reinterpret_cast<uint4*>(p + 16) = make_uint4(o[4], o[5], o[6], o[7]);
                }
            }
        }
        fence_proxy_async_shared();
        __syncthreads();
        if (tid == 0) {
            bulk_store(out + r * row_bytes, stage, static_cast<uint32_t>(row_bytes));
            bulk_commit();
        }
#pragma unroll
        for (uint32_t k = 0; k < kMaxW; ++k) cur[k] = nxt[k];
    }
    if (tid == 0) bulk_wait0();
}


// ======================================================== staging pull ===
// Host -> HBM staging of a group's fetched blocks by TMA instead of one copy-engine
// transfer per block: each copy engine transfer pays a fixed ~4.7 us setup
// (37 GB/s for cfg1's ~0.5 MB blocks, profiles/r2/s3/pcie_staging.md), while 1-D
// bulk loads of the mapped pinned image into shared stages + bulk stores to the
// slots keep ~2 MB in flight across a small grid (51 GB/s, any block size).
// One thread per CTA; the CTAs take the (job, piece) pairs round-robin.
__global__ void __launch_bounds__(32) k_stage_pull(const __grid_constant__ PullJobs jobs, uint32_t P, uint32_t S) {
    extern __shared__ __align__(128) uint8_t pull_smem[];
    __shared__ __align__(8) uint64_t bar[kMaxPullStages];
    pdl_wait();
    if (threadIdx.x != 0) return;
    const uint32_t total = jobs.first_piece[jobs.n];
    for (uint32_t s = 0; s < S; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // global piece g -> (job, byte offset): binary search of the per-job piece prefix
    auto locate = [&](uint32_t g, uint32_t& bytes) -> uint64_t {
        uint32_t lo = 0, hi = jobs.n;  // first_piece[lo] <= g < first_piece[hi]
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (jobs.first_piece[mid] <= g) lo = mid;
            else hi = mid;
        }
        const uint64_t off = static_cast<uint64_t>(g - jobs.first_piece[lo]) * P;
        const uint64_t left = jobs.job[lo].bytes - off;
        bytes = static_cast<uint32_t>(left < P ? left : P);
        return (static_cast<uint64_t>(lo) << 40) | off;
    };
    uint32_t phases = 0, issue = blockIdx.x, done = blockIdx.x, si = 0, sd = 0;
    auto load = [&](uint32_t g, uint32_t slot) {
        uint32_t bytes;
        const uint64_t jo = locate(g, bytes);
        const PullJob& jb = jobs.job[jo >> 40];
        mbar_arrive_expect_tx(&bar[slot], bytes);
        bulk_load(pull_smem + slot * P, jb.src + (jo & ((1ull << 40) - 1)), bytes, &bar[slot]);
    };
    for (uint32_t k = 0; k < S && issue < total; ++k, issue += gridDim.x, si = si + 1 == S ? 0 : si + 1)
        load(issue, si);
    for (; done < total; done += gridDim.x) {
        mbar_wait(&bar[sd], (phases >> sd) & 1u);
        phases ^= 1u << sd;
        uint32_t bytes;
        const uint64_t jo = locate(done, bytes);
        bulk_store(jobs.job[jo >> 40].dst + (jo & ((1ull << 40) - 1)), pull_smem + sd * P, bytes);
        bulk_commit();
        bulk_wait_read0();  // the stage is free again
        if (issue < total) {
            load(issue, sd);
            issue += gridDim.x;
        }
        sd = sd + 1 == S ? 0 : sd + 1;
    }
    bulk_wait0();
}

// ------------------------------------------------------------ host helpers ---

bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("RFL_PDL");  // default on; RFL_PDL=0 for plain launches
        return !(e && e[0] == '0');
    }();
    return on;
}

// <<<>>> with the programmatic-stream-serialization attribute when PDL is on
// (inside stream capture this becomes a programmatic graph edge).
template <typename... KArgs, typename... Args>
void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, const char* what,
              Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    cuda_check(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...), what);
}

template <typename K>
void set_smem(K kernel, size_t bytes) {
    cuda_check(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)),
               "cudaFuncSetAttribute");
}

// Densify shape override for A/B runs: RFL_DENSIFY="v<6|9>:<threads>:<tile KB>:<U>:<CTAs/SM>"
// (instantiated shapes: 256:*:16:2, 256:*:8:3, 256:*:8:4; other values fall back to 256:*:8:3).
struct DensifyCfg {  // version 0 = the measured default (shape rule in densify_t)
    int version = 0, threads = 256, tile_kb = 40, u = 8, minb = 3, nbuf = 1;
};
const DensifyCfg& densify_cfg() {
    static const DensifyCfg c = [] {
        DensifyCfg d;
        const char* e = std::getenv("RFL_DENSIFY");
        int v = 0, t = 256, kb = 40, u = 8, mb = 3, nb = 1;
        if (e && std::sscanf(e, "v%d", &v) == 1 && (v == 6 || v == 9)) {
            const int got = std::sscanf(std::strchr(e, ':') ? std::strchr(e, ':') : e + 2, ":%d:%d:%d:%d:%d", &t, &kb,
                                        &u, &mb, &nb);
            d.version = v;
            if (got >= 1) d.threads = t;
            if (got >= 2 && kb >= 4 && kb <= 200) d.tile_kb = kb;
            if (got >= 3) d.u = u;
            if (got >= 4) d.minb = mb;
            if (got >= 5 && (nb == 1 || nb == 2)) d.nbuf = nb;
        }
        return d;
    }();
    return c;
}
// K3d shape override: RFL_DENSIFY_D8=<tile KB>:<CTAs/SM 2|3>:<tile buffers 1|2> (A/B)
struct D8Shape {
    int tile_kb = 0, minb = 0, nbuf = 0;  // 0 = the default shape rule
};
const D8Shape& d8_shape() {
    static const D8Shape c = [] {
        D8Shape d;
        const char* e = std::getenv("RFL_DENSIFY_D8");
        int kb = 0, mb = 0, nb = 0;
        if (e && std::sscanf(e, "%d:%d:%d", &kb, &mb, &nb) == 3 && kb >= 4 && kb <= 200 && (mb == 2 || mb == 3) &&
            (nb == 1 || nb == 2)) {
            d.tile_kb = kb;
            d.minb = mb;
            d.nbuf = nb;
        }
        return d;
    }();
    return c;
}

template <typename IdxT, typename SrcT, typename DstT, int THREADS, int U, int MINB, int VAR = 6>
void densify_v6(const ArenaView& av, const RowRef* refs, uint64_t n, bool norm, float target, void* out,
                uint64_t* out_gidx, cudaStream_t st, uint64_t max_tile_bytes, int nbuf = 1) {
    const uint64_t esz = sizeof(DstT);
    uint64_t tile_cols = av.n_var;
    if (av.n_var * esz > max_tile_bytes) tile_cols = (max_tile_bytes / esz) & ~15ull;
    int bulk = ((av.n_var * esz) % 16 == 0) && (reinterpret_cast<uintptr_t>(out) % 16 == 0);
    if (bulk && VAR == 9 && nbuf == 2 && tile_cols < av.n_var) bulk = 2;  // two alternating tiles (v9 only)
    const size_t smem = ((tile_cols * esz + 127) & ~127ull) * (bulk == 2 ? 2 : 1);
    auto kern = [] {
        if constexpr (VAR == 9) return k_csr_densify9<IdxT, SrcT, DstT, THREADS, U, MINB>;
        else return k_csr_densify6<IdxT, SrcT, DstT, THREADS, U, MINB>;
    }();
    set_smem(kern, smem);
    int per_sm = 0;
    cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THREADS, smem), "occupancy");
    const uint64_t grid = std::min<uint64_t>(n, static_cast<uint64_t>(std::max(per_sm, 1)) * device_sm_count());
    launch_k(kern, dim3(static_cast<unsigned>(grid)), dim3(THREADS), smem, st, "k_csr_densify6 launch", dev_view(av),
             refs, n, static_cast<uint32_t>(tile_cols), norm ? 1 : 0, target, static_cast<DstT*>(out), out_gidx, bulk);
}

template <typename IdxT, typename SrcT, typename DstT>
void densify_t(const ArenaView& av, const RowRef* refs, uint64_t n, bool norm, float target, void* out,
               uint64_t* out_gidx, cudaStream_t st, uint64_t avg_nnz) {
    const DensifyCfg& dc = densify_cfg();
    if (dc.version == 0) {
        // Default (profiles/r1_densify_v9.md): v9 (lane-parallel row lookups, two rows
        // of entries in registers).  Dense rows wider than 48 KB: 16 entries per
        // thread, 80 KB tiles, 2 CTAs/SM (cfg1 f32 0.885, cfg2 norm+log1p 0.888 of
        // measured HBM); narrower rows (e.g. cfg1 -> bf16, 40 KB): 8 per thread,
        // 40 KB tiles, 3 CTAs/SM (0.81), so a row still fills its tile.
        (void)avg_nnz;
        const bool wide = av.n_var * sizeof(DstT) > 48 * 1024;
        if constexpr (sizeof(IdxT) <= 4) {
            if (wide) return densify_v6<IdxT, SrcT, DstT, 256, 16, 2, 9>(av, refs, n, norm, target, out, out_gidx, st, 80 << 10);
            return densify_v6<IdxT, SrcT, DstT, 256, 8, 3, 9>(av, refs, n, norm, target, out, out_gidx, st, 40 << 10);
        } else {  // u64 indices: the v6 register budget
            if (wide) return densify_v6<IdxT, SrcT, DstT, 256, 16, 2>(av, refs, n, norm, target, out, out_gidx, st, 80 << 10);
            return densify_v6<IdxT, SrcT, DstT, 256, 8, 3>(av, refs, n, norm, target, out, out_gidx, st, 40 << 10);
        }
    }
    const uint64_t tb = static_cast<uint64_t>(dc.tile_kb) * 1024;
    if constexpr (sizeof(IdxT) == 4 && sizeof(SrcT) == 4) {
        if (dc.version == 9) {
            const int nb = dc.nbuf;
            if (dc.u == 16) return densify_v6<IdxT, SrcT, DstT, 256, 16, 2, 9>(av, refs, n, norm, target, out, out_gidx, st, tb, nb);
            if (dc.minb == 4) return densify_v6<IdxT, SrcT, DstT, 256, 8, 4, 9>(av, refs, n, norm, target, out, out_gidx, st, tb, nb);
            return densify_v6<IdxT, SrcT, DstT, 256, 8, 3, 9>(av, refs, n, norm, target, out, out_gidx, st, tb, nb);
        }
    }
    if (dc.u == 16) return densify_v6<IdxT, SrcT, DstT, 256, 16, 2>(av, refs, n, norm, target, out, out_gidx, st, tb);
    if (dc.minb == 4) return densify_v6<IdxT, SrcT, DstT, 256, 8, 4>(av, refs, n, norm, target, out, out_gidx, st, tb);
    return densify_v6<IdxT, SrcT, DstT, 256, 8, 3>(av, refs, n, norm, target, out, out_gidx, st, tb);
}

template <typename IdxT>
void densify_idx(const ArenaView& a, const RowRef* refs, uint64_t n, OutDtype od, bool norm, float target, void* out,
                 uint64_t* g, cudaStream_t st, uint64_t avg_nnz) {
    switch (a.vdt) {
        case VDtype::f32:
            if (od == OutDtype::bf16) return densify_t<IdxT, float, __nv_bfloat16>(a, refs, n, norm, target, out, g, st, avg_nnz);
            return densify_t<IdxT, float, float>(a, refs, n, norm, target, out, g, st, avg_nnz);
        case VDtype::f64:
            if (od == OutDtype::bf16) return densify_t<IdxT, double, __nv_bfloat16>(a, refs, n, norm, target, out, g, st, avg_nnz);
            if (od == OutDtype::f32) return densify_t<IdxT, double, float>(a, refs, n, norm, target, out, g, st, avg_nnz);
            return densify_t<IdxT, double, double>(a, refs, n, false, target, out, g, st, avg_nnz);
        case VDtype::i32:
            if (od == OutDtype::bf16) return densify_t<IdxT, int32_t, __nv_bfloat16>(a, refs, n, norm, target, out, g, st, avg_nnz);
            if (od == OutDtype::f32) return densify_t<IdxT, int32_t, float>(a, refs, n, norm, target, out, g, st, avg_nnz);
            return densify_t<IdxT, int32_t, int32_t>(a, refs, n, false, target, out, g, st, avg_nnz);
        case VDtype::u8:
            if (od == OutDtype::bf16) return densify_t<IdxT, uint8_t, __nv_bfloat16>(a, refs, n, norm, target, out, g, st, avg_nnz);
            if (od == OutDtype::f32) return densify_t<IdxT, uint8_t, float>(a, refs, n, norm, target, out, g, st, avg_nnz);
            return densify_t<IdxT, uint8_t, uint8_t>(a, refs, n, false, target, out, g, st, avg_nnz);
    }
}

}  // namespace

int device_sm_count() {
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    static std::atomic<int> counts[64];  // (zero-initialised: static storage)
    if (dev < 64) {
        const int c = counts[dev].load(std::memory_order_relaxed);
        if (c) return c;
    }
    int c = 0;
    cuda_check(cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev), "sm count");
    if (dev < 64) counts[dev].store(c, std::memory_order_relaxed);
    return c;
}

namespace {
uint64_t scan_status_bytes(uint64_t n_rows) {
    const uint64_t tiles = (n_rows + kScanThreads - 1) / kScanThreads;
    return ((1 + tiles) * sizeof(unsigned long long) + 15) & ~15ull;
}
void launch_scan(const ArenaView& a, const RowRef* refs, uint64_t n, uint64_t* out_prefix, RowJob* jobs,
                 uint64_t* out_gidx, void* scratch, cudaStream_t st, const uint64_t* counts = nullptr) {
    cuda_check(cudaMemsetAsync(scratch, 0, scan_status_bytes(n), st), "memset scratch");
    const unsigned tiles = static_cast<unsigned>((n + kScanThreads - 1) / kScanThreads);
    const uint32_t vs = static_cast<uint32_t>(value_size(a.vdt));
    auto* sc = static_cast<unsigned long long*>(scratch);
    if (a.idt == IDtype::u32)
        k_row_scan<uint32_t><<<tiles, kScanThreads, 0, st>>>(dev_view(a), vs, refs, n, out_prefix, jobs, out_gidx, sc,
                                                             counts);
    else
        k_row_scan<uint64_t><<<tiles, kScanThreads, 0, st>>>(dev_view(a), vs, refs, n, out_prefix, jobs, out_gidx, sc,
                                                             counts);
    cuda_check(cudaGetLastError(), "k_row_scan launch");
}
}  // namespace

// K2 launcher: the balanced TMA-staged copy (k_csr_copy_tma), from the scan's job
// table (jobs != nullptr) or resolving rows itself; cr > 0 = K5 record mode.
void launch_copy_tma(const ArenaView& a, uint32_t vs, const RowRef* refs, const RowJob* jobs, const uint64_t* P,
                     uint64_t n, void* out_indices, void* out_data, uint64_t* out_gidx, cudaStream_t st,
                     uint64_t cr = 0) {
    auto kern = a.idt == IDtype::u32 ? k_csr_copy_tma<uint32_t> : k_csr_copy_tma<uint64_t>;
    const size_t smem = 2 * kTcStage * kTcWarps;
    static std::atomic<int> per_sm[2];
    int occ = per_sm[a.idt == IDtype::u32 ? 0 : 1].load(std::memory_order_relaxed);
    if (!occ) {
        set_smem(kern, smem);
        cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kTcThreads, smem), "occupancy");
        per_sm[a.idt == IDtype::u32 ? 0 : 1].store(occ, std::memory_order_relaxed);
    }
    const uint32_t blocks = static_cast<uint32_t>(std::max(occ, 1) * device_sm_count());
    const uint32_t n_warps = blocks * kTcWarps;
    const uint32_t is = static_cast<uint32_t>(index_size(a.idt));
    const uint32_t w_idx = std::max(1u, std::min(n_warps - 1, (n_warps * is + (is + vs) / 2) / (is + vs)));
    launch_k(kern, dim3(blocks), dim3(kTcThreads), smem, st, "k_csr_copy_tma launch", dev_view(a), vs, refs, jobs, P,
             n, w_idx, static_cast<uint8_t*>(out_indices), static_cast<uint8_t*>(out_data), out_gidx, cr);
}

size_t csr_gather_scratch_bytes(uint64_t n_rows) { return scan_status_bytes(n_rows) + n_rows * sizeof(RowJob); }

void launch_csr_gather(const ArenaView& a, const RowRef* refs, uint64_t n, uint64_t* out_indptr, void* out_indices,
                       void* out_data, uint64_t* out_gidx, void* scratch, cudaStream_t st) {
    if (a.layout != Layout::csr) invalid("csr_gather: store is not csr");
    if (a.idx16) invalid("csr_gather: narrowed staging needs the host-planned indptr (csr_gather_prefixed)");
    if (n == 0) {
        cuda_check(cudaMemsetAsync(out_indptr, 0, sizeof(uint64_t), st), "memset");
        return;
    }
    RowJob* jobs = reinterpret_cast<RowJob*>(static_cast<uint8_t*>(scratch) + scan_status_bytes(n));
    launch_scan(a, refs, n, out_indptr, jobs, out_gidx, scratch, st);
    launch_copy_tma(a, static_cast<uint32_t>(value_size(a.vdt)), refs, jobs, out_indptr, n, out_indices, out_data,
                    nullptr, st);
}

void launch_d8_decode(const D8Job* jobs, size_t n, uint32_t vs, uint64_t rows_per_record, cudaStream_t st,
                      uint64_t n_var, bool vfloat) {
    const unsigned split = static_cast<unsigned>(std::min<uint64_t>(std::max<uint64_t>(1, (rows_per_record + 7) / 8), 1024));
    for (size_t k0 = 0; k0 < n; k0 += kMaxD8Jobs) {
        D8Jobs j{};
        j.n = static_cast<uint32_t>(std::min<size_t>(kMaxD8Jobs, n - k0));
        j.vs = vs;
        j.n_var = n_var;
        j.vfloat = vfloat ? 1u : 0u;
        for (uint32_t i = 0; i < j.n; ++i) j.job[i] = jobs[k0 + i];
        launch_k(k_d8_decode, dim3(j.n, split), dim3(256), 0, st, "k_d8_decode launch", j);
    }
}

void launch_csr_gather_prefixed(const ArenaView& a, const RowRef* refs, uint64_t n, const uint64_t* prefix,
                                void* out_indices, void* out_data, uint64_t* out_gidx, cudaStream_t st) {
    if (a.layout != Layout::csr) invalid("csr_gather: store is not csr");
    if (n == 0) return;
    if (a.idx16) {
        const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 7) / 8, 16ull * device_sm_count()));
        launch_k(k_csr_gather_idx16, dim3(grid), dim3(256), 0, st, "k_csr_gather_idx16 launch", dev_view(a),
                 static_cast<uint32_t>(value_size(a.vdt)), refs, prefix, n, static_cast<uint32_t*>(out_indices),
                 static_cast<uint8_t*>(out_data), out_gidx);
        return;
    }
    launch_copy_tma(a, static_cast<uint32_t>(value_size(a.vdt)), refs, nullptr, prefix, n, out_indices, out_data,
                     out_gidx, st);
}

void launch_csr_row_scan(const ArenaView& a, const RowRef* refs, uint64_t n, uint64_t* out_prefix, void* scratch,
                         cudaStream_t st) {
    if (n == 0) {
        cuda_check(cudaMemsetAsync(out_prefix, 0, sizeof(uint64_t), st), "memset");
        return;
    }
    launch_scan(a, refs, n, out_prefix, nullptr, nullptr, scratch, st);
}

void launch_csr_pack(const ArenaView& a, const RowRef* refs, uint64_t n, uint64_t chunk_rows, IDtype out_idt,
                     const uint64_t* prefix, uint8_t* out, cudaStream_t st) {
    if (a.layout != Layout::csr) invalid("csr_pack: store is not csr");
    if (n == 0) return;
    const uint32_t vs = static_cast<uint32_t>(value_size(a.vdt));
    static const bool legacy = [] {
        const char* e = std::getenv("RFL_PACK");
        return e && std::string(e) == "warp";
    }();
    if (a.idt == out_idt && !legacy)  // byte-identical index width: the balanced TMA copy in record mode
        return launch_copy_tma(a, vs, refs, nullptr, prefix, n, out, out, nullptr, st, chunk_rows);
    const unsigned grid =
        static_cast<unsigned>(std::min<uint64_t>((n + kPackThreads / 32 - 1) / (kPackThreads / 32), 16ull * device_sm_count()));
    const ArenaDev d = dev_view(a);
    if (a.idt == IDtype::u32 && out_idt == IDtype::u32)
        k_csr_pack<uint32_t, uint32_t><<<grid, kPackThreads, 0, st>>>(d, vs, refs, n, chunk_rows, prefix, out);
    else if (a.idt == IDtype::u32)
        k_csr_pack<uint32_t, uint64_t><<<grid, kPackThreads, 0, st>>>(d, vs, refs, n, chunk_rows, prefix, out);
    else if (out_idt == IDtype::u32)
        k_csr_pack<uint64_t, uint32_t><<<grid, kPackThreads, 0, st>>>(d, vs, refs, n, chunk_rows, prefix, out);
    else
        k_csr_pack<uint64_t, uint64_t><<<grid, kPackThreads, 0, st>>>(d, vs, refs, n, chunk_rows, prefix, out);
    cuda_check(cudaGetLastError(), "k_csr_pack launch");
}

void launch_remap_count(const ArenaView& a, const RowRef* refs, uint64_t n, const uint32_t* colmap, uint64_t* counts,
                        cudaStream_t st) {
    if (n == 0) return;
    const uint32_t vs = static_cast<uint32_t>(value_size(a.vdt));
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 7) / 8, 16ull * device_sm_count()));
    if (a.idt == IDtype::u32)
        k_remap_count<uint32_t><<<grid, 256, 0, st>>>(dev_view(a), vs, refs, n, colmap, counts);
    else
        k_remap_count<uint64_t><<<grid, 256, 0, st>>>(dev_view(a), vs, refs, n, colmap, counts);
    cuda_check(cudaGetLastError(), "k_remap_count launch");
}

void launch_count_scan(const uint64_t* counts, uint64_t n, uint64_t* out_prefix, void* scratch, cudaStream_t st) {
    if (n == 0) {
        cuda_check(cudaMemsetAsync(out_prefix, 0, sizeof(uint64_t), st), "memset");
        return;
    }
    ArenaView none;
    launch_scan(none, nullptr, n, out_prefix, nullptr, nullptr, scratch, st, counts);
}

size_t csr_remap_smem_bytes(uint64_t out_nv) { return 2 * 4 * ((out_nv + 31) / 32); }

void launch_csr_remap(const ArenaView& a, const RowRef* refs, uint64_t n, const uint32_t* colmap, uint64_t out_nv,
                      IDtype out_idt, const uint64_t* prefix, uint8_t* out, unsigned long long* dup_row,
                      uint8_t* dup_flags, cudaStream_t st) {
    if (n == 0) return;
    const uint32_t vs = static_cast<uint32_t>(value_size(a.vdt));
    const uint32_t n_words = static_cast<uint32_t>((out_nv + 31) / 32);
    const size_t smem = csr_remap_smem_bytes(out_nv);
    if (smem > 200 * 1024) invalid("column reprojection: unified n_var too large for the device bitmap");
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(n, 8ull * device_sm_count()));
    const ArenaDev d = dev_view(a);
    auto go = [&](auto kern) {
        set_smem(kern, smem);
        kern<<<grid, kRemapThreads, smem, st>>>(d, vs, refs, n, colmap, n_words, prefix, out, dup_row, dup_flags);
    };
    if (a.idt == IDtype::u32 && out_idt == IDtype::u32) go(k_csr_remap<uint32_t, uint32_t>);
    else if (a.idt == IDtype::u32) go(k_csr_remap<uint32_t, uint64_t>);
    else if (out_idt == IDtype::u32) go(k_csr_remap<uint64_t, uint32_t>);
    else go(k_csr_remap<uint64_t, uint64_t>);
    cuda_check(cudaGetLastError(), "k_csr_remap launch");
}

void launch_dense_remap(const ArenaView& a, const RowRef* refs, uint64_t n, uint64_t in_nv, const uint32_t* inv,
                        uint64_t out_nv, void* out, cudaStream_t st) {
    if (n == 0) return;
    const uint64_t vs = value_size(a.vdt);
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(n, 8ull * device_sm_count()));
    const ArenaDev d = dev_view(a);
    if (vs == 1)
        k_dense_remap<uint8_t><<<grid, 256, 0, st>>>(d, in_nv, refs, n, inv, out_nv, static_cast<uint8_t*>(out));
    else if (vs == 4)
        k_dense_remap<uint32_t><<<grid, 256, 0, st>>>(d, 4 * in_nv, refs, n, inv, out_nv, static_cast<uint32_t*>(out));
    else
        k_dense_remap<uint64_t><<<grid, 256, 0, st>>>(d, 8 * in_nv, refs, n, inv, out_nv, static_cast<uint64_t*>(out));
    cuda_check(cudaGetLastError(), "k_dense_remap launch");
}

void launch_validate_csr(const uint8_t* base, const uint64_t* d_rec_off, const uint64_t* d_first_row, uint64_t n_recs,
                         uint64_t n_var, IDtype idt, unsigned long long* d_bad_row, cudaStream_t st) {
    if (n_recs == 0) return;
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(n_recs, 8ull * device_sm_count()));
    if (idt == IDtype::u32)
        k_validate_csr<uint32_t><<<grid, 256, 0, st>>>(base, d_rec_off, d_first_row, n_recs, n_var, d_bad_row);
    else
        k_validate_csr<uint64_t><<<grid, 256, 0, st>>>(base, d_rec_off, d_first_row, n_recs, n_var, d_bad_row);
    cuda_check(cudaGetLastError(), "k_validate_csr launch");
}

size_t dense_out_elem_size(const ArenaView& a, OutDtype od) {
    if (od == OutDtype::bf16) return 2;
    if (od == OutDtype::f32) return 4;
    return value_size(a.vdt);
}

void launch_csr_densify(const ArenaView& a, const RowRef* refs, uint64_t n, OutDtype od, bool norm, float target,
                        void* out, uint64_t* out_gidx, cudaStream_t st, uint64_t avg_nnz) {
    if (a.layout != Layout::csr) invalid("csr_densify: store is not csr");
    if (norm && od == OutDtype::native && a.vdt != VDtype::f32)
        invalid("csr_densify: normalize_log1p needs a floating output dtype (f32 or bf16)");
    if (n == 0) return;
    if (a.idx16) densify_idx<uint16_t>(a, refs, n, od, norm, target, out, out_gidx, st, avg_nnz);
    else if (a.idt == IDtype::u32) densify_idx<uint32_t>(a, refs, n, od, norm, target, out, out_gidx, st, avg_nnz);
    else densify_idx<uint64_t>(a, refs, n, od, norm, target, out, out_gidx, st, avg_nnz);
}

namespace {
template <typename SrcT, typename DstT>
void densify_d8_t(const ArenaView& av, const RowRef* refs, uint64_t n, bool norm, float target, void* out,
                  uint64_t* out_gidx, cudaStream_t st) {
    // shape rule: rows wider than 48 KB -> two alternating 40 KB tiles at 2 CTAs/SM (the next
    // tile is built while the previous bulk store drains; cfg2 116.8 -> 114.9 us per batch vs one
    // 80 KB tile, profiles/r2/s3/k3d_tiles.txt), else one 40 KB tile at 3
    const uint64_t esz = sizeof(DstT);
    const D8Shape& ov = d8_shape();
    const bool wide = av.n_var * esz > 48 * 1024;
    const uint64_t max_tile = ov.tile_kb ? static_cast<uint64_t>(ov.tile_kb) << 10 : (40u << 10);
    const int minb = ov.minb ? ov.minb : wide ? 2 : 3, nbuf = ov.nbuf ? ov.nbuf : wide ? 2 : 1;
    uint64_t tile_cols = av.n_var;
    if (av.n_var * esz > max_tile) tile_cols = (max_tile / esz) & ~15ull;
    int bulk = ((av.n_var * esz) % 16 == 0) && (reinterpret_cast<uintptr_t>(out) % 16 == 0);
    if (bulk && nbuf == 2 && tile_cols < av.n_var) bulk = 2;
    const size_t smem = ((tile_cols * esz + 127) & ~127ull) * (bulk == 2 ? 2 : 1);
    auto kern = minb == 2 ? k_csr_densify_d8<SrcT, DstT, 256, 2> : k_csr_densify_d8<SrcT, DstT, 256, 3>;
    set_smem(kern, smem);
    int per_sm = 0;
    cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem), "occupancy");
    const uint64_t grid = std::min<uint64_t>(n, static_cast<uint64_t>(std::max(per_sm, 1)) * device_sm_count());
    launch_k(kern, dim3(static_cast<unsigned>(grid)), dim3(256), smem, st, "k_csr_densify_d8 launch", dev_view(av),
             refs, n, static_cast<uint32_t>(tile_cols), norm ? 1 : 0, target, static_cast<DstT*>(out), out_gidx, bulk);
}
}  // namespace

void launch_csr_densify_d8(const ArenaView& a, const RowRef* refs, uint64_t n, OutDtype od, bool norm, float target,
                           void* out, uint64_t* out_gidx, cudaStream_t st) {
    if (a.layout != Layout::csr) invalid("csr_densify_d8: store is not csr");
    if (n == 0) return;
    if (a.vdt == VDtype::f32) {
        if (od == OutDtype::bf16) return densify_d8_t<float, __nv_bfloat16>(a, refs, n, norm, target, out, out_gidx, st);
        return densify_d8_t<float, float>(a, refs, n, norm, target, out, out_gidx, st);
    }
    if (a.vdt == VDtype::i32) {
        if (od == OutDtype::bf16) return densify_d8_t<int32_t, __nv_bfloat16>(a, refs, n, norm, target, out, out_gidx, st);
        if (od == OutDtype::f32) return densify_d8_t<int32_t, float>(a, refs, n, norm, target, out, out_gidx, st);
        return densify_d8_t<int32_t, int32_t>(a, refs, n, false, target, out, out_gidx, st);
    }
    invalid("csr_densify_d8: delta records carry 4-byte values (f32 / i32)");
}

void launch_dense_gather(const ArenaView& a, const RowRef* refs, uint64_t n, OutDtype od, void* out,
                         uint64_t* out_gidx, cudaStream_t st) {
    if (a.layout != Layout::dense) invalid("dense_gather: store is not dense");
    if (n == 0) return;
    const uint64_t in_rb = a.n_var * value_size(a.vdt);
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(n, 8ull * device_sm_count()));
    const ArenaDev d = dev_view(a);
    auto* o = static_cast<uint8_t*>(out);
    // records sit at 16-B aligned offsets, so rows are 16-B aligned whenever row_bytes is
    const bool flat = in_rb % 16 == 0 && reinterpret_cast<uintptr_t>(a.base) % 16 == 0 &&
                      reinterpret_cast<uintptr_t>(out) % 16 == 0;
    if (flat) {
        // 16-B loads per lane per work unit: 2 (profiles/r1_dense_gather.md: best for both
        // dense shapes; a one-wave unit of 3 for cfg3 is slower, 0.58 vs 0.62 -- shorter
        // per-warp chains win over filling the tail wave).  RFL_DG=4 for A/B.
        static const int u_sel = [] {
            const char* e = std::getenv("RFL_DG");
            if (!e) return 0;  // automatic
            if (e[0] == 'b') return e[1] == '4' ? -4 : -2;  // TMA bulk-store variant, 2 or 4 loads per lane
            if (e[0] == 'r') return 8;                      // whole rows through TMA
            return e[0] == '4' ? 4 : 2;
        }();
        auto go = [&](auto kern, int U, int T) {
            const uint64_t upr = (in_rb / 16 + 32 * U - 1) / (32 * U);
            const uint64_t warps_needed = n * upr;
            const unsigned g2 = static_cast<unsigned>(std::max<uint64_t>(
                1, std::min<uint64_t>((warps_needed + T / 32 - 1) / (T / 32), 2048ull * device_sm_count() / T)));
            const uint64_t orb = od == OutDtype::bf16 ? a.n_var * 2 : in_rb;
            launch_k(kern, dim3(g2), dim3(T), 0, st, "k_dense_gather_flat launch", d, in_rb, refs, n, o, orb, out_gidx);
        };
        auto pick = [&](auto mode) {
            constexpr int M = decltype(mode)::value;
            if constexpr (M != kF32ToBf16) {
                // whole rows through TMA when every CTA streams >= 4 rows through its two
                // stages (the grouped launches: cfg3 x2 0.75 -> 0.78, cfg4 raw x4 0.75 -> 0.80;
                // a single 1,024-row cfg3 batch is faster with the warp units, 0.65 vs 0.61,
                // profiles/r2/s3/kb_dense_rows.txt).  RFL_DG=row forces it, other RFL_DG values
                // keep the warp-unit kernels.
                if ((u_sel == 8 || u_sel == 0) && in_rb <= (24u << 10)) {
                    const uint64_t orb = M == kU8ToBf16 ? in_rb * 2 : in_rb;
                    const uint32_t stage = static_cast<uint32_t>(
                        M == kRaw ? ((in_rb + 127) & ~127ull) : ((in_rb + 127) & ~127ull) + orb);
                    const size_t smem = 2ull * stage;
                    auto kern = k_dense_gather_rows<M>;
                    int occ = 0;
                    {  // (loaders on several host threads launch concurrently)
                        static std::mutex mu;
                        static size_t set_to = 0;
                        static int occ_at = 0;
                        std::lock_guard<std::mutex> lk(mu);
                        if (set_to != smem) {
                            set_smem(kern, std::max(smem, set_to));
                            set_to = std::max(smem, set_to);
                            cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_at, kern, 256, smem),
                                       "occupancy");
                        }
                        occ = occ_at;
                    }
                    const uint64_t ctas = static_cast<uint64_t>(std::max(occ, 1)) * device_sm_count();
                    if (u_sel == 8 || n >= 4 * ctas) {
                        const unsigned g = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(n, ctas)));
                        return launch_k(kern, dim3(g), dim3(256), smem, st, "k_dense_gather_rows launch", d, in_rb,
                                        refs, n, o, orb, out_gidx, stage);
                    }
                }
            }
            if (u_sel == 4) return go(k_dense_gather_flat<M, 4, 256>, 4, 256);
            if constexpr (M != kF32ToBf16) {
                // automatic: the u8 -> bf16 expansion writes through TMA bulk stores
                // (cfg3 0.63 -> 0.81), raw copies keep the register path (cfg4 0.63 vs 0.55)
                if (u_sel == -2 || (u_sel == 0 && M == kU8ToBf16)) return go(k_dense_gather_bulk<M, 2, 256>, 2, 256);
                if (u_sel == -4) return go(k_dense_gather_bulk<M, 4, 256>, 4, 256);
            }
            return go(k_dense_gather_flat<M, 2, 256>, 2, 256);
        };
        if (od == OutDtype::bf16 && a.vdt == VDtype::u8) {
            pick(std::integral_constant<int, kU8ToBf16>{});
        } else if (od == OutDtype::bf16 && a.vdt == VDtype::f32) {
            pick(std::integral_constant<int, kF32ToBf16>{});
        } else if (od == OutDtype::native || (od == OutDtype::f32 && a.vdt == VDtype::f32)) {
            pick(std::integral_constant<int, kRaw>{});
        } else {
            invalid("dense_gather: unsupported output dtype for this store");
        }
        return;
    }
    if (od == OutDtype::bf16) {
        if (a.vdt == VDtype::u8)
            k_dense_gather<kU8ToBf16><<<grid, kDenseGatherThreads, 0, st>>>(d, in_rb, refs, n, o, a.n_var * 2, out_gidx);
        else if (a.vdt == VDtype::f32)
            k_dense_gather<kF32ToBf16><<<grid, kDenseGatherThreads, 0, st>>>(d, in_rb, refs, n, o, a.n_var * 2, out_gidx);
        else
            invalid("dense_gather: bf16 cast supports u8 and f32 stores");
    } else if (od == OutDtype::native || (od == OutDtype::f32 && a.vdt == VDtype::f32)) {
        k_dense_gather<kRaw><<<grid, kDenseGatherThreads, 0, st>>>(d, in_rb, refs, n, o, in_rb, out_gidx);
    } else {
        invalid("dense_gather: unsupported output dtype for this store");
    }
    cuda_check(cudaGetLastError(), "k_dense_gather launch");
}

void launch_onehot_gather(const ArenaView& a, const RowRef* refs, uint64_t n, OutDtype od, void* out,
                          uint64_t* out_gidx, cudaStream_t st) {
    if (a.layout != Layout::dense || a.vdt != VDtype::u8 || a.n_var % 64 != 0)
        invalid("onehot_gather: needs one-hot staged dense u8 rows with n_var % 64 == 0");
    if (n == 0) return;
    const uint64_t wpr = a.n_var / 64, upr = (wpr + 63) / 64;
    const uint64_t warps_needed = n * upr;
    const unsigned grid = static_cast<unsigned>(
        std::max<uint64_t>(1, std::min<uint64_t>((warps_needed + 7) / 8, 8ull * device_sm_count())));
    const ArenaDev d = dev_view(a);
    auto* o = static_cast<uint8_t*>(out);
    // RFL_OH=plain (A/B): register 16-B stores; default: whole rows through two shared stages +
    // one bulk store per row (cfg4 950-998 vs 936 M rows/s for plain stores; R-row shared tiles,
    // per-warp bulk stores and 16 KB row groups measured slower, profiles/r2/s3/README.md)
    static const bool plain = [] {
        const char* e = std::getenv("RFL_OH");
        return e && std::string(e) == "plain";
    }();
    const int variant = plain ? 2 : 3;
    if (variant == 3 && od != OutDtype::f32 && a.n_var <= 32768) {
        const uint64_t rb = a.n_var * (od == OutDtype::bf16 ? 2 : 1);
        const size_t smem = 2 * rb;
        auto kern = od == OutDtype::bf16 ? k_onehot_gather_rows<kOhBf16> : k_onehot_gather_rows<kOhU8>;
        const int ki = od == OutDtype::bf16 ? 1 : 0;
        int oc = 0;
        {
            static std::mutex mu;
            static size_t set_to[2] = {0, 0};
            static int occ[2] = {0, 0};
            std::lock_guard<std::mutex> lk(mu);
            if (set_to[ki] < smem) {
                set_smem(kern, std::max<size_t>(smem, 16u << 10));
                set_to[ki] = std::max<size_t>(smem, 16u << 10);
                cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[ki], kern, 64, smem), "occupancy");
            }
            oc = occ[ki];
        }
        const unsigned g = static_cast<unsigned>(std::max<uint64_t>(
            1, std::min<uint64_t>(n, static_cast<uint64_t>(std::max(oc, 1)) * device_sm_count())));
        launch_k(kern, dim3(g), dim3(64), smem, st, "k_onehot_gather_rows launch", dev_view(a), refs, n,
                 static_cast<uint8_t*>(out), out_gidx);
        return;
    }
    if (od == OutDtype::bf16)
        launch_k(k_onehot_gather<kOhBf16>, dim3(grid), dim3(256), 0, st, "k_onehot_gather launch", d, refs, n, o, out_gidx);
    else if (od == OutDtype::f32)  // as launch_dense_gather: u8 rows cast to bf16 only
        invalid("dense_gather: unsupported output dtype for this store");
    else
        launch_k(k_onehot_gather<kOhU8>, dim3(grid), dim3(256), 0, st, "k_onehot_gather launch", d, refs, n, o, out_gidx);
}

namespace {
// RFL_PULL=<piece KB>:<stages>:<CTAs> (A/B; default 16 KB x 4 stages x 32 CTAs = 2 MB in flight)
const std::array<uint32_t, 3>& pull_shape() {
    static const std::array<uint32_t, 3> v = [] {
        std::array<uint32_t, 3> x{16, 4, 32};
        if (const char* e = std::getenv("RFL_PULL")) std::sscanf(e, "%u:%u:%u", &x[0], &x[1], &x[2]);
        x[0] = std::max(1u, std::min(64u, x[0]));
        x[1] = std::max(2u, std::min<uint32_t>(kMaxPullStages, x[1]));
        x[2] = std::max(1u, std::min(256u, x[2]));
        if (x[0] * x[1] > 192) x[1] = 192 / x[0];
        return x;
    }();
    return v;
}
}  // namespace

uint32_t stage_pull_piece_bytes() { return pull_shape()[0] << 10; }

void launch_stage_pull(const PullJobs& jobs, cudaStream_t st) {
    if (jobs.n == 0) return;
    const uint32_t P = pull_shape()[0] << 10, S = pull_shape()[1];
    static const bool attr = [] {
        set_smem(k_stage_pull, 192u << 10);
        return true;
    }();
    (void)attr;
    const uint32_t total = jobs.first_piece[jobs.n];
    const unsigned grid = std::max(1u, std::min(pull_shape()[2], total));
    launch_k(k_stage_pull, dim3(grid), dim3(32), static_cast<size_t>(P) * S, st, "k_stage_pull launch", jobs, P, S);
}

}  // namespace rfl
