// extern "C" boundary (include/riffle_b200.h).  No exception crosses it: each
// entry point maps rfl::Error codes (InvalidArgument / CorruptStore / IoError,
// reference error.hpp:9-32) and CUDA failures to rfl_status and records the
// message in a thread-local buffer.
#include <cuda_runtime.h>

#include <cstring>
#include <memory>
#include <new>
#include <string>

#include "../../include/riffle_b200.h"
#include "engine.hpp"
#include "format.hpp"
#include "kernels.cuh"
#include "preshuffle.hpp"
#include "schedule.hpp"
#include "synth.hpp"

namespace {
thread_local std::string g_err;

template <typename F>
rfl_status guarded(F&& f) {
    try {
        f();
        return RFL_OK;
    } catch (const rfl::Error& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "out of host memory";
        return RFL_ENOMEM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return RFL_EINVAL;
    }
}

rfl::LoaderCfg to_cfg(const rfl_loader_config* c) {
    if (!c) rfl::invalid("null loader config");
    rfl::LoaderCfg o;
    o.f = c->fetch_block_rows;
    o.B = c->buffer_capacity_rows;
    o.b = c->batch_rows;
    o.seed = c->seed;
    o.prefetch_depth = c->prefetch_depth;
    o.drop_last = c->drop_last != 0;
    o.cache_bypass = c->cache_bypass != 0;
    o.rank = c->rank;
    o.world = c->world ? c->world : 1;
    o.even_batches = c->even_batches != 0;
    return o;
}

rfl::ArenaView to_view(const rfl_arena_desc* a) {
    if (!a || !a->base) rfl::invalid("null arena");
    if (a->chunk_rows == 0) rfl::invalid("arena chunk_rows must be >= 1");
    if (a->value_dtype > RFL_U8 || a->index_dtype > RFL_IDX_U64 || a->layout > RFL_LAYOUT_CSR)
        rfl::invalid("arena: bad dtype/layout");
    rfl::ArenaView v;
    v.base = static_cast<const uint8_t*>(a->base);
    v.chunk_rows = a->chunk_rows;
    v.n_var = a->n_var;
    v.layout = static_cast<rfl::Layout>(a->layout);
    v.vdt = static_cast<rfl::VDtype>(a->value_dtype);
    v.idt = static_cast<rfl::IDtype>(a->index_dtype);
    return v;
}

// Scratch for the raw entry points comes from the stream-ordered allocator;
// keep freed blocks in the device pool instead of returning them to the driver
// at every synchronisation (the default threshold of 0 made each call pay a
// fresh allocation).
void* scratch_alloc(size_t bytes, cudaStream_t st) {
    int dev = 0;
    rfl::cuda_ok(cudaGetDevice(&dev), "cudaGetDevice");
    static thread_local int configured = -1;
    if (configured != dev) {
        cudaMemPool_t pool;
        rfl::cuda_ok(cudaDeviceGetDefaultMemPool(&pool, dev), "cudaDeviceGetDefaultMemPool");
        uint64_t keep = ~0ull;
        rfl::cuda_ok(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep), "pool attr");
        configured = dev;
    }
    void* p = nullptr;
    rfl::cuda_ok(cudaMallocAsync(&p, bytes, st), "cudaMallocAsync");
    return p;
}

rfl::OutDtype to_od(uint32_t d) {
    switch (d) {
        case RFL_NATIVE: return rfl::OutDtype::native;
        case RFL_F32: return rfl::OutDtype::f32;
        case RFL_BF16: return rfl::OutDtype::bf16;
        default: rfl::invalid("out_dtype must be RFL_NATIVE, RFL_F32 or RFL_BF16");
    }
}
}  // namespace

struct rfl_store {
    std::shared_ptr<rfl::HostStore> hs;
};
struct rfl_schedule {
    rfl::EpochReplay replay;
    std::vector<uint64_t> consumed;
};
struct rfl_dstore {
    std::shared_ptr<rfl::DStore> ds;
};
struct rfl_loader {
    std::unique_ptr<rfl::GpuLoader> l;
};

extern "C" {

const char* rfl_last_error(void) { return g_err.c_str(); }
const char* rfl_version(void) { return "riffle_b200 0.1 (sm_100a)"; }
int rfl_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

rfl_status rfl_device_can_access_peer(int device, int peer, int* out) {
    return guarded([&] {
        if (!out) rfl::invalid("null argument");
        if (device == peer) {
            *out = 1;
            return;
        }
        int ok = 0;
        rfl::cuda_ok(cudaDeviceCanAccessPeer(&ok, device, peer), "cudaDeviceCanAccessPeer");
        *out = ok;
    });
}

// ------------------------------------------------------------------ stores --
rfl_status rfl_store_open(const char* root, rfl_store** out) {
    return guarded([&] {
        if (!root || !out) rfl::invalid("null argument");
        auto* s = new rfl_store;
        try {
            s->hs = std::make_shared<rfl::HostStore>(root);
        } catch (...) {
            delete s;
            throw;
        }
        *out = s;
    });
}

rfl_status rfl_store_get_info(const rfl_store* s, rfl_store_info* o) {
    return guarded([&] {
        if (!s || !o) rfl::invalid("null argument");
        const auto& m = s->hs->manifest();
        o->format_version = m.format_version;
        o->layout = static_cast<uint32_t>(m.layout);
        o->n_obs = m.n_obs;
        o->n_var = m.n_var;
        o->value_dtype = static_cast<uint32_t>(m.value_dtype);
        o->index_dtype = m.index_dtype ? static_cast<uint32_t>(*m.index_dtype) : 0;
        o->chunk_rows = m.chunk_rows;
        o->chunks_per_shard = m.chunks_per_shard;
        o->codec = static_cast<uint32_t>(m.codec);
        o->has_provenance = m.has_provenance;
    });
}

rfl_status rfl_store_record_size(rfl_store* s, uint64_t chunk, uint64_t* nbytes) {
    return guarded([&] {
        if (!s || !nbytes) rfl::invalid("null argument");
        if (chunk >= s->hs->manifest().chunk_count()) rfl::invalid("chunk out of range");
        *nbytes = s->hs->record_slot(chunk).len;
    });
}

rfl_status rfl_store_read_record(rfl_store* s, uint64_t chunk, void* dst, uint64_t cap) {
    return guarded([&] {
        if (!s || !dst) rfl::invalid("null argument");
        if (chunk >= s->hs->manifest().chunk_count()) rfl::invalid("chunk out of range");
        s->hs->read_record(chunk, dst, cap);
    });
}

void rfl_store_close(rfl_store* s) { delete s; }

rfl_status rfl_synth_store(const char* path, const rfl_synth_config* c) {
    return guarded([&] {
        if (!path || !c) rfl::invalid("null argument");
        if (c->layout > RFL_LAYOUT_CSR || c->value_dtype > RFL_U8 || c->index_dtype > RFL_IDX_U64)
            rfl::invalid("synth: bad layout/dtype");
        rfl::SynthCfg s;
        s.n_obs = c->n_obs;
        s.n_var = c->n_var;
        s.layout = static_cast<rfl::Layout>(c->layout);
        s.value_dtype = static_cast<rfl::VDtype>(c->value_dtype);
        s.index_dtype = static_cast<rfl::IDtype>(c->index_dtype);
        s.codec = static_cast<rfl::Codec>(c->codec);
        s.density = c->density;
        s.seed = c->seed;
        s.chunk_rows = c->chunk_rows;
        s.chunks_per_shard = c->chunks_per_shard;
        s.threads = c->threads;
        s.one_hot = c->one_hot;
        s.counts = c->counts != 0;
        rfl::synth_store(path, s);
    });
}

// ---------------------------------------------------------------- schedule --
rfl_status rfl_loader_config_validate(const rfl_loader_config* c) {
    return guarded([&] { to_cfg(c).validate(); });
}

rfl_status rfl_plan_epoch(uint64_t n_obs, const rfl_loader_config* c, uint64_t epoch, uint64_t* starts,
                          uint64_t* ends) {
    return guarded([&] {
        const rfl::LoaderCfg cfg = to_cfg(c);
        const auto ids = rfl::plan_epoch_ids(n_obs, cfg, epoch);
        for (size_t i = 0; i < ids.size(); ++i) {
            starts[i] = ids[i] * cfg.f;
            ends[i] = std::min(n_obs, (ids[i] + 1) * cfg.f);
        }
    });
}

rfl_status rfl_schedule_create(uint64_t n_obs, const rfl_loader_config* c, uint64_t epoch, rfl_schedule** out) {
    return guarded([&] {
        if (!out) rfl::invalid("null argument");
        *out = new rfl_schedule{rfl::EpochReplay(n_obs, to_cfg(c), epoch), {}};
    });
}

rfl_status rfl_schedule_next(rfl_schedule* s, uint64_t* gidx_out, uint64_t* n_rows) {
    std::vector<uint64_t> g;
    bool more = false;
    const rfl_status st = guarded([&] {
        if (!s || !gidx_out || !n_rows) rfl::invalid("null argument");
        more = s->replay.next(g, s->consumed);
        std::memcpy(gidx_out, g.data(), g.size() * 8);
        *n_rows = g.size();
    });
    if (st != RFL_OK) return st;
    return more ? RFL_OK : RFL_END;
}

rfl_status rfl_schedule_stats(const rfl_schedule* s, uint64_t* peak, uint64_t* blocks) {
    return guarded([&] {
        if (!s) rfl::invalid("null argument");
        if (peak) *peak = s->replay.peak_buffer_rows();
        if (blocks) *blocks = s->replay.blocks_fetched();
    });
}

void rfl_schedule_destroy(rfl_schedule* s) { delete s; }

// ------------------------------------------------------------------ dstore --
rfl_status rfl_dstore_create(rfl_store* s, int device, uint32_t staging, rfl_dstore** out) {
    return guarded([&] {
        if (!s || !out) rfl::invalid("null argument");
        *out = new rfl_dstore{std::make_shared<rfl::DStore>(s->hs, device, staging)};
    });
}

rfl_status rfl_dstore_bytes(const rfl_dstore* d, uint64_t* record_bytes, uint64_t* staged_bytes) {
    return guarded([&] {
        if (!d) rfl::invalid("null argument");
        if (record_bytes) *record_bytes = d->ds->image_bytes();
        if (staged_bytes) *staged_bytes = d->ds->staged_bytes();
    });
}

rfl_status rfl_dstore_arena(const rfl_dstore* d, void** base, const uint64_t** offs, uint64_t* n) {
    return guarded([&] {
        if (!d) rfl::invalid("null argument");
        const bool coded = d->ds->staging() == rfl::kResidentCoded;
        if (d->ds->staging() != rfl::kResident && !coded)
            rfl::invalid("arena only exists for resident / resident_coded stores");
        if (base) *base = const_cast<uint8_t*>(d->ds->d_arena());
        const std::vector<uint64_t>& o = coded ? d->ds->img_off() : d->ds->rec_off();
        if (offs) *offs = o.data();
        if (n) *n = o.size();
    });
}

void rfl_dstore_destroy(rfl_dstore* d) { delete d; }

// ------------------------------------------------------------------ loader --
rfl_status rfl_loader_create(rfl_dstore* d, const rfl_loader_config* c, uint64_t epoch, const rfl_device_config* dev,
                             rfl_loader** out) {
    return guarded([&] {
        if (!d || !out) rfl::invalid("null argument");
        rfl::DeviceCfg dc;
        if (dev) {
            dc.output = dev->output;
            if (dc.output > RFL_OUT_DENSE) rfl::invalid("output must be RFL_OUT_CSR or RFL_OUT_DENSE");
            dc.out_dtype = to_od(dev->out_dtype);
            dc.normalize = dev->transform == RFL_XF_NORMALIZE_LOG1P;
            if (dev->transform > RFL_XF_NORMALIZE_LOG1P) rfl::invalid("unknown transform");
            dc.target_sum = dev->target_sum > 0 ? dev->target_sum : 1e4f;
            dc.out_slots = dev->out_slots ? dev->out_slots : 2;
            dc.stream = static_cast<cudaStream_t>(dev->stream);
            dc.time_kernels = (dev->flags & RFL_DEV_TIME_KERNELS) != 0;
            dc.group = dev->batches_per_launch ? dev->batches_per_launch : 1;
            if (dc.group > 64) rfl::invalid("batches_per_launch must be <= 64");
        } else {
            dc.output = d->ds->manifest().layout == rfl::Layout::csr ? 0 : 1;
        }
        *out = new rfl_loader{std::make_unique<rfl::GpuLoader>(d->ds, to_cfg(c), epoch, dc)};
    });
}

namespace {
void to_batch(const rfl::BatchOut& b, rfl_batch* o) {
    o->epoch_index = b.epoch;
    o->batch_index = b.batch_index;
    o->n_rows = b.n_rows;
    o->nnz = b.nnz;
    o->n_var = b.n_var;
    o->layout = b.layout;
    o->dtype = b.dtype;
    o->index_dtype = b.index_dtype;
    o->reserved = 0;
    o->d_gidx = b.d_gidx;
    o->d_indptr = b.d_indptr;
    o->d_indices = b.d_indices;
    o->d_data = b.d_data;
    o->h_gidx = b.h_gidx;
    o->ready_event = b.ready;
}
}  // namespace

rfl_status rfl_loader_next(rfl_loader* l, rfl_batch* o) {
    bool more = false;
    const rfl_status st = guarded([&] {
        if (!l || !o) rfl::invalid("null argument");
        rfl::BatchOut b;
        more = l->l->next(b);
        if (more) to_batch(b, o);
    });
    if (st != RFL_OK) return st;
    return more ? RFL_OK : RFL_END;
}

rfl_status rfl_loader_next_many(rfl_loader* l, rfl_batch* o, uint32_t max, uint32_t* n) {
    uint32_t got = 0;
    const rfl_status st = guarded([&] {
        if (!l || !o || !n) rfl::invalid("null argument");
        rfl::BatchOut b;
        while (got < max && l->l->next(b)) to_batch(b, o + got++);
        *n = got;
    });
    if (st != RFL_OK) return st;
    return got ? RFL_OK : RFL_END;
}

rfl_status rfl_loader_counters_get(const rfl_loader* l, rfl_loader_counters* o) {
    return guarded([&] {
        if (!l || !o) rfl::invalid("null argument");
        const rfl::Counters c = l->l->counters();
        o->blocks_fetched = c.blocks_fetched;
        o->read_ops = c.read_ops;
        o->bytes_read = c.bytes_read;
        o->chunks_decoded = c.chunks_decoded;
        o->peak_buffer_rows = c.peak_buffer_rows;
        o->h2d_bytes = c.h2d_bytes;
        o->kernels_launched = c.kernels_launched;
        o->decode_ms = c.decode_ms;
        o->assembly_ms = c.assembly_ms;
    });
}

rfl_status rfl_batch_download(const rfl_batch* b, uint64_t* h_indptr, void* h_indices, void* h_data,
                              uint64_t* h_gidx) {
    return guarded([&] {
        if (!b) rfl::invalid("null argument");
        if (b->ready_event) rfl::cuda_ok(cudaEventSynchronize(static_cast<cudaEvent_t>(b->ready_event)), "sync");
        auto d2h = [](void* dst, const void* src, uint64_t n) {
            if (dst && src && n) rfl::cuda_ok(cudaMemcpy(dst, src, n, cudaMemcpyDeviceToHost), "batch D2H");
        };
        static const uint64_t esz[] = {4, 8, 4, 1, 2};  // RFL_F32, F64, I32, U8, BF16
        if (b->dtype > RFL_BF16) rfl::invalid("batch: unknown dtype");
        const uint64_t n_elem = b->layout == RFL_LAYOUT_CSR ? b->nnz : b->n_rows * b->n_var;
        d2h(h_gidx, b->d_gidx, 8 * b->n_rows);
        if (b->layout == RFL_LAYOUT_CSR) {
            d2h(h_indptr, b->d_indptr, 8 * (b->n_rows + 1));
            d2h(h_indices, b->d_indices, (b->index_dtype == RFL_IDX_U32 ? 4 : 8) * b->nnz);
        }
        d2h(h_data, b->d_data, esz[b->dtype] * n_elem);
    });
}

rfl_status rfl_batch_wait(const rfl_batch* b, void* stream) {
    return guarded([&] {
        if (!b) rfl::invalid("null argument");
        if (b->ready_event)
            rfl::cuda_ok(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream),
                                             static_cast<cudaEvent_t>(b->ready_event), 0),
                         "cudaStreamWaitEvent");
    });
}

rfl_status rfl_ids_download_async(const uint64_t* d_gidx, uint64_t n_rows, uint64_t* h_gidx, void* stream) {
    return guarded([&] {
        if (n_rows && (!d_gidx || !h_gidx)) rfl::invalid("null argument");
        if (n_rows)
            rfl::cuda_ok(cudaMemcpyAsync(h_gidx, d_gidx, n_rows * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                                         static_cast<cudaStream_t>(stream)),
                         "ids D2H");
    });
}

rfl_status rfl_loader_sync(rfl_loader* l) {
    return guarded([&] {
        if (!l) rfl::invalid("null argument");
        l->l->sync();
    });
}

void rfl_loader_destroy(rfl_loader* l) { delete l; }

// -------------------------------------------------------------- raw kernels --
rfl_status rfl_csr_gather(const rfl_arena_desc* a, const rfl_rowref* refs, uint64_t n, uint64_t* out_indptr,
                          void* out_indices, void* out_data, uint64_t* out_gidx, void* stream) {
    return guarded([&] {
        const rfl::ArenaView v = to_view(a);
        auto st = static_cast<cudaStream_t>(stream);
        void* scratch = scratch_alloc(rfl::csr_gather_scratch_bytes(n), st);
        rfl::launch_csr_gather(v, reinterpret_cast<const rfl::RowRef*>(refs), n, out_indptr, out_indices, out_data,
                               out_gidx, scratch, st);
        rfl::cuda_ok(cudaFreeAsync(scratch, st), "cudaFreeAsync");
    });
}

rfl_status rfl_csr_gather_prefixed(const rfl_arena_desc* a, const rfl_rowref* refs, uint64_t n, const uint64_t* prefix,
                                   void* out_indices, void* out_data, uint64_t* out_gidx, void* stream) {
    return guarded([&] {
        if (n && !prefix) rfl::invalid("csr_gather_prefixed: prefix is NULL");
        rfl::launch_csr_gather_prefixed(to_view(a), reinterpret_cast<const rfl::RowRef*>(refs), n, prefix, out_indices,
                                        out_data, out_gidx, static_cast<cudaStream_t>(stream));
    });
}

rfl_status rfl_csr_densify(const rfl_arena_desc* a, const rfl_rowref* refs, uint64_t n, uint32_t out_dtype,
                           uint32_t transform, float target, void* out, uint64_t* out_gidx, void* stream) {
    return guarded([&] {
        if (transform > RFL_XF_NORMALIZE_LOG1P) rfl::invalid("unknown transform");
        rfl::launch_csr_densify(to_view(a), reinterpret_cast<const rfl::RowRef*>(refs), n, to_od(out_dtype),
                                transform == RFL_XF_NORMALIZE_LOG1P, target > 0 ? target : 1e4f, out, out_gidx,
                                static_cast<cudaStream_t>(stream));
    });
}

rfl_status rfl_dense_gather(const rfl_arena_desc* a, const rfl_rowref* refs, uint64_t n, uint32_t out_dtype,
                            void* out, uint64_t* out_gidx, void* stream) {
    return guarded([&] {
        rfl::launch_dense_gather(to_view(a), reinterpret_cast<const rfl::RowRef*>(refs), n, to_od(out_dtype), out,
                                 out_gidx, static_cast<cudaStream_t>(stream));
    });
}

rfl_status rfl_onehot_gather(const rfl_arena_desc* a, const rfl_rowref* refs, uint64_t n, uint32_t out_dtype,
                             void* out, uint64_t* out_gidx, void* stream) {
    return guarded([&] {
        rfl::launch_onehot_gather(to_view(a), reinterpret_cast<const rfl::RowRef*>(refs), n, to_od(out_dtype), out,
                                  out_gidx, static_cast<cudaStream_t>(stream));
    });
}

rfl_status rfl_csr_scan(const rfl_arena_desc* a, const rfl_rowref* refs, uint64_t n, uint64_t* out_prefix,
                        void* stream) {
    return guarded([&] {
        auto st = static_cast<cudaStream_t>(stream);
        void* scratch = scratch_alloc(rfl::csr_gather_scratch_bytes(n), st);
        rfl::launch_csr_row_scan(to_view(a), reinterpret_cast<const rfl::RowRef*>(refs), n, out_prefix, scratch, st);
        rfl::cuda_ok(cudaFreeAsync(scratch, st), "cudaFreeAsync");
    });
}

rfl_status rfl_csr_pack(const rfl_arena_desc* a, const rfl_rowref* refs, uint64_t n, uint64_t chunk_rows,
                        uint32_t out_idt, const uint64_t* prefix, void* out, void* stream) {
    return guarded([&] {
        if (chunk_rows == 0 || out_idt > RFL_IDX_U64) rfl::invalid("csr_pack: bad chunk_rows / index dtype");
        rfl::launch_csr_pack(to_view(a), reinterpret_cast<const rfl::RowRef*>(refs), n, chunk_rows,
                             static_cast<rfl::IDtype>(out_idt), prefix, static_cast<uint8_t*>(out),
                             static_cast<cudaStream_t>(stream));
    });
}

// -------------------------------------------------------------- preshuffle --
rfl_status rfl_plan_shuffle(uint64_t total, uint64_t c, uint64_t m, uint64_t seed, uint64_t* n_rounds,
                            uint64_t* round_len, uint64_t* ids) {
    return guarded([&] {
        const rfl::ShufflePlan p = rfl::plan_shuffle(total, c, m, seed);
        if (n_rounds) *n_rounds = p.rounds.size();
        uint64_t k = 0;
        for (size_t r = 0; r < p.rounds.size(); ++r) {
            if (round_len) round_len[r] = p.rounds[r].size();
            for (uint64_t id : p.rounds[r]) {
                if (ids) ids[k] = id;
                ++k;
            }
        }
    });
}

rfl_status rfl_shuffle_order(uint64_t total, uint64_t c, uint64_t m, uint64_t seed, uint64_t* out_src) {
    return guarded([&] {
        if (!out_src) rfl::invalid("null argument");
        const rfl::ShufflePlan p = rfl::plan_shuffle(total, c, m, seed);
        uint64_t o = 0;
        std::vector<uint64_t> assembly;
        for (size_t r = 0; r < p.rounds.size(); ++r) {
            assembly.clear();
            for (uint64_t id : p.rounds[r])
                for (uint64_t g = p.block_start(id); g < p.block_end(id); ++g) assembly.push_back(g);
            const auto perm = rfl::round_permutation(seed, r, assembly.size());
            for (uint64_t k : perm) out_src[o++] = assembly[k];
        }
    });
}

rfl_status rfl_shuffle_round_routes(uint64_t total, uint64_t c, uint64_t m, uint64_t seed, uint64_t out_chunk_rows,
                                    uint64_t out_cps, uint32_t world, uint64_t round, uint64_t* first_out_row,
                                    uint64_t* n_rows, uint64_t* src_rows, uint32_t* src_rank, uint32_t* dst_rank) {
    return guarded([&] {
        if (world < 1 || out_chunk_rows < 1 || out_cps < 1) rfl::invalid("routes: bad geometry");
        const rfl::ShufflePlan p = rfl::plan_shuffle(total, c, m, seed);
        if (round >= p.rounds.size()) rfl::invalid("routes: round out of range");
        uint64_t base = 0;
        for (uint64_t r = 0; r < round; ++r)
            for (uint64_t id : p.rounds[r]) base += p.block_end(id) - p.block_start(id);
        std::vector<uint64_t> asm_rows;
        std::vector<uint32_t> asm_src;
        for (size_t bi = 0; bi < p.rounds[round].size(); ++bi) {
            const uint64_t id = p.rounds[round][bi];
            for (uint64_t g = p.block_start(id); g < p.block_end(id); ++g) {
                asm_rows.push_back(g);
                asm_src.push_back(static_cast<uint32_t>(bi % world));  // block bi staged by rank bi mod W
            }
        }
        if (first_out_row) *first_out_row = base;
        if (n_rows) *n_rows = asm_rows.size();
        if (!src_rows) return;
        const auto perm = rfl::round_permutation(seed, round, asm_rows.size());
        const uint64_t shard_rows = out_chunk_rows * out_cps;
        for (uint64_t k = 0; k < perm.size(); ++k) {
            src_rows[k] = asm_rows[perm[k]];
            if (src_rank) src_rank[k] = asm_src[perm[k]];
            if (dst_rank) dst_rank[k] = static_cast<uint32_t>(((base + k) / shard_rows) % world);  // shard owner
        }
    });
}

namespace {
rfl::ShuffleArgs shuffle_args(const char* const* in_paths, uint64_t n_inputs, const char* out_path,
                              const rfl_shuffle_config* cfg) {
    if (!in_paths && n_inputs) rfl::invalid("null argument");
    if (!out_path || !cfg) rfl::invalid("null argument");
    rfl::ShuffleArgs a;
    for (uint64_t i = 0; i < n_inputs; ++i) a.inputs.emplace_back(in_paths[i]);
    a.out_path = out_path;
    a.c = cfg->block_rows;
    a.m = cfg->buffer_rows;
    a.seed = cfg->seed;
    a.out_chunk_rows = cfg->out_chunk_rows;
    a.out_cps = cfg->out_chunks_per_shard;
    a.out_idt = cfg->out_index_dtype;
    a.device = cfg->device;
    a.outer = cfg->join_outer != 0;
    a.rank = cfg->rank;
    a.world = cfg->world ? cfg->world : 1;
    if (cfg->out_codec > 1) rfl::invalid("run_shuffle: unknown codec");
    a.out_codec = cfg->out_codec;
    return a;
}
void fill_stats(const rfl::ShuffleResult& r, rfl_shuffle_stats* stats) {
    if (!stats) return;
    stats->peak_resident_rows = r.peak_resident_rows;
    stats->rows_written = r.rows_written;
    stats->rounds_executed = r.rounds;
    stats->input_bytes_read = r.input_bytes;
    stats->h2d_bytes = r.h2d_bytes;
    stats->d2h_bytes = r.d2h_bytes;
    stats->gpu_ms = r.gpu_ms;
    stats->send_ms = r.send_ms;
    stats->peer_bytes = r.peer_bytes;
}
}  // namespace

struct rfl_pshuf {
    rfl::RankShuffle* h;
};

rfl_status rfl_pshuf_create(const char* const* in_paths, uint64_t n_inputs, const char* out_path,
                            const rfl_shuffle_config* cfg, rfl_pshuf** out, uint64_t* n_rounds) {
    return guarded([&] {
        if (!out || !n_rounds) rfl::invalid("null argument");
        *out = new rfl_pshuf{rfl::rank_shuffle_create(shuffle_args(in_paths, n_inputs, out_path, cfg), n_rounds)};
    });
}
rfl_status rfl_pshuf_stage(rfl_pshuf* h, uint64_t round, uint64_t* send_bytes) {
    return guarded([&] {
        if (!h || !send_bytes) rfl::invalid("null argument");
        rfl::rank_shuffle_stage(h->h, round, send_bytes);
    });
}
rfl_status rfl_pshuf_recv_buffer(rfl_pshuf* h, uint64_t bytes, void** dev_ptr, void* ipc_handle, int* changed) {
    return guarded([&] {
        if (!h || !dev_ptr || !changed) rfl::invalid("null argument");
        rfl::rank_shuffle_recv(h->h, bytes, dev_ptr, ipc_handle, changed);
    });
}
rfl_status rfl_pshuf_send(rfl_pshuf* h, uint64_t round, void* const* dst) {
    return guarded([&] {
        if (!h || !dst) rfl::invalid("null argument");
        rfl::rank_shuffle_send(h->h, round, dst);
    });
}
rfl_status rfl_pshuf_emit(rfl_pshuf* h, uint64_t round, const uint64_t* recv_bytes) {
    return guarded([&] {
        if (!h || !recv_bytes) rfl::invalid("null argument");
        rfl::rank_shuffle_emit(h->h, round, recv_bytes);
    });
}
rfl_status rfl_pshuf_finish(rfl_pshuf* h, rfl_shuffle_stats* stats) {
    return guarded([&] {
        if (!h) rfl::invalid("null argument");
        fill_stats(rfl::rank_shuffle_finish(h->h), stats);
    });
}
void rfl_pshuf_destroy(rfl_pshuf* h) {
    if (h) rfl::rank_shuffle_destroy(h->h);
    delete h;
}

rfl_status rfl_ipc_open(const void* handle, int device, void** dev_ptr) {
    return guarded([&] {
        if (!handle || !dev_ptr) rfl::invalid("null argument");
        rfl::DeviceGuard g(device);
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, sizeof(h));
        rfl::cuda_ok(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    });
}
rfl_status rfl_ipc_close(void* dev_ptr, int device) {
    return guarded([&] {
        rfl::DeviceGuard g(device);
        rfl::cuda_ok(cudaIpcCloseMemHandle(dev_ptr), "cudaIpcCloseMemHandle");
    });
}

rfl_status rfl_run_shuffle(const char* const* in_paths, uint64_t n_inputs, const char* out_path,
                           const rfl_shuffle_config* cfg, rfl_shuffle_stats* stats) {
    return guarded([&] { fill_stats(rfl::run_shuffle_gpu(shuffle_args(in_paths, n_inputs, out_path, cfg)), stats); });
}

}  // extern "C"
