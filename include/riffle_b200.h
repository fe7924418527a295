/*
 * riffle_b200 — B200-native minibatch assembly and pre-shuffle for riffle
 * stores (the C++ restatement of annbatch, arXiv 2604.01949).
 *
 * This is the drop-in boundary: a flat C ABI (plain pointers and sizes, no
 * C++ or torch types) exported by paper_2604_01949_b200/_lib/libriffle_b200.so.
 * Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/proj/core).  Nothing here throws; every
 * call returns an rfl_status and leaves a thread-local message in
 * rfl_last_error().  Status codes map back to the reference exception
 * hierarchy (include/riffle/error.hpp:9-32):
 *     RFL_EINVAL -> InvalidArgument, RFL_ECORRUPT -> CorruptStore,
 *     RFL_EIO -> IoError, RFL_ECUDA / RFL_ENCCL -> device failures (new),
 *     RFL_ENOMEM -> std::bad_alloc / cudaErrorMemoryAllocation (new: the
 *     reference lets std::bad_alloc propagate).
 */
#ifndef RIFFLE_B200_H
#define RIFFLE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int rfl_status;
enum {
    RFL_OK = 0,
    RFL_EINVAL = 1,
    RFL_ECORRUPT = 2,
    RFL_EIO = 3,
    RFL_ECUDA = 4,
    RFL_ENCCL = 5,
    RFL_END = 6, /* end of epoch: BatchIterator::next() -> nullopt (loader.cpp:259) */
    RFL_ENOMEM = 7 /* host or device allocation failed */
};

/* dtype.hpp:10-16.  RFL_BF16 is an output-only dtype (new). */
enum { RFL_LAYOUT_DENSE = 0, RFL_LAYOUT_CSR = 1 };
enum { RFL_F32 = 0, RFL_F64 = 1, RFL_I32 = 2, RFL_U8 = 3, RFL_BF16 = 4, RFL_NATIVE = 255 };
enum { RFL_IDX_U32 = 0, RFL_IDX_U64 = 1 };
enum { RFL_CODEC_NONE = 0, RFL_CODEC_DEFLATE = 1 };

const char* rfl_last_error(void);
const char* rfl_version(void);
int rfl_device_count(void);
/* cudaDeviceCanAccessPeer(device, peer) (1 also for device == peer): whether a
 * kernel on `device` can store into memory of `peer` (the pre-shuffle's
 * peer-write exchange); otherwise the exchange runs as an NCCL all-to-all. */
rfl_status rfl_device_can_access_peer(int device, int peer, int* out);

/* ---------------------------------------------------------------- stores --
 * StoreReader (include/riffle/store.hpp:136-170): manifest + shard footers,
 * host side.  rfl_store_read_records reads raw (undecoded) chunk records,
 * the "missing lower-level API" of SURVEY §8b, via ShardFooter (shard.hpp:45). */
typedef struct rfl_store rfl_store;

typedef struct rfl_store_info {
    uint32_t format_version;
    uint32_t layout;
    uint64_t n_obs;
    uint64_t n_var;
    uint32_t value_dtype;
    uint32_t index_dtype; /* CSR only */
    uint64_t chunk_rows;
    uint64_t chunks_per_shard;
    uint32_t codec;
    uint32_t has_provenance;
} rfl_store_info;

rfl_status rfl_store_open(const char* root, rfl_store** out);
rfl_status rfl_store_get_info(const rfl_store* s, rfl_store_info* out);
/* byte size of chunk record `chunk` (0 if absent) */
rfl_status rfl_store_record_size(rfl_store* s, uint64_t chunk, uint64_t* nbytes);
/* pread the raw record bytes of `chunk` into dst (capacity >= record size) */
rfl_status rfl_store_read_record(rfl_store* s, uint64_t chunk, void* dst, uint64_t cap);
void rfl_store_close(rfl_store* s);

/* synth_store (include/riffle/synth.hpp:15-39, src/synth.cpp:59-143):
 * byte-identical stores for identical configs.  threads: 0 = all cores. */
typedef struct rfl_synth_config {
    uint64_t n_obs;
    uint64_t n_var;
    uint32_t layout;
    uint32_t value_dtype;
    uint32_t index_dtype;
    uint32_t codec; /* must be RFL_CODEC_NONE */
    double density;
    uint64_t seed;
    uint64_t chunk_rows;
    uint64_t chunks_per_shard;
    uint32_t threads;
    uint32_t one_hot; /* > 0: procedural one-hot dense u8 rows with this many channel planes (not in
                         the reference); 0: synth_store */
    uint32_t counts;  /* != 0: procedural counts-like csr rows (not in the reference) */
    uint32_t reserved;
} rfl_synth_config;
rfl_status rfl_synth_store(const char* path, const rfl_synth_config* cfg);

/* --------------------------------------------------------------- loader --
 * LoaderConfig (loader.hpp:12-22) plus the per-rank partition of SURVEY §8e:
 * rank k of `world` takes plan positions i == k (mod world); world == 1 is
 * exactly the reference. */
typedef struct rfl_loader_config {
    uint64_t fetch_block_rows;     /* f */
    uint64_t buffer_capacity_rows; /* B */
    uint64_t batch_rows;           /* b */
    uint64_t seed;
    uint32_t prefetch_depth; /* host read-ahead in blocks; never changes output */
    uint32_t drop_last;
    uint32_t cache_bypass; /* O_DIRECT best effort for file-streamed staging */
    uint32_t rank;
    uint32_t world;
    /* new: 1 = every rank of `world` ends the epoch after the smallest per-rank
     * batch count (plan positions are dealt round-robin, so ranks can differ by
     * a batch and a DDP step per batch would hang at epoch end); 0 = each rank
     * drains its own share (world == 1: the reference either way) */
    uint32_t even_batches;
} rfl_loader_config;

/* LoaderConfig::validate (loader.cpp:159-168) */
rfl_status rfl_loader_config_validate(const rfl_loader_config* cfg);
/* plan_epoch (loader.cpp:170-181): ceil(n_obs/f) blocks written as [start,end) */
rfl_status rfl_plan_epoch(uint64_t n_obs, const rfl_loader_config* cfg, uint64_t epoch,
                          uint64_t* starts, uint64_t* ends);

/* Index-only epoch schedule: the exact MiniBatch::global_indices stream of
 * BatchIterator::next (loader.cpp:257-306) replayed on row ids, host side. */
typedef struct rfl_schedule rfl_schedule;
rfl_status rfl_schedule_create(uint64_t n_obs, const rfl_loader_config* cfg, uint64_t epoch,
                               rfl_schedule** out);
/* writes up to batch_rows ids; RFL_END at end of epoch (idempotent) */
rfl_status rfl_schedule_next(rfl_schedule* s, uint64_t* gidx_out, uint64_t* n_rows);
/* peak_buffer_rows (loader.hpp:71-72) and blocks consumed so far */
rfl_status rfl_schedule_stats(const rfl_schedule* s, uint64_t* peak_buffer_rows,
                              uint64_t* blocks_fetched);
void rfl_schedule_destroy(rfl_schedule* s);

/* Device-side store image shared by many iterators (loader.hpp:55-57).
 *   RFL_STAGE_RESIDENT:      every chunk record copied once into HBM.
 *   RFL_STAGE_STREAM_PINNED: records kept in pinned host memory (re-encoded
 *                            losslessly where possible); the blocks fetched
 *                            for a group are pulled into HBM slots by one TMA
 *                            kernel on a side stream.
 *   RFL_STAGE_STREAM_FILE:   records pread (O_DIRECT if cache_bypass) into
 *                            pinned staging buffers, then as above. */
/*   RFL_STAGE_RESIDENT_CODED: the staging image of stream_pinned (u8 column
 *                            deltas / u16 ids / one-hot codes) held in HBM
 *                            (stores whose verbatim image exceeds HBM);
 *                            dense output of delta records is densified
 *                            straight from it, other outputs expand the
 *                            fetched blocks device-to-device. */
enum { RFL_STAGE_RESIDENT = 0, RFL_STAGE_STREAM_PINNED = 1, RFL_STAGE_STREAM_FILE = 2, RFL_STAGE_RESIDENT_CODED = 3 };
typedef struct rfl_dstore rfl_dstore;
rfl_status rfl_dstore_create(rfl_store* s, int device, uint32_t staging, rfl_dstore** out);
/* device address + byte offsets of every chunk record (resident), or of every
 * staged record of the HBM-resident coded image (resident_coded) */
rfl_status rfl_dstore_arena(const rfl_dstore* d, void** base, const uint64_t** chunk_offsets,
                            uint64_t* n_chunks);
/* Decoded record bytes of the store, and bytes of its re-encoded staging
 * image (stream_pinned / resident_coded; 0 when the records are staged verbatim). */
rfl_status rfl_dstore_bytes(const rfl_dstore* d, uint64_t* record_bytes, uint64_t* staged_bytes);
void rfl_dstore_destroy(rfl_dstore* d);

/* Output of one minibatch, on the device. */
enum { RFL_OUT_CSR = 0, RFL_OUT_DENSE = 1 };
enum { RFL_XF_NONE = 0, RFL_XF_NORMALIZE_LOG1P = 1 };
enum { RFL_DEV_TIME_KERNELS = 1 };

typedef struct rfl_device_config {
    uint32_t output;    /* RFL_OUT_CSR | RFL_OUT_DENSE (CSR stores); dense stores: DENSE */
    uint32_t out_dtype; /* RFL_NATIVE | RFL_F32 | RFL_BF16 (dense output) */
    uint32_t transform; /* RFL_XF_* (CSR -> dense only) */
    float target_sum;   /* normalize target T (default 1e4 when 0) */
    uint32_t out_slots; /* ring of output buffers (>= 1; default 2) */
    uint32_t flags;     /* RFL_DEV_TIME_KERNELS: CUDA events around each batch's kernels (counters) */
    void* stream; /* cudaStream_t for assembly; NULL = loader-owned */
    uint32_t batches_per_launch; /* consecutive batches replayed, staged and assembled together
                                    (one staging pull, one decode, one assembly launch; 0 = 1);
                                    each stays valid for out_slots further launches */
    uint32_t reserved2;
} rfl_device_config;

typedef struct rfl_batch {
    uint64_t epoch_index;
    uint64_t batch_index;
    uint64_t n_rows;
    uint64_t nnz; /* CSR output */
    uint64_t n_var;
    uint32_t layout;         /* of this output */
    uint32_t dtype;          /* element dtype of d_data */
    uint32_t index_dtype;    /* CSR output: the store's index dtype */
    uint32_t reserved;
    void* d_gidx;            /* u64[n_rows]     MiniBatch::global_indices */
    void* d_indptr;          /* u64[n_rows+1]   CSR, indptr[0] == 0 */
    void* d_indices;         /* u32|u64[nnz]    CSR */
    void* d_data;            /* CSR values [nnz] or dense [n_rows, n_var] */
    const uint64_t* h_gidx;  /* host copy of global_indices */
    void* ready_event;       /* cudaEvent_t recorded after assembly */
} rfl_batch;

typedef struct rfl_loader_counters {
    uint64_t blocks_fetched; /* LoaderCounters (loader.hpp:42-45) */
    uint64_t read_ops;       /* IoStats (store.hpp:18-42) */
    uint64_t bytes_read;
    uint64_t chunks_decoded;
    uint64_t peak_buffer_rows;
    uint64_t h2d_bytes;      /* bytes staged host->device (new) */
    uint64_t kernels_launched;
    double decode_ms;        /* RFL_DEV_TIME_KERNELS: device time of the staged-record expansion */
    double assembly_ms;      /* ... and of the batch assembly kernels, over finished batches */
} rfl_loader_counters;

typedef struct rfl_loader rfl_loader;
/* BatchIterator ctor / open_epoch (loader.hpp:58-81) */
rfl_status rfl_loader_create(rfl_dstore* d, const rfl_loader_config* cfg, uint64_t epoch,
                             const rfl_device_config* dev, rfl_loader** out);
/* BatchIterator::next (loader.cpp:257-306); RFL_END at end (idempotent).
 * Buffers stay valid until out_slots further calls. */
rfl_status rfl_loader_next(rfl_loader* l, rfl_batch* out);
/* Up to `max` further batches into out[0..*n) (*n < max only at the end of the
 * epoch; RFL_END when none is left): one C call for several batches. */
rfl_status rfl_loader_next_many(rfl_loader* l, rfl_batch* out, uint32_t max, uint32_t* n);
rfl_status rfl_loader_counters_get(const rfl_loader* l, rfl_loader_counters* out);
/* Host copy of a batch (the reference's MiniBatch, loader.hpp:35-40): waits
 * for its ready_event, then copies whichever of indptr (u64[n_rows+1]),
 * indices (index_dtype[nnz]), data (nnz or n_rows*n_var elements of dtype)
 * and gidx (u64[n_rows]) are non-NULL. */
rfl_status rfl_batch_download(const rfl_batch* b, uint64_t* h_indptr, void* h_indices, void* h_data,
                              uint64_t* h_gidx);
/* Order a consumer stream after a batch: cudaStreamWaitEvent(stream, ready_event).
 * Work the caller queues on `stream` afterwards sees the finished batch
 * (the reference returns MiniBatch by value, so reading it needs no wait). */
rfl_status rfl_batch_wait(const rfl_batch* b, void* stream);
/* Queue the copy of n_rows global row ids (u64, a batch's d_gidx) into host
 * memory h_gidx on `stream` (no host wait; pinned h_gidx makes it
 * asynchronous).  Ordered after the batch when `stream` is the loader's stream
 * or was ordered by rfl_batch_wait.  (New: the one-call form of the
 * per-step result read, instead of a torch copy.) */
rfl_status rfl_ids_download_async(const uint64_t* d_gidx, uint64_t n_rows, uint64_t* h_gidx, void* stream);
rfl_status rfl_loader_sync(rfl_loader* l);
void rfl_loader_destroy(rfl_loader* l);

/* ----------------------------------------------------- raw kernel entry --
 * The sm_100a kernels behind the loader, on caller-owned device memory, for
 * parity tests and custom pipelines.  A row reference names one source row:
 * the byte offset of its chunk record inside `arena` and its global row id
 * (row-within-chunk = gidx % chunk_rows). */
typedef struct rfl_rowref {
    uint64_t rec_off;
    uint64_t gidx;
} rfl_rowref;

typedef struct rfl_arena_desc {
    const void* base;      /* device pointer to record arena */
    uint64_t chunk_rows;
    uint64_t n_var;
    uint32_t layout;
    uint32_t value_dtype;
    uint32_t index_dtype;
    uint32_t reserved;
} rfl_arena_desc;

/* K1/K2: gather rows into a CSR block (indptr rebased to 0; warp-level indptr
 * scan + 128-bit shifted gathers).  CsrBuffer::take + batch append
 * (loader.cpp:145-154), CsrBlock::append_rows (block.cpp:92-108),
 * read_rows_csr (store.cpp:590-614).  out_gidx may be NULL. */
rfl_status rfl_csr_gather(const rfl_arena_desc* a, const rfl_rowref* d_refs, uint64_t n_rows,
                          uint64_t* d_out_indptr, void* d_out_indices, void* d_out_data,
                          uint64_t* d_out_gidx, void* stream);
/* K2 with the indptr planned on the host: d_prefix[n_rows+1] is the exclusive
 * nnz prefix of the rows (the host schedule knows every row's nnz), so no
 * device scan runs; output indices/data start at entry d_prefix[0].  d_prefix
 * may be the caller's output indptr (rebased to 0 it is the batch's indptr,
 * CsrBlock::append_rows block.cpp:92-108).  Entries are read only up to each
 * row's own nnz in its record. */
rfl_status rfl_csr_gather_prefixed(const rfl_arena_desc* a, const rfl_rowref* d_refs, uint64_t n_rows,
                                   const uint64_t* d_prefix, void* d_out_indices, void* d_out_data,
                                   uint64_t* d_out_gidx, void* stream);
/* K3: gather + densify (to_dense, block.cpp:135-146) with optional fused
 * library-size normalisation + log1p; out_dtype RFL_NATIVE|RFL_F32|RFL_BF16. */
rfl_status rfl_csr_densify(const rfl_arena_desc* a, const rfl_rowref* d_refs, uint64_t n_rows,
                           uint32_t out_dtype, uint32_t transform, float target_sum,
                           void* d_out, uint64_t* d_out_gidx, void* stream);
/* K4: dense row gather (DenseBuffer::take, loader.cpp:105-117) with optional
 * u8/f32 -> bf16 cast. */
rfl_status rfl_dense_gather(const rfl_arena_desc* a, const rfl_rowref* d_refs, uint64_t n_rows,
                            uint32_t out_dtype, void* d_out, uint64_t* d_out_gidx, void* stream);
/* K4o: the same dense row gather, reading rows staged as one-hot channel codes
 * (a resident_coded one-hot store's arena: rfl_dstore_arena; 2 bits per
 * position, n_var / 16 bytes per row, n_var % 64 == 0) -- DenseBuffer::take
 * (loader.cpp:105-117) of the rows the codes stand for; out_dtype
 * RFL_NATIVE (u8) or RFL_BF16.  Bit-identical to rfl_dense_gather over the
 * verbatim records. */
rfl_status rfl_onehot_gather(const rfl_arena_desc* a, const rfl_rowref* d_refs, uint64_t n_rows,
                             uint32_t out_dtype, void* d_out, uint64_t* d_out_gidx, void* stream);

/* K1 scan only: d_out_prefix[i] = exclusive nnz prefix of the rows,
 * d_out_prefix[n] = total nnz (the pre-shuffle's record offsets). */
rfl_status rfl_csr_scan(const rfl_arena_desc* a, const rfl_rowref* d_refs, uint64_t n_rows,
                        uint64_t* d_out_prefix, void* stream);
/* K5: rows -> consecutive encoded CSR chunk records of chunk_rows rows
 * (encode_csr_record, store.cpp:52-64), d_prefix from rfl_csr_scan; output
 * byte size = sum over records of 12 + is*(rows+1) + (is+vs)*nnz. */
rfl_status rfl_csr_pack(const rfl_arena_desc* a, const rfl_rowref* d_refs, uint64_t n_rows,
                        uint64_t chunk_rows, uint32_t out_index_dtype, const uint64_t* d_prefix,
                        void* d_out, void* stream);

/* ----------------------------------------------------------- preshuffle --
 * plan_shuffle (preshuffle.cpp:150-181).  Two-call protocol: pass NULL
 * arrays to learn n_rounds; round_len[n_rounds], ids[ceil(total/c)]. */
rfl_status rfl_plan_shuffle(uint64_t total_rows, uint64_t block_rows, uint64_t buffer_rows,
                            uint64_t seed, uint64_t* n_rounds, uint64_t* round_len,
                            uint64_t* ids);
/* Global input row of every output row of run_shuffle (index-computable:
 * round assembly in block order, permuted by stream(1+r), :336-338). */
rfl_status rfl_shuffle_order(uint64_t total_rows, uint64_t block_rows, uint64_t buffer_rows,
                             uint64_t seed, uint64_t* out_src);

/* Multi-GPU routing of round `round`: for each of its output rows
 * in output order (global output row = first_out_row + k): the global input
 * row, the source rank (block b of the round is staged by rank b mod world)
 * and the destination rank (owner of output shard s == rank (mod world)).
 * Pass NULL arrays to learn n_rows. */
rfl_status rfl_shuffle_round_routes(uint64_t total_rows, uint64_t block_rows, uint64_t buffer_rows,
                                    uint64_t seed, uint64_t out_chunk_rows, uint64_t out_chunks_per_shard,
                                    uint32_t world, uint64_t round, uint64_t* first_out_row,
                                    uint64_t* n_rows, uint64_t* src_rows, uint32_t* src_rank,
                                    uint32_t* dst_rank);

typedef struct rfl_shuffle_config {
    uint64_t block_rows;  /* c */
    uint64_t buffer_rows; /* m */
    uint64_t seed;
    uint64_t out_chunk_rows;       /* ShuffleOutputConfig (preshuffle.hpp:44-50) */
    uint64_t out_chunks_per_shard;
    int32_t out_index_dtype;       /* -1 = first input's */
    int32_t device;
    uint32_t join_outer;           /* DatasetCollection JoinMode (collection.hpp:27): 1 outer (union), 0 inner (intersection) */
    uint32_t rank;                 /* multi-GPU: this rank writes shards s == rank (mod world) */
    uint32_t world;
    uint32_t out_codec;            /* ShuffleOutputConfig::codec: 0 none, 1 deflate (zlib raw DEFLATE, codec.cpp:16-36) */
} rfl_shuffle_config;

typedef struct rfl_shuffle_stats {
    uint64_t peak_resident_rows; /* ShuffleRunStats (preshuffle.hpp:69-77) */
    uint64_t rows_written;
    uint64_t rounds_executed;
    uint64_t input_bytes_read;
    uint64_t h2d_bytes;
    uint64_t d2h_bytes;
    double gpu_ms;   /* device time of gather/permute/pack kernels */
    double send_ms;  /* multi-GPU: device time of the send-side pack kernels (local + peer messages) */
    uint64_t peer_bytes; /* multi-GPU: message bytes this rank addressed to other ranks */
} rfl_shuffle_stats;

/* run_shuffle (preshuffle.cpp:185-378) on one GPU: byte-identical output
 * store + provenance sidecar. */
rfl_status rfl_run_shuffle(const char* const* in_paths, uint64_t n_inputs, const char* out_path,
                           const rfl_shuffle_config* cfg, rfl_shuffle_stats* stats);

/* Multi-GPU pre-shuffle, one process per GPU.  Per round:
 *   rfl_pshuf_stage   stage this rank's blocks (block b of the round -> rank
 *                     b mod world), scan its rows per destination, report the
 *                     message bytes per destination rank;
 *   (caller all-gathers the world x world size matrix)
 *   rfl_pshuf_recv_buffer  receive area >= the bytes addressed to this rank,
 *                     with its CUDA IPC handle (64 bytes) for the peers;
 *   rfl_pshuf_send    one K5 pack kernel per destination writes the rows,
 *                     already encoded as a CSR record, straight into the
 *                     owner's receive buffer through peer memory (NVLink),
 *                     at dst[d] = peer base + sum of aligned sizes of lower
 *                     source ranks;
 *   (caller barrier)
 *   rfl_pshuf_emit    owner: pack the now-complete owned chunks (shards
 *                     s == rank mod world) and write them + provenance.
 * rfl_pshuf_finish flushes this rank's shards; rank 0 writes manifest.json and
 * provenance/meta.json (call after a barrier on the other ranks' finish). */
typedef struct rfl_pshuf rfl_pshuf;
rfl_status rfl_pshuf_create(const char* const* in_paths, uint64_t n_inputs, const char* out_path,
                            const rfl_shuffle_config* cfg, rfl_pshuf** out, uint64_t* n_rounds);
rfl_status rfl_pshuf_stage(rfl_pshuf* h, uint64_t round, uint64_t* send_bytes);
rfl_status rfl_pshuf_recv_buffer(rfl_pshuf* h, uint64_t bytes, void** dev_ptr, void* ipc_handle, int* changed);
rfl_status rfl_pshuf_send(rfl_pshuf* h, uint64_t round, void* const* dst);
rfl_status rfl_pshuf_emit(rfl_pshuf* h, uint64_t round, const uint64_t* recv_bytes);
rfl_status rfl_pshuf_finish(rfl_pshuf* h, rfl_shuffle_stats* stats);
void rfl_pshuf_destroy(rfl_pshuf* h);
/* CUDA IPC helpers for the receive buffers of peer processes */
rfl_status rfl_ipc_open(const void* ipc_handle, int device, void** dev_ptr);
rfl_status rfl_ipc_close(void* dev_ptr, int device);

#ifdef __cplusplus
}
#endif
#endif /* RIFFLE_B200_H */
