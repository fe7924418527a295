/*
 * ORACLE / TEST INFRASTRUCTURE ONLY — a plain-C restatement of the reference's
 * integer algorithms on the hot path.  It is the checker for the product's
 * host schedule and GPU kernels; nothing in paper_2604_01949_b200/ links it.
 * Parity of this restatement is pinned against the compiled reference
 * (oracle/_ref/libriffle_ref.so) and the golden vectors in tests/golden/.
 *
 * Each function cites the reference file:line it restates
 * (paths relative to /root/reference/proj/core).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- rng.hpp:12-17  mix64 (splitmix64 finalizer) ---------------------------- */
uint64_t orc_mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

typedef struct {
    uint64_t root;
    uint64_t s[4];
} orc_rng;

/* rng.hpp:30-36  seeding via splitmix */
static orc_rng rng_make(uint64_t seed) {
    orc_rng r;
    r.root = seed;
    uint64_t sm = seed;
    for (int i = 0; i < 4; ++i) {
        sm += 0x9e3779b97f4a7c15ull;
        r.s[i] = orc_mix64(sm);
    }
    return r;
}

/* rng.hpp:39-41  stream(tag) — pure derivation from the root seed */
static orc_rng rng_stream(const orc_rng* r, uint64_t tag) {
    return rng_make(orc_mix64(r->root ^ orc_mix64(tag + 0x1d8e4e27c47d124full)));
}

static inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

/* rng.hpp:45-55  xoshiro256** next */
static uint64_t rng_next(orc_rng* r) {
    uint64_t* s = r->s;
    const uint64_t result = rotl(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return result;
}

/* rng.hpp:58-64  bounded: rejection below (0-n)%n */
static uint64_t rng_bounded(orc_rng* r, uint64_t n) {
    const uint64_t threshold = (0 - n) % n;
    for (;;) {
        const uint64_t x = rng_next(r);
        if (x >= threshold) return x % n;
    }
}

/* rng.hpp:73-81  Fisher-Yates from the top, j = bounded(i) */
static void rng_shuffle_u64(orc_rng* r, uint64_t* a, uint64_t n) {
    for (uint64_t i = n; i > 1; --i) {
        const uint64_t j = rng_bounded(r, i);
        if (j != i - 1) {
            uint64_t t = a[i - 1];
            a[i - 1] = a[j];
            a[j] = t;
        }
    }
}

/* Exposed for tests: raw draws from Rng(seed) or Rng(seed).stream(tag). */
void orc_rng_next(uint64_t seed, uint64_t tag, int use_tag, uint64_t n, uint64_t* out) {
    orc_rng base = rng_make(seed);
    orc_rng r = use_tag ? rng_stream(&base, tag) : base;
    for (uint64_t i = 0; i < n; ++i) out[i] = rng_next(&r);
}
void orc_rng_bounded(uint64_t seed, uint64_t tag, int use_tag, uint64_t bound, uint64_t n,
                     uint64_t* out) {
    orc_rng base = rng_make(seed);
    orc_rng r = use_tag ? rng_stream(&base, tag) : base;
    for (uint64_t i = 0; i < n; ++i) out[i] = rng_bounded(&r, bound);
}

/* ---- loader.cpp:170-181  plan_epoch: f-row blocks, shuffled by stream(2e) -------- */
/* Block ids are shuffled; block i covers [i*f, min(n,(i+1)*f)).  out_ids has
 * ceil(n/f) entries.  (Shuffling ids is equivalent to shuffling the RowRange
 * vector, since the swap sequence depends only on the length.) */
void orc_plan_epoch_ids(uint64_t n_obs, uint64_t f, uint64_t seed, uint64_t epoch,
                        uint64_t* out_ids) {
    const uint64_t nb = (n_obs + f - 1) / f;
    for (uint64_t i = 0; i < nb; ++i) out_ids[i] = i;
    orc_rng base = rng_make(seed);
    orc_rng r = rng_stream(&base, 2 * epoch);
    rng_shuffle_u64(&r, out_ids, nb);
}

/* ---- loader.cpp:257-306 (+183-227)  BatchIterator, replayed on row ids ---------
 * The sampler's draws depend only on buffer occupancy, so replaying the
 * swap-with-last buffer (DenseBuffer::take, loader.cpp:105-117; CsrBuffer::take
 * has identical slot semantics, :145-154) on global row ids reproduces the
 * exact MiniBatch::global_indices stream.
 *
 * Per-rank sharding (new, absent from the reference): rank k of W
 * takes plan positions i ≡ k (mod W); the sampler is stream(2e+1) when W == 1
 * (identical to the reference) and stream(2e+1).stream(k) otherwise.
 *
 * Outputs: out_gidx (all emitted rows in order, capacity n_obs), out_batch_len
 * (capacity ceil(n_obs/b)+1), counts, peak occupancy, blocks consumed.
 * Returns number of batches. */
int64_t orc_replay_epoch(uint64_t n_obs, uint64_t f, uint64_t B, uint64_t b, uint64_t seed,
                         uint64_t epoch, int drop_last, uint64_t rank, uint64_t world,
                         uint64_t* out_gidx, uint64_t* out_batch_len, uint64_t* out_rows,
                         uint64_t* out_peak, uint64_t* out_blocks) {
    if (f < 1 || B < f || b < 1 || b > B || world < 1 || rank >= world) return -1;
    const uint64_t nb_all = (n_obs + f - 1) / f;
    uint64_t* ids = (uint64_t*)malloc((nb_all ? nb_all : 1) * sizeof(uint64_t));
    orc_plan_epoch_ids(n_obs, f, seed, epoch, ids);
    /* this rank's sub-plan */
    uint64_t nb = 0;
    for (uint64_t i = rank; i < nb_all; i += world) ids[nb++] = ids[i];

    orc_rng base = rng_make(seed);
    orc_rng smp = rng_stream(&base, 2 * epoch + 1);
    if (world > 1) smp = rng_stream(&smp, rank);

    uint64_t* buf = (uint64_t*)malloc((B + f + 1) * sizeof(uint64_t));
    uint64_t occ = 0, next_block = 0, peak = 0, emitted = 0;
    int64_t n_batches = 0;
    int done = 0;

#define CONSUME()                                                              \
    do {                                                                       \
        const uint64_t s = ids[next_block] * f;                                \
        const uint64_t e = s + f < n_obs ? s + f : n_obs;                      \
        for (uint64_t g = s; g < e; ++g) buf[occ++] = g;                       \
        ++next_block;                                                          \
        if (occ > peak) peak = occ;                                            \
    } while (0)

    /* initial fill (loader.cpp:261-266) */
    while (occ < B && next_block < nb) CONSUME();
    while (!done) {
        uint64_t collected = 0;
        const uint64_t batch_start = emitted;
        while (collected < b) {
            if (occ == 0) {
                if (next_block >= nb) break;
                CONSUME();
                continue;
            }
            const uint64_t j = rng_bounded(&smp, occ);
            out_gidx[emitted++] = buf[j];
            buf[j] = buf[occ - 1];
            --occ;
            ++collected;
            /* refill (loader.cpp:219-226) */
            while (occ < B - f && next_block < nb) CONSUME();
        }
        if (collected == 0 || (collected < b && drop_last)) {
            emitted = batch_start;
            done = 1;
            break;
        }
        out_batch_len[n_batches++] = collected;
    }
#undef CONSUME
    *out_rows = emitted;
    *out_peak = peak;
    *out_blocks = next_block;
    free(buf);
    free(ids);
    return n_batches;
}

/* ---- preshuffle.cpp:150-181  plan_shuffle ------------------------------------- */
/* ids permuted by Rng(seed).stream(0); greedy rounds of <= m rows.
 * out_round_len capacity: number of blocks.  Returns the number of rounds. */
int64_t orc_plan_shuffle(uint64_t total, uint64_t c, uint64_t m, uint64_t seed,
                         uint64_t* out_round_len, uint64_t* out_ids) {
    if (c == 0 || m < c) return -1;
    const uint64_t nb = (total + c - 1) / c;
    for (uint64_t i = 0; i < nb; ++i) out_ids[i] = i;
    orc_rng base = rng_make(seed);
    orc_rng r = rng_stream(&base, 0);
    rng_shuffle_u64(&r, out_ids, nb);
    int64_t nr = 0;
    uint64_t cur_blocks = 0, cur_rows = 0;
    for (uint64_t i = 0; i < nb; ++i) {
        const uint64_t s = out_ids[i] * c;
        const uint64_t rows = (s + c < total ? s + c : total) - s;
        if (cur_blocks > 0 && cur_rows + rows > m) {
            out_round_len[nr++] = cur_blocks;
            cur_blocks = 0;
            cur_rows = 0;
        }
        ++cur_blocks;
        cur_rows += rows;
    }
    if (cur_blocks > 0) out_round_len[nr++] = cur_blocks;
    return nr;
}

/* ---- preshuffle.cpp:234-368  run_shuffle output order ---------------------------
 * Round r's assembly is its blocks' rows in block order; output row k of the
 * round is assembly[perm[k]] with perm = iota shuffled by Rng(seed).stream(1+r)
 * (:336-338).  The output store is the concatenation over rounds, so output
 * row o names global input row out_src[o]. */
int orc_shuffle_order(uint64_t total, uint64_t c, uint64_t m, uint64_t seed, uint64_t* out_src) {
    if (c == 0 || m < c) return -1;
    const uint64_t nb = (total + c - 1) / c;
    uint64_t* ids = (uint64_t*)malloc((nb ? nb : 1) * sizeof(uint64_t));
    uint64_t* lens = (uint64_t*)malloc((nb ? nb : 1) * sizeof(uint64_t));
    const int64_t nr = orc_plan_shuffle(total, c, m, seed, lens, ids);
    uint64_t* assembly = (uint64_t*)malloc((m + 1) * sizeof(uint64_t));
    uint64_t* perm = (uint64_t*)malloc((m + 1) * sizeof(uint64_t));
    orc_rng base = rng_make(seed);
    uint64_t bi = 0, o = 0;
    for (int64_t r = 0; r < nr; ++r) {
        uint64_t rows = 0;
        for (uint64_t q = 0; q < lens[r]; ++q, ++bi) {
            const uint64_t s = ids[bi] * c;
            const uint64_t e = s + c < total ? s + c : total;
            for (uint64_t g = s; g < e; ++g) assembly[rows++] = g;
        }
        for (uint64_t k = 0; k < rows; ++k) perm[k] = k;
        orc_rng pr = rng_stream(&base, 1 + (uint64_t)r);
        rng_shuffle_u64(&pr, perm, rows);
        for (uint64_t k = 0; k < rows; ++k) out_src[o++] = assembly[perm[k]];
    }
    free(perm);
    free(assembly);
    free(lens);
    free(ids);
    return 0;
}

/* tests/test_support.hpp:57-66  fnv1a64 (stream hash used for golden checks) */
uint64_t orc_fnv1a64(const void* data, uint64_t n, uint64_t h) {
    const unsigned char* p = (const unsigned char*)data;
    for (uint64_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ull;
    }
    return h;
}
