/* =====================================================================================
 * DCI ORACLE — plain, slow, obviously-correct CPU reference for the DCI hot path (C11).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product path
 * (paper_2503_01281_b200/) never links, imports or calls it, and this file shares no
 * code, header, table or constant generator with the CUDA path.
 *
 * Paper: "DCI: A Coordinated Allocation and Filling Workload-Aware Dual-Cache
 * Allocation GNN Inference Acceleration System", arXiv 2503.01281.
 * Citation key: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n;
 * O-k / Ck = the oracle definition / ambiguity-ledger rows of SURVEY.md §8(c), restated
 * (with every reading we took) in DESIGN.md §3.
 *
 * Every function below follows its definition step by step. There is no blocking,
 * fusion or reordering.  Library primitives used as single steps: qsort (with total-order
 * comparators, so the result is the unique sorted order; a position tie-break makes the
 * "stable" sorts of the definitions exact), unsigned __int128 (gcc).
 *
 * Parity status: every function is pinned by a `-m "not gpu"` test in
 * tests/test_oracle_*.py against something other than itself.
 * ===================================================================================== */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Status codes (mirror nothing; the product library has its own enum). */
enum { OR_OK = 0, OR_EINVAL = -1, OR_ESEED = -2, OR_EDUP = -3, OR_ECAP = -4, OR_ENOMEM = -5 };

/* -------------------------------------------------------------------------------------
 * O-1  Philox4x32-10 (Salmon et al., "Parallel random numbers: as easy as 1, 2, 3",
 * SC'11; Random123).  BASELINE.json north_star: "a counter-based Philox draw keyed by
 * (seed, layer, node, slot)".  One round:
 *   (hi0, lo0) = M0 * c0 ; (hi1, lo1) = M1 * c2
 *   c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)
 * key schedule between rounds: k0 += W0, k1 += W1.  Ten rounds.
 * ------------------------------------------------------------------------------------- */
void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
    uint32_t c[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]};
    uint32_t k[2] = {key_in[0], key_in[1]};
    for (int round = 0; round < 10; ++round) {
        if (round > 0) {
            k[0] += W0;
            k[1] += W1;
        }
        uint64_t p0 = (uint64_t)M0 * (uint64_t)c[0];
        uint64_t p1 = (uint64_t)M1 * (uint64_t)c[2];
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c[1] ^ k[0];
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c[3] ^ k[1];
        uint32_t n3 = lo0;
        c[0] = n0;
        c[1] = n1;
        c[2] = n2;
        c[3] = n3;
    }
    out[0] = c[0];
    out[1] = c[1];
    out[2] = c[2];
    out[3] = c[3];
}

/* O-2  u(seed, pass, hop, v, i) = Philox(ctr=(v, i, hop, pass), key=(seed_lo, seed_hi));
 * u = (uint64)r.y << 32 | r.x.  pass 0 = inference, pass 1 = presample (C4). */
uint64_t oracle_draw(uint64_t seed, uint32_t pass, uint32_t hop, uint32_t v, uint32_t i) {
    uint32_t ctr[4] = {v, i, hop, pass};
    uint32_t key[2] = {(uint32_t)(seed & 0xFFFFFFFFu), (uint32_t)(seed >> 32)};
    uint32_t r[4];
    oracle_philox4x32_10(ctr, key, r);
    return ((uint64_t)r[1] << 32) | (uint64_t)r[0];
}

/* O-3  bounded(u, m) = floor(u * m / 2^64), 1 <= m <= 2^32 (multiply-high, no rejection). */
uint64_t oracle_bounded(uint64_t u, uint64_t m) {
    unsigned __int128 prod = (unsigned __int128)u * (unsigned __int128)m;
    return (uint64_t)(prod >> 64);
}

/* O-4 (Floyd part) given the k bounded draws t[i] in [0, deg-k+i], return the chosen
 * ranks in draw order (NOT sorted).  Robert Floyd's algorithm (Bentley & Floyd, CACM
 * 1987, "A sample of brilliance"): for j = deg-k .. deg-1: t = uniform[0, j];
 * if t already chosen then choose j else choose t. */
void oracle_floyd_from_draws(int64_t deg, int32_t k, const uint64_t* t, int64_t* chosen) {
    for (int32_t i = 0; i < k; ++i) {
        int64_t j = deg - k + i;
        int64_t ti = (int64_t)t[i];
        int seen = 0;
        for (int32_t m = 0; m < i; ++m)
            if (chosen[m] == ti) seen = 1;
        chosen[i] = seen ? j : ti;
    }
}

static int cmp_i64_asc(const void* a, const void* b) {
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return (x > y) - (x < y);
}

/* O-4  select for (v, hop h): f = fanout of this hop, k = min(deg, f) (C1: without
 * replacement).  deg <= f: ranks 0..deg-1.  Else Floyd with t_i = bounded(u(..., i), j+1),
 * j = deg-k+i.  Output sorted ascending (canonical order, O-4).  Returns k. */
int32_t oracle_select(uint64_t seed, uint32_t pass, uint32_t hop, int32_t v, int64_t deg, int32_t f,
                      int64_t* ranks_out) {
    if (deg <= 0) return 0;
    if (deg <= f) {
        for (int64_t r = 0; r < deg; ++r) ranks_out[r] = r;
        return (int32_t)deg;
    }
    int32_t k = f;
    uint64_t* t = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)k);
    for (int32_t i = 0; i < k; ++i) {
        int64_t j = deg - k + i;
        uint64_t u = oracle_draw(seed, pass, hop, (uint32_t)v, (uint32_t)i);
        t[i] = oracle_bounded(u, (uint64_t)(j + 1));
    }
    oracle_floyd_from_draws(deg, k, t, ranks_out);
    free(t);
    qsort(ranks_out, (size_t)k, sizeof(int64_t), cmp_i64_asc);
    return k;
}

/* A textbook open-addressing hash map node id -> local id (linear probing), used as the
 * "map" of O-6.  Capacity is a power of two at least twice the number of keys. */
typedef struct {
    int32_t* keys;
    int32_t* vals;
    uint64_t mask;
} IdMap;

static int idmap_init(IdMap* m, int64_t max_keys) {
    uint64_t cap = 16;
    while (cap < (uint64_t)(2 * max_keys + 2)) cap <<= 1;
    m->keys = (int32_t*)malloc(sizeof(int32_t) * cap);
    m->vals = (int32_t*)malloc(sizeof(int32_t) * cap);
    m->mask = cap - 1;
    if (!m->keys || !m->vals) return 0;
    for (uint64_t i = 0; i < cap; ++i) m->keys[i] = -1;
    return 1;
}

static void idmap_free(IdMap* m) {
    free(m->keys);
    free(m->vals);
}

/* returns the slot of key (key present iff m->keys[slot] == key) */
static uint64_t idmap_slot(const IdMap* m, int32_t key) {
    uint64_t s = ((uint64_t)(uint32_t)key * 2654435761u) & m->mask;
    while (m->keys[s] != -1 && m->keys[s] != key) s = (s + 1) & m->mask;
    return s;
}

/* -------------------------------------------------------------------------------------
 * O-5 / O-6  one mini-batch of L-hop uniform neighbour sampling with DGL block
 * semantics (C2: every node of F_h is re-sampled at hop h; F_{h+1} = F_h ++ new),
 * DGL fan-out order (C3: hop h uses fanouts[L-1-h]), first-occurrence relabelling in
 * (dst-major, rank-ascending) order (C6).  P:116-117; Table I P:89-99.
 *
 * Element access (O-5): nbr(v, r) = indices_cur[indptr[v] + r]; it is an adjacency-cache
 * hit iff r < cached_len[v] (C16).  cached_len == NULL means no cache.
 * edge_counts != NULL: presample counting, edge_counts[indptr[v]+r] += 1 (O-8, C8).
 *
 * Outputs: F_out[0..|F_L|), sizes_out[0..L] = |F_h|, per hop h: bptr_out[h][0..|F_h|],
 * bsrc_out[h][0..sum k).  adj_hm[0] += hits, adj_hm[1] += misses.
 * ------------------------------------------------------------------------------------- */
int32_t oracle_sample_batch(int64_t N, const int64_t* indptr, const int32_t* indices_cur,
                            const int32_t* cached_len, const int32_t* seeds, int32_t B,
                            const int32_t* fanouts, int32_t L, uint64_t seed, uint32_t pass,
                            int32_t* F_out, int64_t F_cap, int64_t* sizes_out, int32_t** bptr_out,
                            int32_t** bsrc_out, const int64_t* bsrc_caps, uint64_t* adj_hm,
                            int32_t* edge_counts) {
    if (B < 0 || L < 1) return OR_EINVAL;
    int32_t fmax = 1;
    for (int32_t h = 0; h < L; ++h) {
        if (fanouts[h] < 1) return OR_EINVAL;
        if (fanouts[h] > fmax) fmax = fanouts[h];
    }
    /* F is built in F_out itself (capacity F_cap); map: node id -> local id */
    IdMap map;
    if (!idmap_init(&map, F_cap > B ? F_cap : B)) {
        idmap_free(&map);
        return OR_ENOMEM;
    }
    int64_t nF = 0;
    int32_t rc = OR_OK;
    /* O-6: validate seeds (range, duplicates: C22) */
    for (int32_t i = 0; i < B && rc == OR_OK; ++i) {
        int32_t s = seeds[i];
        if (s < 0 || (int64_t)s >= N) {
            rc = OR_ESEED;
            break;
        }
        uint64_t slot = idmap_slot(&map, s);
        if (map.keys[slot] == s) {
            rc = OR_EDUP;
            break;
        }
        if (nF >= F_cap) {
            rc = OR_ECAP;
            break;
        }
        map.keys[slot] = s;
        map.vals[slot] = (int32_t)nF;
        F_out[nF++] = s;
    }
    int64_t* ranks = (int64_t*)malloc(sizeof(int64_t) * (size_t)fmax);
    if (rc == OR_OK) sizes_out[0] = nF;
    for (int32_t h = 0; h < L && rc == OR_OK; ++h) {
        int32_t f = fanouts[L - 1 - h];
        int64_t n_h = nF; /* frozen frontier size */
        int32_t* bptr = bptr_out[h];
        int32_t* bsrc = bsrc_out[h];
        int64_t nsrc = 0;
        bptr[0] = 0;
        for (int64_t d = 0; d < n_h && rc == OR_OK; ++d) {
            int32_t v = F_out[d];
            int64_t deg = indptr[v + 1] - indptr[v];
            int32_t k = oracle_select(seed, pass, (uint32_t)h, v, deg, f, ranks);
            for (int32_t s = 0; s < k; ++s) {
                int64_t r = ranks[s];
                int32_t u = indices_cur[indptr[v] + r];
                if (cached_len != NULL && r < (int64_t)cached_len[v])
                    adj_hm[0] += 1;
                else
                    adj_hm[1] += 1;
                if (edge_counts != NULL) edge_counts[indptr[v] + r] += 1;
                uint64_t slot = idmap_slot(&map, u);
                int32_t local;
                if (map.keys[slot] != u) {
                    if (nF >= F_cap) {
                        rc = OR_ECAP;
                        break;
                    }
                    local = (int32_t)nF;
                    map.keys[slot] = u;
                    map.vals[slot] = local;
                    F_out[nF++] = u;
                } else {
                    local = map.vals[slot];
                }
                if (nsrc >= bsrc_caps[h]) {
                    rc = OR_ECAP;
                    break;
                }
                bsrc[nsrc++] = local;
            }
            bptr[d + 1] = (int32_t)nsrc;
        }
        if (rc == OR_OK) sizes_out[h + 1] = nF;
    }
    free(ranks);
    idmap_free(&map);
    return rc;
}

/* O-7  feature gather: X[i][:] = feats[F[i]][:]; a feature-cache hit iff
 * slot_of[F[i]] >= 0.  slot_of == NULL: no cache (all misses); X == NULL: count only. */
int32_t oracle_gather(const int32_t* F, int64_t nF, const float* feats, int32_t D,
                      const int32_t* slot_of, float* X, int64_t ldx, uint64_t* feat_hm) {
    for (int64_t i = 0; i < nF; ++i) {
        int32_t v = F[i];
        if (X != NULL)
            for (int32_t c = 0; c < D; ++c) X[i * ldx + c] = feats[(int64_t)v * D + c];
        if (slot_of != NULL && slot_of[v] >= 0)
            feat_hm[0] += 1;
        else
            feat_hm[1] += 1;
    }
    return OR_OK;
}

/* O-8  presample: for each presample batch b run O-6 with
 * pass 1 on the ORIGINAL CSC and no cache; edge_counts[indptr[v]+r] += 1 per sampled
 * (v, r) per hop (C8); node_visits[u] += 1 per u in F_L (C7).  Times are measured by the
 * GPU; the oracle does not produce them.  seeds: num_seeds ids cut into batches of B
 * (last batch ragged).  Counts accumulate into the caller's arrays. */
int32_t oracle_presample(int64_t N, const int64_t* indptr, const int32_t* indices,
                         const int32_t* seeds, int64_t num_seeds, int32_t B, const int32_t* fanouts,
                         int32_t L, uint64_t seed, int32_t* node_visits, int32_t* edge_counts) {
    if (B < 1 || L < 1 || L > 8) return OR_EINVAL;
    int32_t rc = OR_OK;
    for (int64_t b0 = 0; b0 < num_seeds && rc == OR_OK; b0 += B) {
        int32_t nb = (int32_t)(num_seeds - b0 < B ? num_seeds - b0 : B);
        /* worst-case capacities: |F_h| <= min(N, nb * prod(1+f)) */
        int64_t cap[9];
        cap[0] = nb;
        for (int32_t h = 0; h < L; ++h) {
            int64_t c = cap[h] * (1 + fanouts[L - 1 - h]);
            cap[h + 1] = c < N ? c : N;
        }
        int32_t* F = (int32_t*)malloc(sizeof(int32_t) * (size_t)(cap[L] > 0 ? cap[L] : 1));
        int64_t sizes[9];
        int32_t* bp[8];
        int32_t* bs[8];
        int64_t bcap[8];
        for (int32_t h = 0; h < L; ++h) {
            bp[h] = (int32_t*)malloc(sizeof(int32_t) * (size_t)(cap[h] + 1));
            bcap[h] = cap[h] * fanouts[L - 1 - h];
            bs[h] = (int32_t*)malloc(sizeof(int32_t) * (size_t)(bcap[h] > 0 ? bcap[h] : 1));
        }
        uint64_t hm[2] = {0, 0};
        rc = oracle_sample_batch(N, indptr, indices, NULL, seeds + b0, nb, fanouts, L, seed, 1, F, cap[L], sizes,
                                 bp, bs, bcap, hm, edge_counts);
        if (rc == OR_OK)
            for (int64_t i = 0; i < sizes[L]; ++i) node_visits[F[i]] += 1;
        free(F);
        for (int32_t h = 0; h < L; ++h) {
            free(bp[h]);
            free(bs[h]);
        }
    }
    return rc;
}

/* O-10  Eq. (1): C_adj = floor(C * S / (S + F)), C_feat = C - C_adj,
 * S = sum t_sample, F = sum t_feature (integer ns, C19).  Explicit ratio (num/den,
 * den > 0) replaces S/(S+F) (C20).  S + F == 0 -> C_adj = floor(C/2). */
int32_t oracle_allocate(uint64_t C, const uint64_t* t_sample, const uint64_t* t_feature, int32_t n,
                        int64_t ratio_num, int64_t ratio_den, uint64_t* c_adj, uint64_t* c_feat) {
    unsigned __int128 adj;
    if (ratio_den > 0) {
        if (ratio_num < 0 || ratio_num > ratio_den) return OR_EINVAL;
        adj = (unsigned __int128)C * (unsigned __int128)ratio_num / (unsigned __int128)ratio_den;
    } else {
        unsigned __int128 S = 0, Fs = 0;
        for (int32_t k = 0; k < n; ++k) {
            S += t_sample[k];
            Fs += t_feature[k];
        }
        if (S + Fs == 0)
            adj = C / 2;
        else
            adj = (unsigned __int128)C * S / (S + Fs);
    }
    *c_adj = (uint64_t)adj;
    *c_feat = C - (uint64_t)adj;
    return OR_OK;
}

/* key/id pairs sorted by key descending, id ascending (a total order: ids are distinct) */
typedef struct {
    int64_t key;
    int64_t id;
} KeyId;

static int cmp_key_desc_id_asc(const void* a, const void* b) {
    const KeyId* x = (const KeyId*)a;
    const KeyId* y = (const KeyId*)b;
    if (x->key != y->key) return x->key > y->key ? -1 : 1;
    return (x->id > y->id) - (x->id < y->id);
}

static int cmp_i32_asc(const void* a, const void* b) {
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

/* O-11  feature fill (C10-C12): cap rows; admit the first `cap` nodes of
 * sort(nodes, key = (visits desc, id asc)); slots in ascending id.  When the
 * above-average set fits, this is exactly the paper's "greater than the average, then
 * backfill" set (C11).  slot_of_out[v] = slot or -1; admitted_out[j] = node in slot j. */
int64_t oracle_feat_fill(int64_t N, const int32_t* visits, int64_t cap, int32_t* slot_of_out,
                         int32_t* admitted_out) {
    if (cap > N) cap = N;
    if (cap < 0) cap = 0;
    KeyId* order = (KeyId*)malloc(sizeof(KeyId) * (size_t)(N > 0 ? N : 1));
    for (int64_t v = 0; v < N; ++v) {
        order[v].key = visits[v];
        order[v].id = v;
    }
    qsort(order, (size_t)N, sizeof(KeyId), cmp_key_desc_id_asc);
    int32_t* admitted = (int32_t*)malloc(sizeof(int32_t) * (size_t)(cap > 0 ? cap : 1));
    for (int64_t j = 0; j < cap; ++j) admitted[j] = (int32_t)order[j].id;
    qsort(admitted, (size_t)cap, sizeof(int32_t), cmp_i32_asc);
    for (int64_t v = 0; v < N; ++v) slot_of_out[v] = -1;
    for (int64_t j = 0; j < cap; ++j) {
        slot_of_out[admitted[j]] = (int32_t)j;
        if (admitted_out) admitted_out[j] = admitted[j];
    }
    free(order);
    free(admitted);
    return cap;
}

/* O-12  adjacency fill, Algorithm 1 with Fig. 6:
 *  level-2 (per node, C13/C14): perm_v = stable sort of 0..deg-1 by count desc
 *          (= sort by (count desc, position asc));
 *          indices_R[indptr[v]+p] = indices[indptr[v]+perm_v[p]]  (always applied, C17)
 *  cap_e = floor(C_adj / 4) 4-byte elements (C18).
 *  whole-fit (Alg. 1 lines 1-3): E <= cap_e -> cached_len = deg for every node.
 *  else level-1 (C13): walk nodes in sort(key = (total desc, id asc)), rem = cap_e,
 *          cached_len[v] = min(deg_v, rem), rem -= cached_len[v] (C15: node-major prefix,
 *          last node partial).
 *  acache = concatenation of the cached prefixes of indices_R in that walk order;
 *  cache_off[v] = running offset (in elements).  Returns the number of cached elements. */
int64_t oracle_adj_fill(int64_t N, int64_t E, const int64_t* indptr, const int32_t* indices,
                        const int32_t* counts, uint64_t c_adj_bytes, int32_t* indices_R,
                        int32_t* cached_len, int64_t* cache_off, int32_t* acache) {
    /* level 2: per-node stable sort of elements by access count, descending */
    int64_t maxdeg = 1;
    for (int64_t v = 0; v < N; ++v)
        if (indptr[v + 1] - indptr[v] > maxdeg) maxdeg = indptr[v + 1] - indptr[v];
    KeyId* perm = (KeyId*)malloc(sizeof(KeyId) * (size_t)maxdeg);
    for (int64_t v = 0; v < N; ++v) {
        int64_t a = indptr[v], deg = indptr[v + 1] - indptr[v];
        for (int64_t p = 0; p < deg; ++p) {
            perm[p].key = counts[a + p];
            perm[p].id = p;
        }
        qsort(perm, (size_t)deg, sizeof(KeyId), cmp_key_desc_id_asc);
        for (int64_t p = 0; p < deg; ++p) indices_R[a + p] = indices[a + perm[p].id];
    }
    free(perm);
    uint64_t cap_e = c_adj_bytes / 4;
    /* node totals (Alg. 1 lines 5-8) and level-1 order (Alg. 1 line 9; ties by id) */
    KeyId* order = (KeyId*)malloc(sizeof(KeyId) * (size_t)(N > 0 ? N : 1));
    for (int64_t v = 0; v < N; ++v) {
        int64_t total = 0;
        for (int64_t e = indptr[v]; e < indptr[v + 1]; ++e) total += counts[e];
        order[v].key = total;
        order[v].id = v;
    }
    qsort(order, (size_t)N, sizeof(KeyId), cmp_key_desc_id_asc);
    for (int64_t v = 0; v < N; ++v) {
        cached_len[v] = 0;
        cache_off[v] = 0;
    }
    int64_t off = 0;
    uint64_t rem = (uint64_t)E <= cap_e ? (uint64_t)E : cap_e; /* whole-fit: cache everything */
    for (int64_t i = 0; i < N; ++i) {
        int64_t v = order[i].id;
        int64_t deg = indptr[v + 1] - indptr[v];
        int64_t take = (uint64_t)deg < rem ? deg : (int64_t)rem;
        cached_len[v] = (int32_t)take;
        cache_off[v] = off;
        for (int64_t p = 0; p < take; ++p) acache[off + p] = indices_R[indptr[v] + p];
        off += take;
        rem -= (uint64_t)take;
    }
    free(order);
    return off;
}

/* O-13 mean / sum aggregator over one sampled block (P:107
 * "aggregating" the neighbours' features; BJ north_star's optional consumer; reading C23):
 * op = 0: H[d][c] = (1 / k_d) * sum_{j = bptr[d]}^{bptr[d+1]-1} X[bsrc[j]][c]
 *         ("avg", GCN in Table III), k_d = 0 -> 0;
 * op = 1: the sum (GraphSAGE's "sum" there).  Accumulated in double. */
void oracle_block_aggregate(const int32_t* bptr, const int32_t* bsrc, int64_t n_dst, const float* X,
                            int64_t ldx, int32_t D, int32_t op, double* H) {
    for (int64_t d = 0; d < n_dst; ++d) {
        int64_t k = bptr[d + 1] - bptr[d];
        for (int32_t c = 0; c < D; ++c) {
            double acc = 0.0;
            for (int64_t j = bptr[d]; j < bptr[d + 1]; ++j) acc += (double)X[(int64_t)bsrc[j] * ldx + c];
            if (op == 1)
                H[d * D + c] = acc;
            else
                H[d * D + c] = k > 0 ? acc / (double)k : 0.0;
        }
    }
}

/* O-14 DUCATI-style unified-budget knapsack fill, as simplified by SPEC
 * (S:496-504): items are feature rows (value = visits * cost_feat, size = row_bytes) and
 * adjacency elements (value = count * cost_adj, size = 4 B); sort by value density
 * (value / size) descending, ties by kind (feature first) then id (node id / CSC position);
 * admit every item that still fits the remaining budget, in that order.  Admitted adjacency
 * elements are regrouped per node by the level-2 order (count desc, position asc): the
 * cached prefix of node v has length = #admitted elements of v ("re-sorting admitted
 * elements within each node by count so the prefix hit rule still applies").
 * Outputs: slot_of[N] (admitted rows, slots in ascending id), cached_len[N]; returns bytes used. */
typedef struct {
    double density;
    int32_t kind; /* 0 feature row, 1 adjacency element */
    int64_t id;   /* node id or CSC position */
    int64_t size;
} Item;

static int cmp_item(const void* a, const void* b) {
    const Item* x = (const Item*)a;
    const Item* y = (const Item*)b;
    if (x->density != y->density) return x->density > y->density ? -1 : 1;
    if (x->kind != y->kind) return x->kind < y->kind ? -1 : 1;
    return (x->id > y->id) - (x->id < y->id);
}

uint64_t oracle_knapsack_fill(int64_t N, int64_t E, const int64_t* indptr, const int32_t* visits,
                              const int32_t* counts, uint64_t C, int64_t row_bytes, double cost_feat,
                              double cost_adj, int32_t* slot_of, int32_t* cached_len) {
    Item* items = (Item*)malloc(sizeof(Item) * (size_t)(N + E > 0 ? N + E : 1));
    int64_t n = 0;
    for (int64_t v = 0; v < N; ++v) {
        Item it = {(double)visits[v] * cost_feat / (double)row_bytes, 0, v, row_bytes};
        items[n++] = it;
    }
    for (int64_t e = 0; e < E; ++e) {
        Item it = {(double)counts[e] * cost_adj / 4.0, 1, e, 4};
        items[n++] = it;
    }
    qsort(items, (size_t)n, sizeof(Item), cmp_item);
    uint64_t left = C;
    char* adm_node = (char*)calloc((size_t)(N > 0 ? N : 1), 1);
    char* adm_elem = (char*)calloc((size_t)(E > 0 ? E : 1), 1);
    for (int64_t i = 0; i < n; ++i) {
        if ((uint64_t)items[i].size > left) continue;
        left -= (uint64_t)items[i].size;
        if (items[i].kind == 0)
            adm_node[items[i].id] = 1;
        else
            adm_elem[items[i].id] = 1;
    }
    int32_t slot = 0;
    for (int64_t v = 0; v < N; ++v) slot_of[v] = adm_node[v] ? slot++ : -1;
    for (int64_t v = 0; v < N; ++v) {
        int32_t c = 0;
        for (int64_t e = indptr[v]; e < indptr[v + 1]; ++e) c += adm_elem[e];
        cached_len[v] = c;
    }
    free(items);
    free(adm_node);
    free(adm_elem);
    return C - left;
}

/* One inference step on the CPU (bench.py cpu_baseline): O-6 with pass 0 over the
 * current CSC and the adjacency cache, then O-7.  Thin composition, no new arithmetic. */
int32_t oracle_sample_gather(int64_t N, const int64_t* indptr, const int32_t* indices_cur,
                             const int32_t* cached_len, const int32_t* slot_of, const float* feats,
                             int32_t D, const int32_t* seeds, int32_t B, const int32_t* fanouts,
                             int32_t L, uint64_t seed, int32_t* F_out, int64_t F_cap,
                             int64_t* sizes_out, int32_t** bptr_out, int32_t** bsrc_out,
                             const int64_t* bsrc_caps, float* X, int64_t ldx, uint64_t* counters4) {
    uint64_t adj[2] = {0, 0}, feat[2] = {0, 0};
    int32_t rc = oracle_sample_batch(N, indptr, indices_cur, cached_len, seeds, B, fanouts, L, seed, 0,
                                     F_out, F_cap, sizes_out, bptr_out, bsrc_out, bsrc_caps, adj, NULL);
    if (rc != OR_OK) return rc;
    oracle_gather(F_out, sizes_out[L], feats, D, slot_of, X, ldx, feat);
    counters4[0] = adj[0];
    counters4[1] = adj[1];
    counters4[2] = feat[0];
    counters4[3] = feat[1];
    return OR_OK;
}
