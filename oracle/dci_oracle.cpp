// =====================================================================================
// DCI ORACLE — plain, slow, obviously-correct CPU reference for the DCI hot path.
//
// TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load this library. The product path
// (paper_2503_01281_b200/) never links, imports or calls it, and this file shares no
// code, header, table or constant generator with the CUDA path.
//
// Paper: "DCI: A Coordinated Allocation and Filling Workload-Aware Dual-Cache
// Allocation GNN Inference Acceleration System", arXiv 2503.01281.
// Citation key: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n;
// O-k / Ck = the oracle definition / ambiguity-ledger rows of SURVEY.md §8(c), restated
// (with every reading we took) in DESIGN.md §3.
//
// Every function below follows its definition step by step. There is no blocking,
// fusion or reordering; library primitives used as single steps: std::sort,
// std::stable_sort, std::unordered_map, unsigned __int128.
//
// Parity status: every function is pinned by a `-m "not gpu"` test in
// tests/test_oracle_*.py against something other than itself.
// =====================================================================================
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <unordered_map>
#include <vector>

extern "C" {

// Status codes (mirrors nothing; the product library has its own enum).
enum { OR_OK = 0, OR_EINVAL = -1, OR_ESEED = -2, OR_EDUP = -3, OR_ECAP = -4 };

// -------------------------------------------------------------------------------------
// O-1  Philox4x32-10 (Salmon et al., "Parallel random numbers: as easy as 1, 2, 3",
// SC'11; Random123).  BASELINE.json north_star: "a counter-based Philox draw keyed by
// (seed, layer, node, slot)".  One round:
//   (hi0, lo0) = M0 * c0 ; (hi1, lo1) = M1 * c2
//   c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)
// key schedule between rounds: k0 += W0, k1 += W1.  Ten rounds.
// -------------------------------------------------------------------------------------
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
        c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
    }
    out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
}

// O-2  u(seed, pass, hop, v, i) = Philox(ctr=(v, i, hop, pass), key=(seed_lo, seed_hi));
// u = (uint64)r.y << 32 | r.x.  pass 0 = inference, pass 1 = presample (C4).
uint64_t oracle_draw(uint64_t seed, uint32_t pass, uint32_t hop, uint32_t v, uint32_t i) {
    uint32_t ctr[4] = {v, i, hop, pass};
    uint32_t key[2] = {(uint32_t)(seed & 0xFFFFFFFFu), (uint32_t)(seed >> 32)};
    uint32_t r[4];
    oracle_philox4x32_10(ctr, key, r);
    return ((uint64_t)r[1] << 32) | (uint64_t)r[0];
}

// O-3  bounded(u, m) = floor(u * m / 2^64), 1 <= m <= 2^32 (multiply-high, no rejection).
uint64_t oracle_bounded(uint64_t u, uint64_t m) {
    unsigned __int128 prod = (unsigned __int128)u * (unsigned __int128)m;
    return (uint64_t)(prod >> 64);
}

// O-4 (Floyd part) given the k bounded draws t[i] in [0, deg-k+i], return the chosen
// ranks in draw order (NOT sorted).  Robert Floyd's algorithm (Bentley & Floyd, CACM
// 1987, "A sample of brilliance"): for j = deg-k .. deg-1: t = uniform[0, j];
// if t already chosen then choose j else choose t.
void oracle_floyd_from_draws(int64_t deg, int32_t k, const uint64_t* t, int64_t* chosen) {
    for (int32_t i = 0; i < k; ++i) {
        int64_t j = deg - k + i;
        int64_t ti = (int64_t)t[i];
        bool seen = false;
        for (int32_t m = 0; m < i; ++m)
            if (chosen[m] == ti) seen = true;
        chosen[i] = seen ? j : ti;
    }
}

// O-4  select for (v, hop h): f = fanout of this hop, k = min(deg, f) (C1: without
// replacement).  deg <= f: ranks 0..deg-1.  Else Floyd with t_i = bounded(u(..., i), j+1),
// j = deg-k+i.  Output sorted ascending (canonical order, O-4).  Returns k.
int32_t oracle_select(uint64_t seed, uint32_t pass, uint32_t hop, int32_t v, int64_t deg, int32_t f,
                      int64_t* ranks_out) {
    if (deg <= 0) return 0;
    if (deg <= f) {
        for (int64_t r = 0; r < deg; ++r) ranks_out[r] = r;
        return (int32_t)deg;
    }
    int32_t k = f;
    std::vector<uint64_t> t(k);
    for (int32_t i = 0; i < k; ++i) {
        int64_t j = deg - k + i;
        uint64_t u = oracle_draw(seed, pass, hop, (uint32_t)v, (uint32_t)i);
        t[i] = oracle_bounded(u, (uint64_t)(j + 1));
    }
    oracle_floyd_from_draws(deg, k, t.data(), ranks_out);
    std::sort(ranks_out, ranks_out + k);
    return k;
}

// -------------------------------------------------------------------------------------
// O-5 / O-6  one mini-batch of L-hop uniform neighbour sampling with DGL block
// semantics (C2: every node of F_h is re-sampled at hop h; F_{h+1} = F_h ++ new),
// DGL fan-out order (C3: hop h uses fanouts[L-1-h]), first-occurrence relabelling in
// (dst-major, rank-ascending) order (C6).  P:116-117; Table I P:89-99.
//
// Element access (O-5): nbr(v, r) = indices_cur[indptr[v] + r]; it is an adjacency-cache
// hit iff r < cached_len[v] (C16).  cached_len == nullptr means no cache.
// edge_counts != nullptr: presample counting, edge_counts[indptr[v]+r] += 1 (O-8, C8).
//
// Outputs: F_out[0..|F_L|), sizes_out[0..L] = |F_h|, per hop h: bptr_out[h][0..|F_h|],
// bsrc_out[h][0..sum k).  adj_hm[0] += hits, adj_hm[1] += misses.
// -------------------------------------------------------------------------------------
int32_t oracle_sample_batch(int64_t N, const int64_t* indptr, const int32_t* indices_cur,
                            const int32_t* cached_len, const int32_t* seeds, int32_t B,
                            const int32_t* fanouts, int32_t L, uint64_t seed, uint32_t pass,
                            int32_t* F_out, int64_t F_cap, int64_t* sizes_out, int32_t** bptr_out,
                            int32_t** bsrc_out, const int64_t* bsrc_caps, uint64_t* adj_hm,
                            int32_t* edge_counts) {
    if (B < 0 || L < 1) return OR_EINVAL;
    for (int32_t h = 0; h < L; ++h)
        if (fanouts[h] < 1) return OR_EINVAL;
    // O-6: validate seeds (range, duplicates: C22)
    std::vector<int32_t> F;
    std::unordered_map<int32_t, int32_t> map;
    for (int32_t i = 0; i < B; ++i) {
        int32_t s = seeds[i];
        if (s < 0 || (int64_t)s >= N) return OR_ESEED;
        if (map.count(s)) return OR_EDUP;
        map[s] = (int32_t)F.size();
        F.push_back(s);
    }
    sizes_out[0] = (int64_t)F.size();
    std::vector<int64_t> ranks;
    for (int32_t h = 0; h < L; ++h) {
        int32_t f = fanouts[L - 1 - h];
        ranks.assign((size_t)f, 0);
        int64_t n_h = (int64_t)F.size();  // frozen frontier size
        int32_t* bptr = bptr_out[h];
        int32_t* bsrc = bsrc_out[h];
        int64_t nsrc = 0;
        bptr[0] = 0;
        for (int64_t d = 0; d < n_h; ++d) {
            int32_t v = F[(size_t)d];
            int64_t deg = indptr[v + 1] - indptr[v];
            int32_t k = oracle_select(seed, pass, (uint32_t)h, v, deg, f, ranks.data());
            for (int32_t s = 0; s < k; ++s) {
                int64_t r = ranks[(size_t)s];
                int32_t u = indices_cur[indptr[v] + r];
                if (cached_len != nullptr && r < (int64_t)cached_len[v])
                    adj_hm[0] += 1;
                else
                    adj_hm[1] += 1;
                if (edge_counts != nullptr) edge_counts[indptr[v] + r] += 1;
                auto it = map.find(u);
                int32_t local;
                if (it == map.end()) {
                    local = (int32_t)F.size();
                    map[u] = local;
                    F.push_back(u);
                } else {
                    local = it->second;
                }
                if (nsrc >= bsrc_caps[h]) return OR_ECAP;
                bsrc[nsrc++] = local;
            }
            bptr[d + 1] = (int32_t)nsrc;
        }
        sizes_out[h + 1] = (int64_t)F.size();
    }
    if ((int64_t)F.size() > F_cap) return OR_ECAP;
    for (size_t i = 0; i < F.size(); ++i) F_out[i] = F[i];
    return OR_OK;
}

// O-7  feature gather: X[i][:] = feats[F[i]][:]; a feature-cache hit iff
// slot_of[F[i]] >= 0.  slot_of == nullptr: no cache (all misses).
int32_t oracle_gather(const int32_t* F, int64_t nF, const float* feats, int32_t D,
                      const int32_t* slot_of, float* X, int64_t ldx, uint64_t* feat_hm) {
    for (int64_t i = 0; i < nF; ++i) {
        int32_t v = F[i];
        if (X != nullptr)
            for (int32_t c = 0; c < D; ++c) X[i * ldx + c] = feats[(int64_t)v * D + c];
        if (slot_of != nullptr && slot_of[v] >= 0)
            feat_hm[0] += 1;
        else
            feat_hm[1] += 1;
    }
    return OR_OK;
}

// O-8  presample: for each presample batch b run O-6 with
// pass 1 on the ORIGINAL CSC and no cache; edge_counts[indptr[v]+r] += 1 per sampled
// (v, r) per hop (C8); node_visits[u] += 1 per u in F_L (C7).  Times are measured by the
// GPU; the oracle does not produce them.  seeds: num_seeds ids cut into batches of B
// (last batch ragged).  Counts accumulate into the caller's arrays.
int32_t oracle_presample(int64_t N, const int64_t* indptr, const int32_t* indices,
                         const int32_t* seeds, int64_t num_seeds, int32_t B, const int32_t* fanouts,
                         int32_t L, uint64_t seed, int32_t* node_visits, int32_t* edge_counts) {
    if (B < 1 || L < 1) return OR_EINVAL;
    for (int64_t b0 = 0; b0 < num_seeds; b0 += B) {
        int32_t nb = (int32_t)std::min<int64_t>(B, num_seeds - b0);
        // worst-case capacities: |F_h| <= min(N, nb * prod(1+f))
        std::vector<int64_t> cap(L + 1);
        cap[0] = nb;
        for (int32_t h = 0; h < L; ++h) cap[h + 1] = std::min<int64_t>(N, cap[h] * (1 + fanouts[L - 1 - h]));
        std::vector<int32_t> F((size_t)cap[L]);
        std::vector<int64_t> sizes(L + 1);
        std::vector<std::vector<int32_t>> bptr(L), bsrc(L);
        std::vector<int32_t*> bp(L), bs(L);
        std::vector<int64_t> bcap(L);
        for (int32_t h = 0; h < L; ++h) {
            bptr[h].resize((size_t)cap[h] + 1);
            bcap[h] = cap[h] * fanouts[L - 1 - h];
            bsrc[h].resize((size_t)bcap[h]);
            bp[h] = bptr[h].data();
            bs[h] = bsrc[h].data();
        }
        uint64_t hm[2] = {0, 0};
        int32_t rc = oracle_sample_batch(N, indptr, indices, nullptr, seeds + b0, nb, fanouts, L, seed, 1,
                                         F.data(), cap[L], sizes.data(), bp.data(), bs.data(), bcap.data(),
                                         hm, edge_counts);
        if (rc != OR_OK) return rc;
        for (int64_t i = 0; i < sizes[L]; ++i) node_visits[F[(size_t)i]] += 1;
    }
    return OR_OK;
}

// O-10  Eq. (1): C_adj = floor(C * S / (S + F)), C_feat = C - C_adj,
// S = sum t_sample, F = sum t_feature (integer ns, C19).  Explicit ratio (num/den,
// den > 0) replaces S/(S+F) (C20).  S + F == 0 -> C_adj = floor(C/2).
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

// O-11  feature fill (C10-C12): cap rows; admit the first `cap` nodes of
// sort(nodes, key = (visits desc, id asc)); slots in ascending id.  When the
// above-average set fits, this is exactly the paper's "greater than the average, then
// backfill" set (C11).  slot_of_out[v] = slot or -1; admitted_out[j] = node in slot j.
int64_t oracle_feat_fill(int64_t N, const int32_t* visits, int64_t cap, int32_t* slot_of_out,
                         int32_t* admitted_out) {
    if (cap > N) cap = N;
    if (cap < 0) cap = 0;
    std::vector<int32_t> order((size_t)N);
    for (int64_t v = 0; v < N; ++v) order[(size_t)v] = (int32_t)v;
    std::sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
        if (visits[a] != visits[b]) return visits[a] > visits[b];
        return a < b;
    });
    std::vector<int32_t> admitted(order.begin(), order.begin() + cap);
    std::sort(admitted.begin(), admitted.end());
    for (int64_t v = 0; v < N; ++v) slot_of_out[v] = -1;
    for (int64_t j = 0; j < cap; ++j) {
        slot_of_out[admitted[(size_t)j]] = (int32_t)j;
        if (admitted_out) admitted_out[j] = admitted[(size_t)j];
    }
    return cap;
}

// O-12  adjacency fill, Algorithm 1 with Fig. 6:
//  level-2 (per node, C13/C14): perm_v = stable sort of 0..deg-1 by count desc;
//          indices_R[indptr[v]+p] = indices[indptr[v]+perm_v[p]]  (always applied, C17)
//  cap_e = floor(C_adj / 4) 4-byte elements (C18).
//  whole-fit (Alg. 1 lines 1-3): E <= cap_e -> cached_len = deg for every node.
//  else level-1 (C13): walk nodes in sort(key = (total desc, id asc)), rem = cap_e,
//          cached_len[v] = min(deg_v, rem), rem -= cached_len[v] (C15: node-major prefix,
//          last node partial).
//  acache = concatenation of the cached prefixes of indices_R in that walk order;
//  cache_off[v] = running offset (in elements).  Returns the number of cached elements.
int64_t oracle_adj_fill(int64_t N, int64_t E, const int64_t* indptr, const int32_t* indices,
                        const int32_t* counts, uint64_t c_adj_bytes, int32_t* indices_R,
                        int32_t* cached_len, int64_t* cache_off, int32_t* acache) {
    // level 2: per-node stable sort of elements by access count, descending
    for (int64_t v = 0; v < N; ++v) {
        int64_t a = indptr[v], deg = indptr[v + 1] - indptr[v];
        std::vector<int64_t> perm((size_t)deg);
        for (int64_t p = 0; p < deg; ++p) perm[(size_t)p] = p;
        std::stable_sort(perm.begin(), perm.end(),
                         [&](int64_t x, int64_t y) { return counts[a + x] > counts[a + y]; });
        for (int64_t p = 0; p < deg; ++p) indices_R[a + p] = indices[a + perm[(size_t)p]];
    }
    uint64_t cap_e = c_adj_bytes / 4;
    // node totals (Alg. 1 lines 5-8)
    std::vector<int64_t> total((size_t)N, 0);
    for (int64_t v = 0; v < N; ++v)
        for (int64_t e = indptr[v]; e < indptr[v + 1]; ++e) total[(size_t)v] += counts[e];
    // level 1 order (Alg. 1 line 9; ties by id)
    std::vector<int32_t> order((size_t)N);
    for (int64_t v = 0; v < N; ++v) order[(size_t)v] = (int32_t)v;
    std::sort(order.begin(), order.end(), [&](int32_t x, int32_t y) {
        if (total[(size_t)x] != total[(size_t)y]) return total[(size_t)x] > total[(size_t)y];
        return x < y;
    });
    for (int64_t v = 0; v < N; ++v) {
        cached_len[v] = 0;
        cache_off[v] = 0;
    }
    int64_t off = 0;
    if ((uint64_t)E <= cap_e) {
        // whole-fit branch: cache everything (walk order still defines the layout)
        for (int32_t v : order) {
            int64_t deg = indptr[v + 1] - indptr[v];
            cached_len[v] = (int32_t)deg;
            cache_off[v] = off;
            for (int64_t p = 0; p < deg; ++p) acache[off + p] = indices_R[indptr[v] + p];
            off += deg;
        }
        return off;
    }
    uint64_t rem = cap_e;
    for (int32_t v : order) {
        int64_t deg = indptr[v + 1] - indptr[v];
        int64_t take = (int64_t)std::min<uint64_t>((uint64_t)deg, rem);
        cached_len[v] = (int32_t)take;
        cache_off[v] = off;
        for (int64_t p = 0; p < take; ++p) acache[off + p] = indices_R[indptr[v] + p];
        off += take;
        rem -= (uint64_t)take;
    }
    return off;
}

// O-13 mean / sum aggregator over one sampled block (P:107
// "aggregating" the neighbours' features; BJ north_star's optional consumer; reading C23):
// H[d][c] = (1 / k_d) * sum_{j = bptr[d]}^{bptr[d+1]-1} X[bsrc[j]][c], accumulated in double;
// k_d = 0 -> H[d] = 0.
// op = 0: mean ("avg", GCN in Table III); op = 1: sum (GraphSAGE's "sum" there).
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

// O-14 DUCATI-style unified-budget knapsack fill, as simplified by SPEC
// (S:496-504): items are feature rows (value = visits * cost_feat, size = row_bytes) and
// adjacency elements (value = count * cost_adj, size = 4 B); sort by value density
// (value / size) descending, ties by kind (feature first) then id (node id / CSC position);
// admit every item that still fits the remaining budget, in that order.  Admitted adjacency
// elements are regrouped per node by the level-2 order (count desc, position asc): the
// cached prefix of node v has length = #admitted elements of v ("re-sorting admitted
// elements within each node by count so the prefix hit rule still applies").
// Outputs: slot_of[N] (admitted rows, slots in ascending id), cached_len[N]; returns bytes used.
uint64_t oracle_knapsack_fill(int64_t N, int64_t E, const int64_t* indptr, const int32_t* visits,
                              const int32_t* counts, uint64_t C, int64_t row_bytes, double cost_feat,
                              double cost_adj, int32_t* slot_of, int32_t* cached_len) {
    struct Item {
        double density;
        int kind;     // 0 feature row, 1 adjacency element
        int64_t id;   // node id or CSC position
        int64_t size;
    };
    std::vector<Item> items;
    items.reserve((size_t)(N + E));
    for (int64_t v = 0; v < N; ++v)
        items.push_back({(double)visits[v] * cost_feat / (double)row_bytes, 0, v, row_bytes});
    for (int64_t e = 0; e < E; ++e) items.push_back({(double)counts[e] * cost_adj / 4.0, 1, e, 4});
    std::sort(items.begin(), items.end(), [](const Item& a, const Item& b) {
        if (a.density != b.density) return a.density > b.density;
        if (a.kind != b.kind) return a.kind < b.kind;
        return a.id < b.id;
    });
    uint64_t left = C;
    std::vector<char> adm_node((size_t)N, 0), adm_elem((size_t)E, 0);
    for (const Item& it : items) {
        if ((uint64_t)it.size > left) continue;
        left -= (uint64_t)it.size;
        if (it.kind == 0)
            adm_node[(size_t)it.id] = 1;
        else
            adm_elem[(size_t)it.id] = 1;
    }
    int32_t slot = 0;
    for (int64_t v = 0; v < N; ++v) slot_of[v] = adm_node[(size_t)v] ? slot++ : -1;
    for (int64_t v = 0; v < N; ++v) {
        int32_t c = 0;
        for (int64_t e = indptr[v]; e < indptr[v + 1]; ++e) c += adm_elem[(size_t)e];
        cached_len[v] = c;
    }
    return C - left;
}

// One inference step on the CPU (bench.py cpu_baseline): O-6 with pass 0 over the
// current CSC and the adjacency cache, then O-7.  Thin composition, no new arithmetic.
int32_t oracle_sample_gather(int64_t N, const int64_t* indptr, const int32_t* indices_cur,
                             const int32_t* cached_len, const int32_t* slot_of, const float* feats,
                             int32_t D, const int32_t* seeds, int32_t B, const int32_t* fanouts,
                             int32_t L, uint64_t seed, int32_t* F_out, int64_t F_cap,
                             int64_t* sizes_out, int32_t** bptr_out, int32_t** bsrc_out,
                             const int64_t* bsrc_caps, float* X, int64_t ldx, uint64_t* counters4) {
    uint64_t adj[2] = {0, 0}, feat[2] = {0, 0};
    int32_t rc = oracle_sample_batch(N, indptr, indices_cur, cached_len, seeds, B, fanouts, L, seed, 0,
                                     F_out, F_cap, sizes_out, bptr_out, bsrc_out, bsrc_caps, adj, nullptr);
    if (rc != OR_OK) return rc;
    oracle_gather(F_out, sizes_out[L], feats, D, slot_of, X, ldx, feat);
    counters4[0] = adj[0];
    counters4[1] = adj[1];
    counters4[2] = feat[0];
    counters4[3] = feat[1];
    return OR_OK;
}

}  // extern "C"
