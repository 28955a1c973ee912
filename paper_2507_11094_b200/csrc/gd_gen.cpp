// gd_gen.cpp -- synthetic graph and update-stream generators at BASELINE scale
// (host C++, OpenMP).  Same recipes as the reference's generate.py:15-161
// (R-MAT a/b/c = .57/.19/.19, uniform random, distinct pairs, no self-loops;
// update streams: deletes drawn without replacement from the edges, adds from
// non-edges, every touched pair distinct), plus the 2-D grid the survey needs
// for C4.  Randomness is counter-based (splitmix64 of seed and index), so the
// output is identical for any thread count.  The reference's own generators
// need ~9 s per 1M R-MAT edges (SURVEY.md §7 hard part 5); these run at
// memory speed.  Both bench arms use them, so both see the same inputs.
#include <omp.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <vector>

namespace {

inline uint64_t mix(uint64_t x) {  // splitmix64 finaliser
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
inline uint64_t rnd(uint64_t seed, uint64_t stream, uint64_t i) { return mix(mix(seed * 0x100000001b3ULL ^ stream) ^ i); }
inline double unit(uint64_t r) { return (double)(r >> 11) * (1.0 / 9007199254740992.0); }

// parallel LSD radix sort of (key, val) pairs by the low `bits` bits of key
void radix_sort(std::vector<uint64_t>& key, std::vector<int64_t>& val, int bits) {
    size_t n = key.size();
    std::vector<uint64_t> k2(n);
    std::vector<int64_t> v2(n);
    int nt = omp_get_max_threads();
    const int R = 11, B = 1 << R;
    std::vector<size_t> hist((size_t)nt * B);
    for (int shift = 0; shift < bits; shift += R) {
        std::fill(hist.begin(), hist.end(), 0);
#pragma omp parallel num_threads(nt)
        {
            int t = omp_get_thread_num();
            size_t lo = n * t / nt, hi = n * (t + 1) / nt;
            size_t* h = &hist[(size_t)t * B];
            for (size_t i = lo; i < hi; ++i) h[(key[i] >> shift) & (B - 1)]++;
        }
        size_t sum = 0;
        for (int b = 0; b < B; ++b)
            for (int t = 0; t < nt; ++t) {
                size_t c = hist[(size_t)t * B + b];
                hist[(size_t)t * B + b] = sum;
                sum += c;
            }
#pragma omp parallel num_threads(nt)
        {
            int t = omp_get_thread_num();
            size_t lo = n * t / nt, hi = n * (t + 1) / nt;
            size_t* h = &hist[(size_t)t * B];
            for (size_t i = lo; i < hi; ++i) {
                size_t p = h[(key[i] >> shift) & (B - 1)]++;
                k2[p] = key[i];
                v2[p] = val[i];
            }
        }
        key.swap(k2);
        val.swap(v2);
    }
}

int bits_for(uint64_t maxv) {
    int b = 1;
    while (b < 64 && (maxv >> b)) ++b;
    return b;
}

// Keep the first occurrence of every key, in candidate order, up to `want`.
// Returns kept candidate indices (ascending).
std::vector<int64_t> first_distinct(const std::vector<uint64_t>& keys, const std::vector<uint8_t>& ok, size_t want,
                                    uint64_t maxkey) {
    size_t n = keys.size();
    std::vector<uint64_t> k;
    std::vector<int64_t> v;
    k.reserve(n);
    v.reserve(n);
    for (size_t i = 0; i < n; ++i)
        if (ok[i]) {
            k.push_back(keys[i]);
            v.push_back((int64_t)i);
        }
    radix_sort(k, v, bits_for(maxkey));  // stable: equal keys keep candidate order
    std::vector<uint8_t> first(n, 0);
    int64_t nk = (int64_t)k.size();
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nk; ++i)
        if (i == 0 || k[i] != k[i - 1]) first[v[i]] = 1;
    std::vector<int64_t> keep;
    keep.reserve(std::min(want, (size_t)nk));
    for (size_t i = 0; i < n && keep.size() < want; ++i)
        if (first[i]) keep.push_back((int64_t)i);
    return keep;
}

}  // namespace

extern "C" {

__attribute__((visibility("default"))) int gdgen_threads(void) { return omp_get_max_threads(); }

// R-MAT (generate.py:58-104): returns the number of distinct edges written
// (<= m).  undirected: a pair and its reverse count once (key = min,max).
// Weights U[1, max_weight] when weighted, else 1.
__attribute__((visibility("default"))) int64_t gdgen_rmat(int scale, int64_t m, uint64_t seed, double a, double b,
                                                          double c, int undirected, int weighted, int64_t max_weight,
                                                          int64_t* src, int64_t* dst, int64_t* w) {
    size_t cand = (size_t)(m + m / 4 + 1024);
    std::vector<uint64_t> keys(cand);
    std::vector<uint8_t> ok(cand);
    uint64_t n = 1ULL << scale;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)cand; ++i) {
        uint64_t u = 0, v = 0;
        for (int l = 0; l < scale; ++l) {
            double r = unit(rnd(seed, 1 + l, (uint64_t)i));
            int qu = 0, qv = 0;
            if (r < a) {
            } else if (r < a + b) qv = 1;
            else if (r < a + b + c) qu = 1;
            else qu = qv = 1;
            u = (u << 1) | qu;
            v = (v << 1) | qv;
        }
        ok[i] = u != v;
        uint64_t x = u, y = v;
        if (undirected && x > y) std::swap(x, y);
        keys[i] = x * n + y;
        (void)u;
    }
    std::vector<int64_t> keep = first_distinct(keys, ok, (size_t)m, n * n);
    int64_t out = (int64_t)keep.size();
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < out; ++j) {
        int64_t i = keep[j];
        // recompute the oriented pair (keys may be min/max-normalised)
        uint64_t u = 0, v = 0;
        for (int l = 0; l < scale; ++l) {
            double r = unit(rnd(seed, 1 + l, (uint64_t)i));
            int qu = 0, qv = 0;
            if (r < a) {
            } else if (r < a + b) qv = 1;
            else if (r < a + b + c) qu = 1;
            else qu = qv = 1;
            u = (u << 1) | qu;
            v = (v << 1) | qv;
        }
        src[j] = (int64_t)u;
        dst[j] = (int64_t)v;
        w[j] = weighted ? 1 + (int64_t)(rnd(seed, 99, (uint64_t)i) % (uint64_t)max_weight) : 1;
    }
    return out;
}

// Uniform random simple graph (generate.py:15-55, without the spanning chain).
__attribute__((visibility("default"))) int64_t gdgen_uniform(int64_t n, int64_t m, uint64_t seed, int undirected,
                                                             int weighted, int64_t max_weight, int64_t* src,
                                                             int64_t* dst, int64_t* w) {
    size_t cand = (size_t)(m + m / 8 + 1024);
    std::vector<uint64_t> keys(cand);
    std::vector<uint8_t> ok(cand);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)cand; ++i) {
        uint64_t u = rnd(seed, 11, (uint64_t)i) % (uint64_t)n, v = rnd(seed, 12, (uint64_t)i) % (uint64_t)n;
        ok[i] = u != v;
        if (undirected && u > v) std::swap(u, v);
        keys[i] = u * (uint64_t)n + v;
    }
    std::vector<int64_t> keep = first_distinct(keys, ok, (size_t)m, (uint64_t)n * (uint64_t)n);
    int64_t out = (int64_t)keep.size();
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < out; ++j) {
        int64_t i = keep[j];
        src[j] = (int64_t)(rnd(seed, 11, (uint64_t)i) % (uint64_t)n);
        dst[j] = (int64_t)(rnd(seed, 12, (uint64_t)i) % (uint64_t)n);
        w[j] = weighted ? 1 + (int64_t)(rnd(seed, 99, (uint64_t)i) % (uint64_t)max_weight) : 1;
    }
    return out;
}

// rows x cols grid, 4-neighbour, both arcs of every neighbour pair as
// separate directed edges (a road-network proxy for C4); weights U[1, max_w].
__attribute__((visibility("default"))) int64_t gdgen_grid(int64_t rows, int64_t cols, uint64_t seed,
                                                          int64_t max_weight, int64_t* src, int64_t* dst,
                                                          int64_t* w) {
    int64_t per_row = 2 * (cols - 1);
    int64_t horiz = rows * per_row;
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < rows; ++r) {
        for (int64_t c = 0; c + 1 < cols; ++c) {
            int64_t e = r * per_row + 2 * c, v = r * cols + c;
            src[e] = v;
            dst[e] = v + 1;
            src[e + 1] = v + 1;
            dst[e + 1] = v;
        }
    }
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < rows - 1; ++r) {
        for (int64_t c = 0; c < cols; ++c) {
            int64_t e = horiz + r * 2 * cols + 2 * c, v = r * cols + c;
            src[e] = v;
            dst[e] = v + cols;
            src[e + 1] = v + cols;
            dst[e + 1] = v;
        }
    }
    int64_t m = horiz + (rows - 1) * 2 * cols;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < m; ++e) w[e] = 1 + (int64_t)(rnd(seed, 77, (uint64_t)e) % (uint64_t)max_weight);
    return m;
}

// Update stream (generate.py:107-161 semantics): n_del deletes drawn without
// replacement from the m edges, n_add adds from non-edge pairs (distinct, no
// self-loops, not chosen twice), then split into batches of `batch` records,
// each batch shuffled.  Output arrays hold n_del + n_add records; returns the
// number of adds actually found (<= n_add).
__attribute__((visibility("default"))) int64_t gdgen_updates(const int64_t* src, const int64_t* dst, int64_t m,
                                                             int64_t n, int64_t n_del, int64_t n_add, int64_t batch,
                                                             uint64_t seed, int undirected, int64_t max_weight,
                                                             uint8_t* kind, int64_t* us, int64_t* ud, int64_t* uw) {
    auto norm = [&](int64_t u, int64_t v) -> uint64_t {
        if (undirected && u > v) std::swap(u, v);
        return (uint64_t)u * (uint64_t)n + (uint64_t)v;
    };
    uint64_t maxkey = (uint64_t)n * (uint64_t)n;
    // sorted edge keys for membership
    std::vector<uint64_t> ek(m);
    std::vector<int64_t> eidx(m);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i) {
        ek[i] = norm(src[i], dst[i]);
        eidx[i] = i;
    }
    radix_sort(ek, eidx, bits_for(maxkey));
    // deletes: the n_del edges with the smallest random priority (distinct pairs)
    std::vector<uint64_t> pri(m);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i) pri[i] = rnd(seed, 21, (uint64_t)i);
    if (n_del > m) n_del = m;
    // the n_del smallest priorities: collect everything under a threshold
    // that keeps ~2% slack, sort that small set, widen if it fell short
    std::vector<int64_t> order;
    for (double slack = 1.02 + 64.0 / (double)(n_del + 1);; slack *= 1.5) {
        long double frac = std::min<long double>(1.0L, (long double)n_del / (long double)std::max<int64_t>(m, 1) * slack);
        uint64_t thr = frac >= 1.0L ? UINT64_MAX : (uint64_t)(frac * 18446744073709551615.0L);
        std::vector<uint64_t> pk;
        std::vector<int64_t> pv;
        for (int64_t i = 0; i < m; ++i)
            if (pri[i] <= thr) {
                pk.push_back(pri[i]);
                pv.push_back(i);
            }
        if ((int64_t)pk.size() >= n_del || frac >= 1.0L) {
            radix_sort(pk, pv, 64);
            order.assign(pv.begin(), pv.begin() + std::min<int64_t>(n_del, (int64_t)pv.size()));
            break;
        }
    }
    // adds: candidates not in the edge set
    size_t cand = (size_t)(n_add + n_add / 4 + 1024);
    std::vector<uint64_t> ak(cand);
    std::vector<uint8_t> ok(cand);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)cand; ++i) {
        int64_t u = (int64_t)(rnd(seed, 31, (uint64_t)i) % (uint64_t)n);
        int64_t v = (int64_t)(rnd(seed, 32, (uint64_t)i) % (uint64_t)n);
        uint64_t k = norm(u, v);
        ak[i] = k;
        ok[i] = u != v && !std::binary_search(ek.begin(), ek.end(), k);
    }
    std::vector<int64_t> keep = first_distinct(ak, ok, (size_t)n_add, maxkey);
    int64_t na = (int64_t)keep.size();
    // interleave: record r of the stream gets a random priority inside its batch
    int64_t total = n_del + na;
    std::vector<uint64_t> sk(total);
    std::vector<int64_t> sv(total);
    // deletes and adds are spread evenly over the batches before shuffling
    for (int64_t i = 0; i < total; ++i) {
        // position in the merged (del, add) sequence
        sv[i] = i;
    }
    std::vector<int64_t> merged(total);
    {
        int64_t di = 0, ai = 0;
        for (int64_t i = 0; i < total; ++i) {
            // choose the stream that is behind its share
            bool take_del = ai >= na || (di < n_del && di * (int64_t)(na + 1) <= ai * (int64_t)(n_del + 1));
            merged[i] = take_del ? di++ : -(1 + ai++);
        }
    }
    for (int64_t i = 0; i < total; ++i) {
        int64_t bidx = batch > 0 ? i / batch : 0;
        sk[i] = ((uint64_t)bidx << 40) | (rnd(seed, 41, (uint64_t)i) >> 24);
    }
    radix_sort(sk, sv, 64);
    for (int64_t p = 0; p < total; ++p) {
        int64_t t = merged[sv[p]];
        if (t >= 0) {
            int64_t e = order[t];
            kind[p] = 'd';
            us[p] = src[e];
            ud[p] = dst[e];
            uw[p] = 1;
        } else {
            int64_t i = keep[-(t + 1)];
            kind[p] = 'a';
            us[p] = (int64_t)(rnd(seed, 31, (uint64_t)i) % (uint64_t)n);
            ud[p] = (int64_t)(rnd(seed, 32, (uint64_t)i) % (uint64_t)n);
            uw[p] = max_weight > 1 ? 1 + (int64_t)(rnd(seed, 33, (uint64_t)i) % (uint64_t)max_weight) : 1;
        }
    }
    return na;
}

}  // extern "C"
