// gd_pyrand.cpp -- seed-compatible generators.
//
// The reference's generators (pkg/src/graphdyn/generate.py:15-161) draw from
// Python's random.Random(seed): MT19937 seeded by init_by_array over the
// seed's 32-bit words, random() = genrand_res53, randrange / randint through
// _randbelow (getrandbits + rejection), sample() and shuffle() as in CPython
// 3.12's Lib/random.py.  This file restates that generator and the three
// recipes draw for draw, so a given seed yields the SAME edges and update
// stream as the reference -- at native speed (the Python loops need ~9 s per
// 1M R-MAT edges).  Bit-identity is checked against the reference itself in
// tests/test_pyrand_cpu.py.
//
// Sequential by construction (one Mersenne Twister stream); pair
// de-duplication uses an open-addressing hash set instead of a Python set.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

namespace {

// ---------------------------------------------------------------- MT19937 --
struct PyRandom {
    static constexpr int N = 624, M = 397;
    uint32_t mt[N];
    int mti = N + 1;

    void init_genrand(uint32_t s) {
        mt[0] = s;
        for (mti = 1; mti < N; ++mti) mt[mti] = 1812433253U * (mt[mti - 1] ^ (mt[mti - 1] >> 30)) + (uint32_t)mti;
    }
    void init_by_array(const uint32_t* key, size_t len) {
        init_genrand(19650218U);
        size_t i = 1, j = 0;
        for (size_t k = (N > len ? N : len); k; --k) {
            mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1664525U)) + key[j] + (uint32_t)j;
            ++i;
            ++j;
            if (i >= (size_t)N) {
                mt[0] = mt[N - 1];
                i = 1;
            }
            if (j >= len) j = 0;
        }
        for (size_t k = N - 1; k; --k) {
            mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1566083941U)) - (uint32_t)i;
            ++i;
            if (i >= (size_t)N) {
                mt[0] = mt[N - 1];
                i = 1;
            }
        }
        mt[0] = 0x80000000U;
        mti = N;
    }
    // random.seed(int): init_by_array over abs(seed) in 32-bit little-endian words
    explicit PyRandom(uint64_t seed) {
        uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
        init_by_array(key, (seed >> 32) ? 2 : 1);
    }
    uint32_t genrand() {
        static const uint32_t mag01[2] = {0x0U, 0x9908b0dfU};
        uint32_t y;
        if (mti >= N) {
            int kk;
            for (kk = 0; kk < N - M; ++kk) {
                y = (mt[kk] & 0x80000000U) | (mt[kk + 1] & 0x7fffffffU);
                mt[kk] = mt[kk + M] ^ (y >> 1) ^ mag01[y & 1U];
            }
            for (; kk < N - 1; ++kk) {
                y = (mt[kk] & 0x80000000U) | (mt[kk + 1] & 0x7fffffffU);
                mt[kk] = mt[kk + (M - N)] ^ (y >> 1) ^ mag01[y & 1U];
            }
            y = (mt[N - 1] & 0x80000000U) | (mt[0] & 0x7fffffffU);
            mt[N - 1] = mt[M - 1] ^ (y >> 1) ^ mag01[y & 1U];
            mti = 0;
        }
        y = mt[mti++];
        y ^= (y >> 11);
        y ^= (y << 7) & 0x9d2c5680U;
        y ^= (y << 15) & 0xefc60000U;
        y ^= (y >> 18);
        return y;
    }
    double random() {  // genrand_res53
        uint32_t a = genrand() >> 5, b = genrand() >> 6;
        return (a * 67108864.0 + b) * (1.0 / 9007199254740992.0);
    }
    uint64_t getrandbits(int k) {  // k in [1, 64]
        if (k <= 32) return genrand() >> (32 - k);
        uint64_t lo = genrand();
        uint64_t hi = genrand();
        if (k < 64) hi >>= (64 - k);
        return lo | (hi << 32);
    }
    uint64_t randbelow(uint64_t n) {  // n > 0
        int k = 64 - __builtin_clzll(n);
        uint64_t r = getrandbits(k);
        while (r >= n) r = getrandbits(k);
        return r;
    }
    int64_t randint(int64_t a, int64_t b) { return a + (int64_t)randbelow((uint64_t)(b - a + 1)); }
};

// ------------------------------------------------------- pair hash set --
struct PairSet {
    std::vector<uint64_t> slot;  // key + 1; 0 = empty
    uint64_t mask = 0;
    explicit PairSet(size_t expect) {
        size_t cap = 1024;
        while (cap < expect * 2) cap <<= 1;
        slot.assign(cap, 0);
        mask = cap - 1;
    }
    static uint64_t mix(uint64_t x) {
        x ^= x >> 33;
        x *= 0xff51afd7ed558ccdULL;
        x ^= x >> 33;
        x *= 0xc4ceb9fe1a85ec53ULL;
        x ^= x >> 33;
        return x;
    }
    // true when inserted (was absent)
    bool insert(uint64_t key) {
        uint64_t h = mix(key) & mask, v = key + 1;
        while (slot[h]) {
            if (slot[h] == v) return false;
            h = (h + 1) & mask;
        }
        slot[h] = v;
        return true;
    }
    bool contains(uint64_t key) const {
        uint64_t h = mix(key) & mask, v = key + 1;
        while (slot[h]) {
            if (slot[h] == v) return true;
            h = (h + 1) & mask;
        }
        return false;
    }
};

inline uint64_t pkey(uint64_t u, uint64_t v, bool undirected) {
    if (undirected && u > v) std::swap(u, v);
    return (u << 32) | v;
}

}  // namespace

extern "C" {

// rmat_graph (generate.py:58-104).  Writes at most m edges; returns the count.
__attribute__((visibility("default"))) int64_t gdgen_py_rmat(int log2, int64_t m, uint64_t seed, int weighted,
                                                             int64_t max_weight, double a, double b, double c,
                                                             int undirected, int64_t* src, int64_t* dst, int64_t* w) {
    PyRandom rng(seed);
    PairSet pairs((size_t)m);
    int64_t got = 0, attempts = 0;
    const int64_t limit = 20 * (m > 1 ? m : 1) + 1000;
    while (got < m && attempts < limit) {
        ++attempts;
        uint64_t u = 0, v = 0;
        for (int l = 0; l < log2; ++l) {
            double r = rng.random();
            int qu, qv;
            if (r < a) qu = 0, qv = 0;
            else if (r < a + b) qu = 0, qv = 1;
            else if (r < a + b + c) qu = 1, qv = 0;
            else qu = 1, qv = 1;
            u = (u << 1) | (uint64_t)qu;
            v = (v << 1) | (uint64_t)qv;
        }
        if (u == v) continue;
        if (!pairs.insert(pkey(u, v, undirected))) continue;
        int64_t wt = weighted ? rng.randint(1, max_weight) : 1;
        src[got] = (int64_t)u;
        dst[got] = (int64_t)v;
        w[got] = wt;
        ++got;
    }
    return got;
}

// uniform_random_graph (generate.py:15-55).  out arrays hold at least
// m + (connected ? n - 1 : 0) edges; returns the count.
__attribute__((visibility("default"))) int64_t gdgen_py_uniform(int64_t n, int64_t m, uint64_t seed, int weighted,
                                                                int64_t max_weight, int connected, int undirected,
                                                                int64_t* src, int64_t* dst, int64_t* w) {
    PyRandom rng(seed);
    PairSet pairs((size_t)(m + (connected ? n : 0)));
    int64_t got = 0;
    auto add = [&](int64_t u, int64_t v) {
        if (u == v) return;
        if (!pairs.insert(pkey((uint64_t)u, (uint64_t)v, undirected))) return;
        int64_t wt = weighted ? rng.randint(1, max_weight) : 1;
        src[got] = u;
        dst[got] = v;
        w[got] = wt;
        ++got;
    };
    if (connected && n > 1) {
        std::vector<int64_t> order(n);
        for (int64_t i = 0; i < n; ++i) order[i] = i;
        for (int64_t i = n - 1; i >= 1; --i) std::swap(order[i], order[rng.randbelow((uint64_t)i + 1)]);
        for (int64_t i = 0; i + 1 < n; ++i) add(order[i], order[i + 1]);
    }
    int64_t attempts = 0;
    const int64_t limit = 50 * (m > 1 ? m : 1) + 1000;
    while (got < m && attempts < limit) {
        ++attempts;
        int64_t u = (int64_t)rng.randbelow((uint64_t)n);
        int64_t v = (int64_t)rng.randbelow((uint64_t)n);
        add(u, v);
    }
    return got;
}

// generate_updates (generate.py:107-161).  kind 'd' / 'a'; out arrays hold
// at least ceil(percent/100 * m) records; returns the count.
__attribute__((visibility("default"))) int64_t gdgen_py_updates(const int64_t* esrc, const int64_t* edst,
                                                                const int64_t* ew, int64_t m, int64_t node_count,
                                                                double percent, uint64_t seed, double add_fraction,
                                                                int undirected, uint8_t* kind, int64_t* us,
                                                                int64_t* ud, int64_t* uw) {
    PyRandom rng(seed);
    const int64_t count = (int64_t)std::ceil(percent / 100.0 * (double)m);
    const int64_t n_adds = (int64_t)std::nearbyint((double)count * add_fraction);  // round half to even
    int64_t n_dels = count - n_adds;
    PairSet existing((size_t)m);
    std::vector<uint64_t> pool;  // dict.fromkeys: distinct pairs in first-seen order
    pool.reserve((size_t)m);
    int64_t max_weight = 1;
    bool any = false;
    for (int64_t i = 0; i < m; ++i) {
        uint64_t k = pkey((uint64_t)esrc[i], (uint64_t)edst[i], undirected);
        if (existing.insert(k)) pool.push_back(k);
        max_weight = any ? std::max(max_weight, ew[i]) : ew[i];
        any = true;
    }
    const int64_t npool = (int64_t)pool.size();
    if (n_dels > npool) n_dels = npool;
    // rng.sample(pool, n_dels) (Lib/random.py: pool or set selection)
    std::vector<uint64_t> dels((size_t)n_dels);
    int64_t setsize = 21;
    if (n_dels > 5) setsize += (int64_t)std::pow(4.0, std::ceil(std::log((double)(n_dels * 3)) / std::log(4.0)));
    if (npool <= setsize) {
        std::vector<uint64_t> p(pool);
        for (int64_t i = 0; i < n_dels; ++i) {
            uint64_t j = rng.randbelow((uint64_t)(npool - i));
            dels[i] = p[j];
            p[j] = p[npool - i - 1];
        }
    } else {
        PairSet selected((size_t)n_dels);
        for (int64_t i = 0; i < n_dels; ++i) {
            uint64_t j = rng.randbelow((uint64_t)npool);
            while (!selected.insert(j)) j = rng.randbelow((uint64_t)npool);
            dels[i] = pool[j];
        }
    }
    PairSet chosen((size_t)n_adds);
    std::vector<uint64_t> adds;
    adds.reserve((size_t)n_adds);
    int64_t attempts = 0;
    const int64_t limit = 200 * (n_adds > 1 ? n_adds : 1) + 1000;
    while ((int64_t)adds.size() < n_adds && attempts < limit) {
        ++attempts;
        uint64_t u = rng.randbelow((uint64_t)node_count), v = rng.randbelow((uint64_t)node_count);
        if (u == v) continue;
        uint64_t k = pkey(u, v, undirected);
        if (existing.contains(k) || chosen.contains(k)) continue;
        chosen.insert(k);
        adds.push_back((u << 32) | v);  // the drawn orientation, not the normalised key
    }
    int64_t total = 0;
    for (uint64_t k : dels) {
        kind[total] = 'd';
        us[total] = (int64_t)(k >> 32);
        ud[total] = (int64_t)(k & 0xffffffffULL);
        uw[total] = 1;
        ++total;
    }
    for (uint64_t k : adds) {
        kind[total] = 'a';
        us[total] = (int64_t)(k >> 32);
        ud[total] = (int64_t)(k & 0xffffffffULL);
        uw[total] = rng.randint(1, max_weight);
        ++total;
    }
    for (int64_t i = total - 1; i >= 1; --i) {  // rng.shuffle(records)
        int64_t j = (int64_t)rng.randbelow((uint64_t)i + 1);
        std::swap(kind[i], kind[j]);
        std::swap(us[i], us[j]);
        std::swap(ud[i], ud[j]);
        std::swap(uw[i], uw[j]);
    }
    return total;
}

}  // extern "C"
