// hsde_cover.cpp -- the covered-coordinate layout of a reference-layout problem
// (host, multi-threaded; no GPU).  A reference `DecomposedProblem` carries x over
// all n^2 coordinates (chordalsdp/decompose.py:40-79: dense c, A with n^2
// columns); the device path iterates only on the *covered* ones: those a clique
// selects (graphs.py:228, D > 0), plus the column support of A and the support of
// c.  This builds, for `problem.compress`:
//   covered[k]   ascending flat ids,
//   c_cov[k]     = c[covered[k]],
//   pos[e]       = rank of A's column id e in covered,
//   slot_cov[j]  = rank of gather_index[j] in covered,
// from a bit mask over n^2 (n^2 / 8 bytes) with a popcount prefix per 64-bit
// word, instead of sorting ~nnz(A) ids or a 4 n^2-byte rank map.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "../../include/hsde.h"

namespace {

struct Cover {
  int64_t n2 = 0, n_cov = 0;
  std::vector<uint64_t> bits;   // bit i of word w: coordinate 64 w + i is covered
  std::vector<int64_t> prefix;  // covered coordinates before word w
  int threads = 1;
};

template <class F>
void parallel_for(int threads, int64_t n, F f) {  // f(t, begin, end) on contiguous chunks
  if (threads <= 1 || n < (int64_t)1 << 16) {
    f(0, (int64_t)0, n);
    return;
  }
  const int64_t per = (n + threads - 1) / threads;
  std::vector<std::thread> th;
  for (int t = 1; t < threads; ++t) {
    const int64_t b = std::min(n, t * per), e = std::min(n, b + per);
    if (b < e) th.emplace_back([=] { f(t, b, e); });
  }
  f(0, (int64_t)0, std::min(n, per));
  for (auto &x : th) x.join();
}

inline void set_bit(uint64_t *bits, int64_t i) {
  __atomic_fetch_or(bits + (i >> 6), (uint64_t)1 << (i & 63), __ATOMIC_RELAXED);
}

inline int64_t rank_of(const Cover &c, int64_t i) {
  const uint64_t w = c.bits[i >> 6], below = w & (((uint64_t)1 << (i & 63)) - 1);
  return c.prefix[i >> 6] + __builtin_popcountll(below);
}

}  // namespace

extern "C" {

int hsde_cover_build(int64_t n2, const double *c_full, const int64_t *gather_index, int64_t n_gather,
                     const int32_t *a_col32, const int64_t *a_col64, int64_t nnz, hsde_cover_t **out,
                     int64_t *n_cov) {
  if (!out || !n_cov || n2 < 0 || n_gather < 0 || nnz < 0 || (n2 > 0 && !c_full) ||
      (n_gather > 0 && !gather_index) || (nnz > 0 && !a_col32 && !a_col64))
    return HSDE_ERR_ARG;
  Cover *c = new Cover;
  c->n2 = n2;
  const int64_t nw = (n2 + 63) >> 6;
  c->bits.assign((size_t)nw, 0);
  c->prefix.assign((size_t)nw + 1, 0);
  c->threads = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  uint64_t *bits = c->bits.data();
  std::atomic<int> bad{0};
  // support of c: each thread owns whole words
  parallel_for(c->threads, nw, [&](int, int64_t wb, int64_t we) {
    for (int64_t w = wb; w < we; ++w) {
      const int64_t i0 = w << 6, i1 = std::min(n2, i0 + 64);
      uint64_t m = 0;
      for (int64_t i = i0; i < i1; ++i) m |= (uint64_t)(c_full[i] != 0.0) << (i - i0);
      bits[w] = m;
    }
  });
  // clique-selected coordinates and A's column support (atomic or: threads share words)
  parallel_for(c->threads, n_gather, [&](int, int64_t b, int64_t e) {
    for (int64_t j = b; j < e; ++j) {
      const int64_t i = gather_index[j];
      if (i < 0 || i >= n2) {
        bad = 1;
        continue;
      }
      set_bit(bits, i);
    }
  });
  parallel_for(c->threads, nnz, [&](int, int64_t b, int64_t e) {
    for (int64_t k = b; k < e; ++k) {
      const int64_t i = a_col32 ? (int64_t)a_col32[k] : a_col64[k];
      if (i < 0 || i >= n2) {
        bad = 1;
        continue;
      }
      set_bit(bits, i);
    }
  });
  if (bad) {
    delete c;
    return HSDE_ERR_ARG;
  }
  // popcount prefix: per-chunk counts (chunk t of parallel_for), then offsets
  std::vector<int64_t> chunk(c->threads + 1, 0);
  parallel_for(c->threads, nw, [&](int t, int64_t wb, int64_t we) {
    int64_t s = 0;
    for (int64_t w = wb; w < we; ++w) s += __builtin_popcountll(bits[w]);
    chunk[t + 1] = s;
  });
  for (int t = 0; t < c->threads; ++t) chunk[t + 1] += chunk[t];
  parallel_for(c->threads, nw, [&](int t, int64_t wb, int64_t we) {
    int64_t s = chunk[t];
    for (int64_t w = wb; w < we; ++w) {
      c->prefix[w] = s;
      s += __builtin_popcountll(bits[w]);
    }
  });
  const int64_t total = nw ? c->prefix[nw - 1] + __builtin_popcountll(bits[nw - 1]) : 0;
  c->prefix[nw] = total;
  c->n_cov = total;
  *n_cov = total;
  *out = reinterpret_cast<hsde_cover_t *>(c);
  return HSDE_OK;
}

int hsde_cover_fill(const hsde_cover_t *cv, const double *c_full, const int64_t *gather_index, int64_t n_gather,
                    const int32_t *a_col32, const int64_t *a_col64, int64_t nnz, int64_t *covered,
                    double *c_cov, int32_t *pos, int32_t *slot_cov) {
  const Cover *c = reinterpret_cast<const Cover *>(cv);
  if (!c || (c->n_cov > 0 && (!covered || !c_cov || !c_full)) || (nnz > 0 && !pos) ||
      (n_gather > 0 && !slot_cov) || c->n_cov >= ((int64_t)1 << 31))
    return HSDE_ERR_ARG;
  const int64_t nw = (c->n2 + 63) >> 6;
  const uint64_t *bits = c->bits.data();
  parallel_for(c->threads, nw, [&](int, int64_t wb, int64_t we) {
    for (int64_t w = wb; w < we; ++w) {
      uint64_t m = bits[w];
      int64_t k = c->prefix[w];
      while (m) {
        const int64_t i = (w << 6) + __builtin_ctzll(m);
        covered[k] = i;
        c_cov[k] = c_full[i];
        ++k;
        m &= m - 1;
      }
    }
  });
  parallel_for(c->threads, nnz, [&](int, int64_t b, int64_t e) {
    for (int64_t k = b; k < e; ++k) pos[k] = (int32_t)rank_of(*c, a_col32 ? (int64_t)a_col32[k] : a_col64[k]);
  });
  parallel_for(c->threads, n_gather, [&](int, int64_t b, int64_t e) {
    for (int64_t j = b; j < e; ++j) slot_cov[j] = (int32_t)rank_of(*c, gather_index[j]);
  });
  return HSDE_OK;
}

void hsde_cover_destroy(hsde_cover_t *cv) { delete reinterpret_cast<Cover *>(cv); }

}  // extern "C"
