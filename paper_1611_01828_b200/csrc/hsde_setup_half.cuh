// hsde_setup_half.cuh -- device construction of the symmetric half-pass
// layouts (DevProblem::half).  Included by hsde_capi.cu inside its anonymous
// namespace (uses hsde_handle, ShardDev, dalloc, pool_malloc, CK / RC).
//
// The covered coordinates come in mirror pairs {(i, j), (j, i)}; a clique
// slot (a, b) and its transpose slot (b, a) cover the two members of a pair.
// An SDP's constraint matrices are symmetric, so column l of A equals column
// mirror(l) exactly -- checked here; any mismatch (or an ownership split of a
// pair across shards) leaves the full-column passes in place.
//
//   pairs      representatives l <= mirror(l), ascending
//   SELL-32    A' g: slice of 32 pairs, element k of lane j at beg + 32 k + j,
//              16-bit row index, zero padded to the slice's longest column;
//              pairs sorted by column length within windows of kSellSigma
//              (SELL-C-sigma: padding 1.48 -> 1.02 on config 4)
//   row-SELL   A t: tiles of kRowTile pairs x groups of 32 rows, element k of
//              row position 32 g + j at beg + 32 k + j, 16-bit column within the
//              tile, entries of the owned pairs only, ascending column in a row;
//              rows sorted by their tile length within the tile

__global__ void k_mirror_map(DevProblem P, int *mir) {
  for (int k = blockIdx.x; k < P.p; k += gridDim.x) {
    const int d = P.cl_size[k];
    const int64_t off = P.cl_off[k];
    for (int e = threadIdx.x; e < d * d; e += blockDim.x) {
      const int a = e / d, b = e - a * d;
      mir[P.slot_cov[off + e]] = P.slot_cov[off + (int64_t)b * d + a];
    }
  }
}

// bit 0: mirror map inconsistent; bit 1: some column differs from its
// mirror's; bit 2: a pair split across shards
__global__ void k_half_check(DevProblem P, const int *mir, int *flag, int *rep) {
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < P.n_c; l += gridDim.x * blockDim.x) {
    const int q = mir[l];
    int f = 0;
    if (q < 0 || q >= P.n_c || mir[q] != l) {
      f = 1;
    } else {
      if (P.owned && P.owned[l] != P.owned[q]) f |= 4;
      if (l < q) {
        const int64_t b0 = P.at_cp[l], n0 = P.at_cp[l + 1] - b0;
        const int64_t b1 = P.at_cp[q], n1 = P.at_cp[q + 1] - b1;
        if (n0 != n1) {
          f |= 2;
        } else {
          for (int64_t k = 0; k < n0; ++k)
            if (P.at_row[b0 + k] != P.at_row[b1 + k] || P.at_val[b0 + k] != P.at_val[b1 + k]) {
              f |= 2;
              break;
            }
        }
      }
    }
    if (f) atomicOr(flag, f);
    rep[l] = (q >= l) ? 1 : 0;
  }
}

__global__ void k_pair_list(int n_c, const int *mir, const int *rep, const int *pos, int *pl, int *pm) {
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < n_c; l += gridDim.x * blockDim.x)
    if (rep[l]) {
      pl[pos[l]] = l;
      pm[pos[l]] = mir[l];
    }
}

// per pair: column length, owned-entry count, and the SELL sort key
// (window, descending length)
__global__ void k_pair_lengths(DevProblem P, const int *pl, int n_pair, int *plen, int *own_len,
                               unsigned *key, int *idx) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n_pair; q += gridDim.x * blockDim.x) {
    const int l = pl[q];
    const int len = (int)(P.at_cp[l + 1] - P.at_cp[l]);
    plen[q] = len;
    own_len[q] = owns(P, l) ? len : 0;
    key[q] = ((unsigned)(q / kSellSigma) << 16) | (unsigned)(65535 - len);
    idx[q] = q;
  }
}

// SELL order: pair of position p, its length; slice widths (32 * longest)
__global__ void k_sell_order(const int *perm, const int *pl, const int *pm, const int *plen, int n_pair,
                             int *sl_pl, int *sl_pm, int64_t *slice_w) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int n_slice = (n_pair + 31) >> 5;
  for (int sl = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; sl < n_slice; sl += warps) {
    const int p = sl * 32 + lane;
    int len = 0;
    if (p < n_pair) {
      const int q = perm[p];
      sl_pl[p] = pl[q];
      sl_pm[p] = pm[q];
      len = plen[q];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) len = max(len, __shfl_xor_sync(0xffffffffu, len, o));
    if (lane == 0) slice_w[sl] = 32 * (int64_t)len;
  }
}

__global__ void k_fill_sell(DevProblem P, const int *sl_pl, int n_pair, const int64_t *sl_beg,
                            uint16_t *sl_row, double *sl_val) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n_pair; q += gridDim.x * blockDim.x) {
    const int l = sl_pl[q];
    const int64_t cb = P.at_cp[l], n = P.at_cp[l + 1] - cb;
    const int64_t base = sl_beg[q >> 5] + (q & 31);
    for (int64_t k = 0; k < n; ++k) {
      sl_row[base + 32 * k] = (uint16_t)P.at_row[cb + k];
      sl_val[base + 32 * k] = P.at_val[cb + k];
    }
  }
}

// entries of the owned pairs with key (tile * m + row) << 12 | column-in-tile
__global__ void k_row_keys(DevProblem P, const int *pl, int n_pair, const int *own_len,
                           const int64_t *epos, unsigned long long *keys, double *vals) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n_pair; q += gridDim.x * blockDim.x) {
    if (!own_len[q]) continue;
    const int l = pl[q];
    const int64_t cb = P.at_cp[l], n = P.at_cp[l + 1] - cb;
    const unsigned long long tile = (unsigned long long)(q / P.rt_tile);
    const unsigned long long lc = (unsigned long long)(q - (int)tile * P.rt_tile);
    for (int64_t k = 0; k < n; ++k) {
      const unsigned long long r = (unsigned long long)P.at_row[cb + k];
      keys[epos[q] + k] = ((tile * (unsigned long long)P.m + r) << 12) | lc;
      vals[epos[q] + k] = P.at_val[cb + k];
    }
  }
}

__global__ void k_cell_count(const unsigned long long *keys, int64_t n, int *cnt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(cnt + (keys[e] >> 12), 1);  // integer counts: order-independent
}

// row sort keys within each tile: (tile, descending count)
__global__ void k_row_keys_sort(const int *cnt, int m, int64_t ncell, unsigned long long *key, int *row) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncell;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = c / m;
    key[c] = ((unsigned long long)t << 32) | (unsigned long long)(0xffffffffu - (unsigned)cnt[c]);
    row[c] = (int)(c - t * m);
  }
}

// sorted rows -> inverse positions and the group widths (first row of a group
// is its longest)
__global__ void k_row_positions(const int *cnt, const int *rt_row, int m, int ntile, int G, int *rowpos,
                                int64_t *w) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < (int64_t)ntile * m;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = c / m;
    const int q = (int)(c - t * m);
    const int r = rt_row[c];
    rowpos[t * m + r] = q;
    if ((q & 31) == 0) w[t * G + (q >> 5)] = 32 * (int64_t)cnt[t * m + r];
  }
}

__global__ void k_fill_rows(const unsigned long long *keys, const double *vals, int64_t n, int m,
                            int G, const int64_t *cell_start, const int *rowpos, const int64_t *rt_beg,
                            uint16_t *rt_col, double *rt_val) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long c = keys[e] >> 12;
    const int t = (int)(c / (unsigned long long)m);
    const int q = rowpos[c];
    const int64_t rank = e - cell_start[c];
    const int64_t dst = rt_beg[(int64_t)t * G + (q >> 5)] + 32 * rank + (q & 31);
    rt_col[dst] = (uint16_t)(keys[e] & 4095ull);
    rt_val[dst] = vals[e];
  }
}

__global__ void k_widen(const int *in, int64_t *out, int64_t n) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    out[k] = in[k];
}

template <class T>
int excl_scan(hsde_handle *h, const T *in, T *out, int64_t n) {
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, (int)n, h->st);
  void *tmp = nullptr;
  CK(pool_malloc(h, &tmp, tb));
  cub::DeviceScan::ExclusiveSum(tmp, tb, in, out, (int)n, h->st);
  pool_free(h, tmp);
  return 0;
}

template <class T>
T d2h_one(hsde_handle *h, const T *p) {
  T v{};
  cudaMemcpyAsync(&v, p, sizeof(T), cudaMemcpyDeviceToHost, h->st);
  cudaStreamSynchronize(h->st);
  return v;
}

// Build the half-pass layouts of one shard; leaves P.half = 0 when the
// problem does not qualify.
int build_half(hsde_handle *h, ShardDev &s) {
  DevProblem &P = s.P;
  P.half = 0;
  const int n_c = P.n_c, m = P.m;
  if (std::getenv("HSDE_NO_HALF") || n_c == 0 || m == 0 || m > 12288 || P.nnz == 0) return 0;
  int *mir = nullptr, *flag = nullptr, *rep = nullptr, *pos = nullptr;
  CK(pool_malloc(h, (void **)&mir, sizeof(int) * (n_c + 1)));
  CK(pool_malloc(h, (void **)&rep, sizeof(int) * (n_c + 1)));
  CK(pool_malloc(h, (void **)&pos, sizeof(int) * (n_c + 1)));
  CK(pool_malloc(h, (void **)&flag, sizeof(int)));
  CK(cudaMemsetAsync(mir, 0xff, sizeof(int) * n_c, h->st));
  CK(cudaMemsetAsync(flag, 0, sizeof(int), h->st));
  CK(cudaMemsetAsync(rep + n_c, 0, sizeof(int), h->st));
  k_mirror_map<<<std::min(P.p, 148 * 8), kBlock, 0, h->st>>>(P, mir);
  k_half_check<<<grid_for(n_c), kBlock, 0, h->st>>>(P, mir, flag, rep);
  CKL();
  const int bad = d2h_one(h, flag);
  if (bad) {
    pool_free(h, mir);
    pool_free(h, rep);
    pool_free(h, pos);
    pool_free(h, flag);
    return 0;
  }
  RC(excl_scan(h, rep, pos, (int64_t)n_c + 1));
  const int n_pair = d2h_one(h, pos + n_c);
  int *pl = nullptr, *pm = nullptr;
  RC(dalloc(h, &pl, n_pair));
  RC(dalloc(h, &pm, n_pair));
  k_pair_list<<<grid_for(n_c), kBlock, 0, h->st>>>(n_c, mir, rep, pos, pl, pm);
  CKL();
  pool_free(h, mir);
  pool_free(h, rep);
  pool_free(h, pos);
  pool_free(h, flag);
  // SELL-32 slices (A' g), pairs sorted by length within windows (stable)
  const int n_slice = (n_pair + 31) / 32;
  int64_t *sl_beg = nullptr;
  int *own_len = nullptr, *plen = nullptr, *pidx = nullptr, *perm = nullptr, *sl_pl = nullptr,
      *sl_pm = nullptr;
  unsigned *pkey = nullptr, *pkey_s = nullptr;
  int64_t *own_pos = nullptr, *slw = nullptr;
  RC(dalloc(h, &sl_beg, n_slice + 1));
  RC(dalloc(h, &sl_pl, n_pair));
  RC(dalloc(h, &sl_pm, n_pair));
  CK(pool_malloc(h, (void **)&slw, sizeof(int64_t) * (n_slice + 1)));
  CK(pool_malloc(h, (void **)&own_len, sizeof(int) * (n_pair + 1)));
  CK(pool_malloc(h, (void **)&own_pos, sizeof(int64_t) * (n_pair + 1)));
  CK(pool_malloc(h, (void **)&plen, sizeof(int) * (n_pair + 1)));
  CK(pool_malloc(h, (void **)&pidx, sizeof(int) * (n_pair + 1)));
  CK(pool_malloc(h, (void **)&perm, sizeof(int) * (n_pair + 1)));
  CK(pool_malloc(h, (void **)&pkey, sizeof(unsigned) * (n_pair + 1)));
  CK(pool_malloc(h, (void **)&pkey_s, sizeof(unsigned) * (n_pair + 1)));
  CK(cudaMemsetAsync(slw + n_slice, 0, sizeof(int64_t), h->st));
  CK(cudaMemsetAsync(own_len + n_pair, 0, sizeof(int), h->st));
  k_pair_lengths<<<grid_for(n_pair), kBlock, 0, h->st>>>(P, pl, n_pair, plen, own_len, pkey, pidx);
  CKL();
  {
    int kbits = 16;
    while ((1ll << (kbits - 16)) <= (long long)(n_pair / kSellSigma)) ++kbits;
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, pkey, pkey_s, pidx, perm, n_pair, 0, kbits, h->st);
    void *tmp = nullptr;
    CK(pool_malloc(h, &tmp, tb));
    cub::DeviceRadixSort::SortPairs(tmp, tb, pkey, pkey_s, pidx, perm, n_pair, 0, kbits, h->st);
    pool_free(h, tmp);
  }
  k_sell_order<<<grid_for((int64_t)n_slice * 32), kBlock, 0, h->st>>>(perm, pl, pm, plen, n_pair, sl_pl, sl_pm,
                                                                      slw);
  CKL();
  pool_free(h, plen);
  pool_free(h, pidx);
  pool_free(h, perm);
  pool_free(h, pkey);
  pool_free(h, pkey_s);
  RC(excl_scan(h, slw, sl_beg, (int64_t)n_slice + 1));
  const int64_t n_sell = d2h_one(h, sl_beg + n_slice);
  uint16_t *sl_row = nullptr;
  double *sl_val = nullptr;
  RC(dalloc(h, &sl_row, n_sell));
  RC(dalloc(h, &sl_val, n_sell));
  CK(cudaMemsetAsync(sl_row, 0, sizeof(uint16_t) * std::max<int64_t>(n_sell, 1), h->st));
  CK(cudaMemsetAsync(sl_val, 0, sizeof(double) * std::max<int64_t>(n_sell, 1), h->st));
  k_fill_sell<<<grid_for(n_pair), kBlock, 0, h->st>>>(P, sl_pl, n_pair, sl_beg, sl_row, sl_val);
  CKL();
  pool_free(h, slw);
  // row-SELL tiles (A t) over the owned pairs
  {
    int64_t *own_len64 = nullptr;
    CK(pool_malloc(h, (void **)&own_len64, sizeof(int64_t) * (n_pair + 1)));
    // widen the per-pair owned lengths for an int64 scan
    k_widen<<<grid_for(n_pair + 1), kBlock, 0, h->st>>>(own_len, own_len64, (int64_t)n_pair + 1);
    CKL();
    RC(excl_scan(h, own_len64, own_pos, (int64_t)n_pair + 1));
    pool_free(h, own_len64);
  }
  const int64_t n_ent = d2h_one(h, own_pos + n_pair);
  P.rt_tile = kRowTileDefault;
  P.rt_split = kRowTileSplit;
  {
    // small problems: smaller tiles and more CTAs per tile until the pass has
    // >= 2 CTAs per SM (config 0: 4 -> 48 CTAs, k_spmv_half 37 -> 19 us)
    const int G0 = (m + 31) / 32;
    while (P.rt_tile > 256 && (int64_t)((n_pair + P.rt_tile - 1) / P.rt_tile) * P.rt_split < 296) P.rt_tile /= 2;
    if ((int64_t)((n_pair + P.rt_tile - 1) / P.rt_tile) * P.rt_split < 296) P.rt_split = std::max(1, std::min(4, G0));
  }
  if (const char *e = std::getenv("HSDE_RT_TILE")) P.rt_tile = std::max(256, std::min(kRowTile, atoi(e)));
  if (const char *e = std::getenv("HSDE_RT_SPLIT")) P.rt_split = std::max(1, std::min(16, atoi(e)));
  const int ntile = (n_pair + P.rt_tile - 1) / P.rt_tile, G = (m + 31) / 32;
  unsigned long long *keys = nullptr, *keys_s = nullptr;
  double *vals = nullptr, *vals_s = nullptr;
  const int64_t ne = std::max<int64_t>(n_ent, 1);
  CK(pool_malloc(h, (void **)&keys, sizeof(unsigned long long) * ne));
  CK(pool_malloc(h, (void **)&keys_s, sizeof(unsigned long long) * ne));
  CK(pool_malloc(h, (void **)&vals, sizeof(double) * ne));
  CK(pool_malloc(h, (void **)&vals_s, sizeof(double) * ne));
  k_row_keys<<<grid_for(n_pair), kBlock, 0, h->st>>>(P, pl, n_pair, own_len, own_pos, keys, vals);
  CKL();
  pool_free(h, own_len);
  pool_free(h, own_pos);
  int end_bit = 12;
  while ((1ull << (end_bit - 12)) < (unsigned long long)ntile * m) ++end_bit;
  if (n_ent > INT32_MAX) {
    h->err = "too many constraint nonzeros for the half-pass layout";
    return HSDE_ERR_ARG;
  }
  {
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys_s, vals, vals_s, (int)n_ent, 0, end_bit,
                                    h->st);
    void *tmp = nullptr;
    CK(pool_malloc(h, &tmp, tb));
    cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys_s, vals, vals_s, (int)n_ent, 0, end_bit,
                                    h->st);
    pool_free(h, tmp);
  }
  pool_free(h, keys);
  pool_free(h, vals);
  const int64_t ncell = (int64_t)ntile * m;
  int *cnt = nullptr;
  int64_t *cnt64 = nullptr, *cell_start = nullptr, *gw = nullptr, *rt_beg = nullptr;
  CK(pool_malloc(h, (void **)&cnt, sizeof(int) * (ncell + 1)));
  CK(pool_malloc(h, (void **)&cnt64, sizeof(int64_t) * (ncell + 1)));
  CK(pool_malloc(h, (void **)&cell_start, sizeof(int64_t) * (ncell + 1)));
  CK(pool_malloc(h, (void **)&gw, sizeof(int64_t) * ((int64_t)ntile * G + 1)));
  RC(dalloc(h, &rt_beg, (int64_t)ntile * G + 1));
  CK(cudaMemsetAsync(cnt, 0, sizeof(int) * (ncell + 1), h->st));
  CK(cudaMemsetAsync(gw + (int64_t)ntile * G, 0, sizeof(int64_t), h->st));
  k_cell_count<<<148 * 8, kBlock, 0, h->st>>>(keys_s, n_ent, cnt);
  k_widen<<<grid_for(ncell + 1), kBlock, 0, h->st>>>(cnt, cnt64, ncell + 1);
  CKL();
  // rows of each tile sorted by their entry count (descending, stable)
  int *rt_row = nullptr, *rowpos = nullptr, *ridx = nullptr;
  unsigned long long *rkey = nullptr, *rkey_s = nullptr;
  RC(dalloc(h, &rt_row, std::max<int64_t>(ncell, 1)));
  CK(pool_malloc(h, (void **)&rowpos, sizeof(int) * (ncell + 1)));
  CK(pool_malloc(h, (void **)&ridx, sizeof(int) * (ncell + 1)));
  CK(pool_malloc(h, (void **)&rkey, sizeof(unsigned long long) * (ncell + 1)));
  CK(pool_malloc(h, (void **)&rkey_s, sizeof(unsigned long long) * (ncell + 1)));
  k_row_keys_sort<<<grid_for(ncell), kBlock, 0, h->st>>>(cnt, m, ncell, rkey, ridx);
  CKL();
  {
    int kbits = 32;
    while ((1ll << (kbits - 32)) <= (long long)ntile) ++kbits;
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, rkey, rkey_s, ridx, rt_row, (int)ncell, 0, kbits, h->st);
    void *tmp = nullptr;
    CK(pool_malloc(h, &tmp, tb));
    cub::DeviceRadixSort::SortPairs(tmp, tb, rkey, rkey_s, ridx, rt_row, (int)ncell, 0, kbits, h->st);
    pool_free(h, tmp);
  }
  k_row_positions<<<grid_for(ncell), kBlock, 0, h->st>>>(cnt, rt_row, m, ntile, G, rowpos, gw);
  CKL();
  pool_free(h, ridx);
  pool_free(h, rkey);
  pool_free(h, rkey_s);
  RC(excl_scan(h, cnt64, cell_start, ncell + 1));
  RC(excl_scan(h, gw, rt_beg, (int64_t)ntile * G + 1));
  const int64_t n_rt = d2h_one(h, rt_beg + (int64_t)ntile * G);
  uint16_t *rt_col = nullptr;
  double *rt_val = nullptr;
  RC(dalloc(h, &rt_col, n_rt));
  RC(dalloc(h, &rt_val, n_rt));
  CK(cudaMemsetAsync(rt_col, 0, sizeof(uint16_t) * std::max<int64_t>(n_rt, 1), h->st));
  CK(cudaMemsetAsync(rt_val, 0, sizeof(double) * std::max<int64_t>(n_rt, 1), h->st));
  k_fill_rows<<<148 * 8, kBlock, 0, h->st>>>(keys_s, vals_s, n_ent, m, G, cell_start, rowpos, rt_beg,
                                             rt_col, rt_val);
  CKL();
  pool_free(h, rowpos);
  CK(cudaStreamSynchronize(h->st));
  pool_free(h, keys_s);
  pool_free(h, vals_s);
  pool_free(h, cnt);
  pool_free(h, cnt64);
  pool_free(h, cell_start);
  pool_free(h, gw);
  RC(dalloc(h, &s.W.rtpart, std::max<int64_t>(ncell, 1)));
  RC(dalloc(h, &s.W.xq, std::max(n_pair, 1)));
  P.n_pair = n_pair;
  P.pair_l = pl;
  P.pair_m = pm;
  P.n_slice = n_slice;
  P.sl_beg = sl_beg;
  P.sl_row = sl_row;
  P.sl_val = sl_val;
  P.sl_pl = sl_pl;
  P.sl_pm = sl_pm;
  P.rt_row = rt_row;
  P.rt_ntile = ntile;
  P.rt_G = G;
  P.rt_beg = rt_beg;
  P.rt_col = rt_col;
  P.rt_val = rt_val;
  P.half = 1;
  return 0;
}
