// debug_api.cuh -- step-level entry points (one per hot-path row).
// Included at the end of sr_sort.cu: they drive the same kernels and the same
// Sorter machinery as sr_sort_keys / sr_sort_pairs, one step at a time, and
// synchronise the stream before returning.

namespace {

template <typename F>
int32_t step_call(void* stream, F&& f) {
  return guarded([&] {
    init_pool();
    Ctx c((cudaStream_t)stream);
    f(c);
    check_cuda(cudaStreamSynchronize(c.st), "cudaStreamSynchronize");
  });
}

bool ok_dtype(int32_t d) { return d == SR_INT32 || d == SR_INT64; }

template <typename K>
void presort_scan_t(Ctx& c, const K* keys, int64_t n, int strict, int tile, sr_presort_stats* hs_out, int64_t* rows,
                    int64_t cap) {
  const int64_t G = ceil_div<int64_t>(n, tile);
  TileSummary* d_sums = c.alloc<TileSummary>(G);
  RunDesc* d_asc = c.alloc<RunDesc>(G + 1);
  RunDesc* d_desc = c.alloc<RunDesc>(G + 1);
  DevStats* d_st = c.alloc<DevStats>(1);
  c.memset0(d_st, sizeof(DevStats));
  c.launch("presort_scan", n * sizeof(K), [&] {
    if (strict)
      k_presort_scan<K, true, false, 256><<<(unsigned)G, 256, 0, c.st>>>(keys, n, tile, d_sums, nullptr, nullptr,
                                                                         nullptr, nullptr, 0, (int)G, nullptr, nullptr, nullptr);
    else
      k_presort_scan<K, false, false, 256><<<(unsigned)G, 256, 0, c.st>>>(keys, n, tile, d_sums, nullptr, nullptr,
                                                                          nullptr, nullptr, 0, (int)G, nullptr, nullptr, nullptr);
  });
  c.launch("presort_resolve", G * 32, [&] {
    k_presort_resolve<K, 1024><<<1, 1024, 0, c.st>>>(keys, n, d_sums, (int)G, tile, d_asc, d_desc, d_st, 0, 1, nullptr);
  });
  DevStats hs = *reinterpret_cast<DevStats*>(c.readback(d_st, sizeof(DevStats)));
  hs_out->n = hs.n;
  hs_out->descents = hs.descents;
  hs_out->asc_breaks = hs.asc_breaks;
  hs_out->n_asc_runs = hs.n_asc_runs;
  hs_out->n_desc_runs = hs.n_desc_runs;
  hs_out->asc_cover = hs.asc_cover;
  hs_out->desc_cover = hs.desc_cover;
  if (rows && cap > 0) {
    std::vector<RunDesc> asc(hs.n_asc_runs), desc(hs.n_desc_runs);
    if (hs.n_asc_runs)
      check_cuda(cudaMemcpy(asc.data(), d_asc, sizeof(RunDesc) * hs.n_asc_runs, cudaMemcpyDeviceToHost), "d2h");
    if (hs.n_desc_runs)
      check_cuda(cudaMemcpy(desc.data(), d_desc, sizeof(RunDesc) * hs.n_desc_runs, cudaMemcpyDeviceToHost), "d2h");
    int64_t k = 0;
    for (auto& r : asc) if (k < cap) { rows[4 * k] = r.start; rows[4 * k + 1] = r.len; rows[4 * k + 2] = 0; rows[4 * k + 3] = 0; k++; }
    for (auto& r : desc) if (k < cap) { rows[4 * k] = r.start; rows[4 * k + 1] = r.len; rows[4 * k + 2] = 1; rows[4 * k + 3] = 0; k++; }
  }
}

template <typename K, bool HAS_V>
void tile_sort_t(Ctx& c, K* keys, uint32_t* vals, int64_t n, int tile) {
  Sorter<K, HAS_V> s(c, keys, vals, n);
  std::vector<Item> items;
  for (int64_t p = 0; p < n; p += tile) items.push_back(Item{p, 0, (int32_t)std::min<int64_t>(tile, n - p), kItemSort});
  Item* d_items = c.alloc<Item>(items.size());
  int64_t* d_cnt = c.alloc<int64_t>(1);
  c.upload(d_items, items);
  std::vector<int64_t> cnt{(int64_t)items.size()};
  c.upload(d_cnt, cnt);
  s.finish(d_items, d_cnt, 0, (int64_t)items.size(), 2 * n * (sizeof(K) + (HAS_V ? 4 : 0)));
}

template <typename K, bool HAS_V>
void merge_t(Ctx& c, const K* a, const uint32_t* va, int64_t na, const K* b, const uint32_t* vb, int64_t nb, K* out,
             uint32_t* vout) {
  const int64_t n = na + nb;
  Sorter<K, HAS_V> s(c, out, vout, n);
  s.ensure_ws();
  check_cuda(cudaMemcpyAsync(s.wk, a, na * sizeof(K), cudaMemcpyDeviceToDevice, c.st), "d2d");
  check_cuda(cudaMemcpyAsync(s.wk + na, b, nb * sizeof(K), cudaMemcpyDeviceToDevice, c.st), "d2d");
  if (HAS_V) {
    check_cuda(cudaMemcpyAsync(s.wv, va, na * 4, cudaMemcpyDeviceToDevice, c.st), "d2d");
    check_cuda(cudaMemcpyAsync(s.wv + na, vb, nb * 4, cudaMemcpyDeviceToDevice, c.st), "d2d");
  }
  MergeJob j{0, na, nb, 0, 1, 0};
  std::vector<MergeJob> jobs{j};
  s.run_merges(jobs, ceil_div<int64_t>(n, kMergeNV), 2 * n * (sizeof(K) + (HAS_V ? 4 : 0)));
}

template <typename K>
void splitters_t(Ctx& c, const K* keys, int64_t n, int nb, int64_t* hspl, uint8_t* heq, int32_t* m) {
  Sorter<K, false> s(c, const_cast<K*>(keys), nullptr, n);
  typename Sorter<K, false>::Level L;
  std::vector<OvfSeg> whole{{0, n}};
  s.level_alloc(L, whole, choose_tile(n), 0, nb);
  s.level_splitters(L);
  int mm = *reinterpret_cast<int*>(c.readback(L.d_m, sizeof(int)));
  std::vector<K> spl(std::max(mm, 1));
  std::vector<uint8_t> eq(std::max(mm, 1));
  if (mm) {
    check_cuda(cudaMemcpy(spl.data(), L.d_spl, mm * sizeof(K), cudaMemcpyDeviceToHost), "d2h");
    check_cuda(cudaMemcpy(eq.data(), L.d_eq, mm, cudaMemcpyDeviceToHost), "d2h");
  }
  for (int i = 0; i < mm; i++) { hspl[i] = (int64_t)spl[i]; heq[i] = eq[i]; }
  *m = mm;
}

template <typename K, bool HAS_V>
void partition_level_t(Ctx& c, const K* keys, const uint32_t* vals, int64_t n, int nbk, K* out, uint32_t* vout,
                       int64_t* counts) {
  // primary = out, workspace = a copy of the input; the level reads the
  // workspace (src = 1) and scatters into out.
  Sorter<K, HAS_V> s(c, out, vout, n);
  s.ensure_ws();
  check_cuda(cudaMemcpyAsync(s.wk, keys, n * sizeof(K), cudaMemcpyDeviceToDevice, c.st), "d2d");
  if (HAS_V) check_cuda(cudaMemcpyAsync(s.wv, vals, n * 4, cudaMemcpyDeviceToDevice, c.st), "d2d");
  typename Sorter<K, HAS_V>::Level L;
  std::vector<OvfSeg> whole{{0, n}};
  int64_t cs = std::min<int64_t>(65536, std::max<int64_t>(4096, pow2ceil(std::max<int64_t>(1, n / 512))));
  s.level_alloc(L, whole, cs, 1, nbk);
  s.level_splitters(L);
  s.level_count(L);
  s.level_scan_plan(L);
  DevStats hs = *reinterpret_cast<DevStats*>(c.readback(L.d_st, sizeof(DevStats)));
  if (hs.error) fail(SR_ERR_INTERNAL, "plan kernel inconsistency");
  DevStats forced = hs;
  forced.noneq_total = 1;  // never skip: the step must write every range key
  s.level_scatter(L, &forced);
  // fill the equality buckets' keys (the scatter moves only their payloads)
  std::vector<Item> items(hs.n_items);
  if (hs.n_items)
    check_cuda(cudaMemcpy(items.data(), L.d_items, sizeof(Item) * hs.n_items, cudaMemcpyDeviceToHost), "d2h");
  std::vector<Item> fills;
  for (auto& it : items)
    if ((it.kind & 0xf) == kItemFill) fills.push_back(it);
  if (!fills.empty()) {
    Item* d_items = c.alloc<Item>(fills.size());
    int64_t* d_cnt = c.alloc<int64_t>(1);
    c.upload(d_items, fills);
    std::vector<int64_t> cnt{(int64_t)fills.size()};
    c.upload(d_cnt, cnt);
    s.finish(d_items, d_cnt, 0, (int64_t)fills.size(), 0);
  }
  const SegDesc& sd = L.segs[0];
  if (L.atomic) {  // keys only: bucket totals
    std::vector<uint32_t> tot(sd.nbins);
    check_cuda(cudaMemcpy(tot.data(), L.d_tot, tot.size() * 4, cudaMemcpyDeviceToHost), "d2h");
    for (int b = 0; b < 2 * nbk + 1; b++) counts[b] = b < sd.nbins ? tot[b] : 0;
    return;
  }
  // bucket counts from the scanned matrix (first chunk column of every bin)
  std::vector<uint32_t> mat((size_t)sd.nbins * sd.nchunks);
  check_cuda(cudaMemcpy(mat.data(), L.d_mat, mat.size() * 4, cudaMemcpyDeviceToHost), "d2h");
  for (int b = 0; b < 2 * nbk + 1; b++) {
    int64_t p0 = b < sd.nbins ? (int64_t)mat[(size_t)b * sd.nchunks] : n;
    int64_t p1 = b + 1 < sd.nbins ? (int64_t)mat[(size_t)(b + 1) * sd.nchunks] : n;
    counts[b] = p1 - p0;
  }
}

}  // namespace

extern "C" {

int32_t sr_presort_scan(const void* keys, int64_t n, int32_t dtype, int32_t strict, int32_t tile,
                        sr_presort_stats* hs, int64_t* host_runs, int64_t cap, void* stream) {
  if (!ok_dtype(dtype)) return SR_ERR_UNSUPPORTED_DTYPE;
  if (!hs || n < 1 || !keys || tile < 1024 || tile > 65536 || (tile & (tile - 1))) return SR_ERR_INVALID_ARGUMENT;
  return step_call(stream, [&](Ctx& c) {
    if (dtype == SR_INT32) presort_scan_t<int32_t>(c, (const int32_t*)keys, n, strict, tile, hs, host_runs, cap);
    else presort_scan_t<int64_t>(c, (const int64_t*)keys, n, strict, tile, hs, host_runs, cap);
  });
}

int32_t sr_reverse_range(void* keys, void* vals, int64_t n, int32_t dtype, int64_t s, int64_t e, void* stream) {
  if (!ok_dtype(dtype)) return SR_ERR_UNSUPPORTED_DTYPE;
  if (!keys || s < 0 || e > n || s > e) return SR_ERR_INVALID_ARGUMENT;
  if (e - s < 2) return SR_OK;
  return step_call(stream, [&](Ctx& c) {
    std::vector<RunDesc> r{RunDesc{s, e - s, 0, 0}};
    if (dtype == SR_INT32) {
      if (vals) Sorter<int32_t, true>(c, (int32_t*)keys, (uint32_t*)vals, n).reverse_ranges(r);
      else Sorter<int32_t, false>(c, (int32_t*)keys, nullptr, n).reverse_ranges(r);
    } else {
      if (vals) Sorter<int64_t, true>(c, (int64_t*)keys, (uint32_t*)vals, n).reverse_ranges(r);
      else Sorter<int64_t, false>(c, (int64_t*)keys, nullptr, n).reverse_ranges(r);
    }
  });
}

int32_t sr_tile_sort(void* keys, void* vals, int64_t n, int32_t dtype, int32_t tile, void* stream) {
  if (!ok_dtype(dtype)) return SR_ERR_UNSUPPORTED_DTYPE;
  if (!keys || n < 0 || tile < 1 || tile > kCap) return SR_ERR_INVALID_ARGUMENT;
  if (n == 0) return SR_OK;
  return step_call(stream, [&](Ctx& c) {
    if (dtype == SR_INT32) {
      if (vals) tile_sort_t<int32_t, true>(c, (int32_t*)keys, (uint32_t*)vals, n, tile);
      else tile_sort_t<int32_t, false>(c, (int32_t*)keys, nullptr, n, tile);
    } else {
      if (vals) tile_sort_t<int64_t, true>(c, (int64_t*)keys, (uint32_t*)vals, n, tile);
      else tile_sort_t<int64_t, false>(c, (int64_t*)keys, nullptr, n, tile);
    }
  });
}

int32_t sr_merge_path(const void* a, int64_t na, const void* b, int64_t nb, int32_t dtype, const int64_t* diags,
                      int64_t* out, int64_t nd, void* stream) {
  if (!ok_dtype(dtype)) return SR_ERR_UNSUPPORTED_DTYPE;
  if (na < 0 || nb < 0 || nd < 0 || (nd && (!diags || !out))) return SR_ERR_INVALID_ARGUMENT;
  for (int64_t i = 0; i < nd; i++)
    if (diags[i] < 0 || diags[i] > na + nb) return SR_ERR_INVALID_ARGUMENT;
  if (nd == 0) return SR_OK;
  return step_call(stream, [&](Ctx& c) {
    int64_t* d_diag = c.alloc<int64_t>(nd);
    int64_t* d_out = c.alloc<int64_t>(nd);
    std::vector<int64_t> dg(diags, diags + nd);
    c.upload(d_diag, dg);
    unsigned grid = (unsigned)ceil_div<int64_t>(nd, 256);
    c.launch("merge_path", 0, [&] {
      if (dtype == SR_INT32)
        k_merge_path_diags<int32_t><<<grid, 256, 0, c.st>>>((const int32_t*)a, na, (const int32_t*)b, nb, d_diag, nd, d_out);
      else
        k_merge_path_diags<int64_t><<<grid, 256, 0, c.st>>>((const int64_t*)a, na, (const int64_t*)b, nb, d_diag, nd, d_out);
    });
    check_cuda(cudaMemcpyAsync(out, d_out, nd * 8, cudaMemcpyDeviceToHost, c.st), "d2h");
  });
}

int32_t sr_merge(const void* a, const void* va, int64_t na, const void* b, const void* vb, int64_t nb, void* out,
                 void* vout, int32_t dtype, void* stream) {
  if (!ok_dtype(dtype)) return SR_ERR_UNSUPPORTED_DTYPE;
  if (na < 0 || nb < 0 || (na + nb > 0 && !out)) return SR_ERR_INVALID_ARGUMENT;
  const bool pv = vout != nullptr;
  if (pv && ((na && !va) || (nb && !vb))) return SR_ERR_INVALID_ARGUMENT;
  if (na + nb == 0) return SR_OK;
  return step_call(stream, [&](Ctx& c) {
    if (dtype == SR_INT32) {
      if (pv) merge_t<int32_t, true>(c, (const int32_t*)a, (const uint32_t*)va, na, (const int32_t*)b, (const uint32_t*)vb, nb, (int32_t*)out, (uint32_t*)vout);
      else merge_t<int32_t, false>(c, (const int32_t*)a, nullptr, na, (const int32_t*)b, nullptr, nb, (int32_t*)out, nullptr);
    } else {
      if (pv) merge_t<int64_t, true>(c, (const int64_t*)a, (const uint32_t*)va, na, (const int64_t*)b, (const uint32_t*)vb, nb, (int64_t*)out, (uint32_t*)vout);
      else merge_t<int64_t, false>(c, (const int64_t*)a, nullptr, na, (const int64_t*)b, nullptr, nb, (int64_t*)out, nullptr);
    }
  });
}

int32_t sr_splitters(const void* keys, int64_t n, int32_t dtype, int32_t nbuckets, int64_t* hspl, uint8_t* heq,
                     int32_t* m, void* stream) {
  if (!ok_dtype(dtype)) return SR_ERR_UNSUPPORTED_DTYPE;
  if (!keys || n < 1 || !hspl || !heq || !m || nbuckets < 2 || nbuckets > kMaxBuckets || (nbuckets & (nbuckets - 1)))
    return SR_ERR_INVALID_ARGUMENT;
  return step_call(stream, [&](Ctx& c) {
    if (dtype == SR_INT32) splitters_t<int32_t>(c, (const int32_t*)keys, n, nbuckets, hspl, heq, m);
    else splitters_t<int64_t>(c, (const int64_t*)keys, n, nbuckets, hspl, heq, m);
  });
}

int32_t sr_partition_level(const void* keys, const void* vals, int64_t n, int32_t dtype, int32_t nbuckets, void* out,
                           void* vout, int64_t* counts, void* stream) {
  if (!ok_dtype(dtype)) return SR_ERR_UNSUPPORTED_DTYPE;
  if (!keys || !out || n < 1 || !counts || nbuckets < 2 || nbuckets > kMaxBuckets || (nbuckets & (nbuckets - 1)))
    return SR_ERR_INVALID_ARGUMENT;
  if ((vals == nullptr) != (vout == nullptr)) return SR_ERR_INVALID_ARGUMENT;
  return step_call(stream, [&](Ctx& c) {
    if (dtype == SR_INT32) {
      if (vals) partition_level_t<int32_t, true>(c, (const int32_t*)keys, (const uint32_t*)vals, n, nbuckets, (int32_t*)out, (uint32_t*)vout, counts);
      else partition_level_t<int32_t, false>(c, (const int32_t*)keys, nullptr, n, nbuckets, (int32_t*)out, nullptr, counts);
    } else {
      if (vals) partition_level_t<int64_t, true>(c, (const int64_t*)keys, (const uint32_t*)vals, n, nbuckets, (int64_t*)out, (uint32_t*)vout, counts);
      else partition_level_t<int64_t, false>(c, (const int64_t*)keys, nullptr, n, nbuckets, (int64_t*)out, nullptr, counts);
    }
  });
}

}  // extern "C"
