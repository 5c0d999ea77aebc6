// binsort.cu -- S0 on the device: bin-edge costs, the bin-major layout of the (cell, class) slots,
// the bin-start table, the three work-item lists (sorted larger first per window group) and the
// points themselves in bin-major order (north_star "bin sort").
//
// The host keeps only what sizes launches: it reads back the per-candidate statistics (to choose B,
// DESIGN.md §binning) and the per-group item counts.  Everything proportional to the cells, the bins
// or the items stays on the device:
//
//   k_bin_cand      slot counts -> per-bin counts of every candidate edge B      (atomics per occupied slot)
//   k_bin_stats     per (window, B): spreading chunks, occupied bins, largest bin
//   k_slot_keys     slot -> key in the bin-major order (bin, class, cell in bin); counts per key
//   [scan]          key offsets = sorted start of every slot (exclusive sum)
//   k_slot_cursor   the near-field cell table (start, count) per slot
//   k_bin_pass      bin starts; per-bin item counts (spreading chunks, per-bin interpolation chunks)
//   [scans]         item offsets per list
//   k_group_bounds  per-group [begin, end) of every list
//   k_emit_*        the items, in key order (= the order the host loops produced)
//   [radix sort on (group, -count), stable] + gather: group by group, larger items first, ties in order
//   k_point_keys    slot key of every (window, point); [stable radix sort]; k_point_gather -> u_sorted, perm
#include <cuda_runtime.h>
#include <cub/cub.cuh>

#include <cstdlib>

#include "akm_internal.cuh"

namespace akm {

__device__ __forceinline__ void slot_cell(const WinGeom& g, long long q, int c[3], int& cls) {
  cls = (int)(q & 1);
  long long ci = q >> 1;
  c[2] = (int)(ci % g.ncell[2]);
  ci /= g.ncell[2];
  c[1] = (int)(ci % g.ncell[1]);
  c[0] = (int)(ci / g.ncell[1]);
}

__device__ __forceinline__ int cand_nb(const WinGeom& g, int a, int B) {
  return (a >= 3 - g.d) ? (g.ncell[a] + B - 1) / B : 1;
}

__global__ void k_bin_cand(const WinTable* __restrict__ tabp, const int* __restrict__ hist,
                           const long long* __restrict__ hist_off, BinCandParam cp, int* __restrict__ bc) {
  const WinTable& tab = *tabp;
  const int w = blockIdx.y;
  const WinGeom& g = tab.w[w];
  const long long slots = 2LL * g.ncell[0] * g.ncell[1] * g.ncell[2];
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < slots; q += (long long)gridDim.x * blockDim.x) {
    const int v = hist[hist_off[w] + q];
    if (!v) continue;
    int c[3], cls;
    slot_cell(g, q, c, cls);
    for (int k = 0; k < kBinCands; ++k) {
      if (!(cp.mask[w] & (1 << k))) continue;
      const int B = cp.B[k];
      long long b = 0;
      for (int a = 0; a < 3; ++a) b = b * cand_nb(g, a, B) + ((a >= 3 - g.d) ? c[a] / B : 0);
      atomicAdd(bc + cp.off[w][k] + b, v);
    }
  }
}

// stats[(w * kBinCands + k) * 3 + {0, 1, 2}] = spreading chunks, occupied bins, largest bin
__global__ void k_bin_stats(const WinTable* __restrict__ tabp, BinCandParam cp, const int* __restrict__ bc,
                            long long ch_s, int* __restrict__ stats) {
  const WinTable& tab = *tabp;
  const int w = blockIdx.y / kBinCands, k = blockIdx.y % kBinCands;
  if (!(cp.mask[w] & (1 << k))) return;
  const WinGeom& g = tab.w[w];
  const int B = cp.B[k];
  const long long nb = (long long)cand_nb(g, 0, B) * cand_nb(g, 1, B) * cand_nb(g, 2, B);
  int chunks = 0, occ = 0, mx = 0;
  for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < nb; b += (long long)gridDim.x * blockDim.x) {
    const int v = bc[cp.off[w][k] + b];
    if (v) {
      chunks += (int)((v + ch_s - 1) / ch_s);
      occ += 1;
      mx = max(mx, v);
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    chunks += __shfl_xor_sync(0xffffffffu, chunks, o);
    occ += __shfl_xor_sync(0xffffffffu, occ, o);
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0 && (chunks || occ)) {
    int* st = stats + (w * kBinCands + k) * 3;
    atomicAdd(st + 0, chunks);
    atomicAdd(st + 1, occ);
    atomicMax(st + 2, mx);
  }
}

cudaError_t launch_bin_costs(const WinTable& tab, const WinTable* dtab, const int* hist, const long long* hist_off,
                             const BinCandParam& cp, long long bc_total, int* bc, long long ch_s, int* stats,
                             cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(bc, 0, sizeof(int) * (size_t)std::max<long long>(bc_total, 1), s);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(stats, 0, sizeof(int) * tab.P * kBinCands * 3, s);
  if (e != cudaSuccess) return e;
  long long maxslots = 1;
  for (int w = 0; w < tab.P; ++w)
    maxslots = std::max(maxslots, 2LL * tab.w[w].ncell[0] * tab.w[w].ncell[1] * tab.w[w].ncell[2]);
  const int blocks = (int)std::min<long long>((maxslots + 255) / 256, 148 * 4);
  k_bin_cand<<<dim3(blocks, tab.P), 256, 0, s>>>(dtab, hist, hist_off, cp, bc);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_bin_stats<<<dim3(std::max(1, blocks / 4), tab.P * kBinCands), 256, 0, s>>>(dtab, cp, bc, ch_s, stats);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ bin-major layout
__device__ __forceinline__ long long slot_key(const WinGeom& g, const BinLayout& L, int w, const int c[3], int cls,
                                              long long& bin) {
  const int B = g.B;
  long long b = 0, sub = 0, bb = 1;
  for (int a = 0; a < 3; ++a) {
    const bool real = a >= 3 - g.d;
    const int Ba = real ? B : 1;
    b = b * g.nbin[a] + (real ? c[a] / B : 0);
    sub = sub * Ba + (real ? c[a] % B : 0);
    bb *= Ba;
  }
  bin = b;
  return L.keybase[w] + (b * 2 + cls) * bb + sub;
}

__global__ void k_slot_keys(const WinTable* __restrict__ tabp, const int* __restrict__ hist,
                            const long long* __restrict__ hist_off, BinLayout L, long long* __restrict__ key_cnt,
                            int* __restrict__ i0cnt, int* __restrict__ i1cnt, int ch_i) {
  const WinTable& tab = *tabp;
  const int w = blockIdx.y;
  const WinGeom& g = tab.w[w];
  const long long slots = 2LL * g.ncell[0] * g.ncell[1] * g.ncell[2];
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < slots; q += (long long)gridDim.x * blockDim.x) {
    const int v = hist[hist_off[w] + q];
    int c[3], cls;
    slot_cell(g, q, c, cls);
    long long bin;
    const long long key = slot_key(g, L, w, c, cls, bin);
    key_cnt[key] = v;
    const int items = (v + ch_i - 1) / ch_i;
    i0cnt[key] = items;
    if (i1cnt) i1cnt[key] = cls ? items : 0;
  }
}

// cursor[slot] = window-relative sorted start of the slot (optional); the near-field table (start,
// count) per slot (optional)
__global__ void k_slot_cursor(const WinTable* __restrict__ tabp, const long long* __restrict__ hist_off, BinLayout L,
                              const long long* __restrict__ key_cnt, const long long* __restrict__ key_off,
                              int* __restrict__ cursor, int2* __restrict__ cell_tab) {
  const WinTable& tab = *tabp;
  const int w = blockIdx.y;
  const WinGeom& g = tab.w[w];
  const long long slots = 2LL * g.ncell[0] * g.ncell[1] * g.ncell[2];
  const long long wbase = key_off[L.keybase[w]];
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < slots; q += (long long)gridDim.x * blockDim.x) {
    int c[3], cls;
    slot_cell(g, q, c, cls);
    long long bin;
    const long long key = slot_key(g, L, w, c, cls, bin);
    const int off = (int)(key_off[key] - wbase);
    if (cursor) cursor[hist_off[w] + q] = off;
    if (cell_tab) {
      const int v = (int)key_cnt[key];
      cell_tab[hist_off[w] + q] = make_int2(v ? off : 0, v);
    }
  }
}

__device__ __forceinline__ void bin_range(const WinGeom& g, const BinLayout& L, int w, long long b, long long nbins,
                                          long long n, const long long* key_off, long long wbase, long long& start,
                                          long long& c1, long long& end) {
  long long bb = 1;
  for (int a = 3 - g.d; a < 3; ++a) bb *= g.B;
  const long long k0 = L.keybase[w] + b * 2 * bb;
  start = key_off[k0] - wbase;
  c1 = key_off[k0 + bb] - wbase;
  end = (b + 1 < nbins) ? key_off[k0 + 2 * bb] - wbase : n;
}

__device__ __forceinline__ long long nbins_of(const WinGeom& g) {
  return (long long)g.nbin[0] * g.nbin[1] * g.nbin[2];
}

// bin starts; per-bin counts of the spreading chunks (ch_s) and per-bin interpolation chunks (ch_ib),
// for item set 0 (all points) and, with a split, set 1 (class-0 sources, class-1 targets)
__global__ void k_bin_pass(const WinTable* __restrict__ tabp, BinLayout L, const long long* __restrict__ key_off,
                           long long n, long long ch_s, int ch_ib, int* __restrict__ bin_start, int* __restrict__ s0,
                           int* __restrict__ b0, int* __restrict__ s1, int* __restrict__ b1) {
  const WinTable& tab = *tabp;
  const int w = blockIdx.y;
  const WinGeom& g = tab.w[w];
  const long long nbins = nbins_of(g);
  const long long wbase = key_off[L.keybase[w]];
  for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < nbins; b += (long long)gridDim.x * blockDim.x) {
    long long start, c1, end;
    bin_range(g, L, w, b, nbins, n, key_off, wbase, start, c1, end);
    bin_start[g.bt_off + b] = (int)start;
    if (b == nbins - 1) bin_start[g.bt_off + nbins] = (int)n;
    const long long o = L.binbase[w] + b;
    s0[o] = (int)((end - start + ch_s - 1) / ch_s);
    b0[o] = (int)((end - start + ch_ib - 1) / ch_ib);
    if (s1) {
      s1[o] = (int)((c1 - start + ch_s - 1) / ch_s);
      b1[o] = (int)((end - c1 + ch_ib - 1) / ch_ib);
    }
  }
}

// bounds[(list * 2 + {0, 1}) * ngroups + grp]: begin / end of each group in each list (the segment
// arrays of the sort), from the exclusive scans (cnt/off) over the list's index space (keys or bins,
// group-ordered)
__global__ void k_group_bounds(ListScanParam lp, int ngroups, int* __restrict__ bounds) {
  const int list = threadIdx.x;
  if (list >= lp.nlists) return;
  const int* cnt = lp.cnt[list];
  const int* off = lp.off[list];
  const long long len = lp.len[list];
  const int total = len > 0 ? off[len - 1] + cnt[len - 1] : 0;
  for (int gi = 0; gi < ngroups; ++gi) {
    const long long a = lp.gbeg[list][gi], e = lp.gbeg[list][gi + 1];
    bounds[(list * 2 + 0) * ngroups + gi] = a < len ? off[a] : total;
    bounds[(list * 2 + 1) * ngroups + gi] = e < len ? off[e] : total;
  }
}

__global__ void k_emit_cell_items(const WinTable* __restrict__ tabp, BinLayout L, const long long* __restrict__ key_cnt,
                                  const long long* __restrict__ key_off, const int* __restrict__ i0off,
                                  const int* __restrict__ i1off, int ch_i, WorkItem* __restrict__ it0,
                                  WorkItem* __restrict__ it1) {
  const WinTable& tab = *tabp;
  const int w = blockIdx.y;
  const WinGeom& g = tab.w[w];
  const long long slots = 2LL * g.ncell[0] * g.ncell[1] * g.ncell[2];
  const long long wbase = key_off[L.keybase[w]];
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < slots; q += (long long)gridDim.x * blockDim.x) {
    int c[3], cls;
    slot_cell(g, q, c, cls);
    long long bin;
    const long long key = slot_key(g, L, w, c, cls, bin);
    const int v = (int)key_cnt[key];
    if (!v) continue;
    const int off = (int)(key_off[key] - wbase);
    const int j0 = i0off[key];
    for (int t = 0, qq = 0; qq < v; ++t, qq += ch_i) {
      const WorkItem wi{w, {c[0], c[1], c[2]}, off + qq, min(ch_i, v - qq)};
      it0[j0 + t] = wi;
      if (it1 && cls) it1[i1off[key] + t] = wi;
    }
  }
}

__device__ __forceinline__ void emit_chunks(WorkItem* out, int j, int w, const int bc[3], long long a, long long e,
                                            long long ch) {
  for (long long q = a; q < e; q += ch, ++j) out[j] = WorkItem{w, {bc[0], bc[1], bc[2]}, (int)q, (int)min(ch, e - q)};
}

__global__ void k_emit_bin_items(const WinTable* __restrict__ tabp, BinLayout L, const long long* __restrict__ key_off,
                                 long long n, long long ch_s, int ch_ib, const int* __restrict__ s0off,
                                 const int* __restrict__ b0off, const int* __restrict__ s1off,
                                 const int* __restrict__ b1off, WorkItem* __restrict__ s0, WorkItem* __restrict__ b0,
                                 WorkItem* __restrict__ s1, WorkItem* __restrict__ b1) {
  const WinTable& tab = *tabp;
  const int w = blockIdx.y;
  const WinGeom& g = tab.w[w];
  const long long nbins = nbins_of(g);
  const long long wbase = key_off[L.keybase[w]];
  for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < nbins; b += (long long)gridDim.x * blockDim.x) {
    long long start, c1, end;
    bin_range(g, L, w, b, nbins, n, key_off, wbase, start, c1, end);
    if (end == start) continue;
    int bcrd[3];
    long long r = b;
    bcrd[2] = (int)(r % g.nbin[2]);
    r /= g.nbin[2];
    bcrd[1] = (int)(r % g.nbin[1]);
    bcrd[0] = (int)(r / g.nbin[1]);
    const long long o = L.binbase[w] + b;
    emit_chunks(s0, s0off[o], w, bcrd, start, end, ch_s);
    emit_chunks(b0, b0off[o], w, bcrd, start, end, ch_ib);
    if (s1) {
      emit_chunks(s1, s1off[o], w, bcrd, start, c1, ch_s);
      emit_chunks(b1, b1off[o], w, bcrd, c1, end, ch_ib);
    }
  }
}

// sort key = (group of the item's window, maxc - count): one device-wide stable radix sort then orders
// the list group by group, larger items first inside a group, ties in list order
__global__ void k_item_keys(const WorkItem* __restrict__ it, long long cnt, int maxc, int cbits, WinGroupMap gm,
                            unsigned* __restrict__ keys, int* __restrict__ idx) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cnt; i += (long long)gridDim.x * blockDim.x) {
    keys[i] = ((unsigned)gm.group[it[i].win] << cbits) | (unsigned)(maxc - it[i].count);
    idx[i] = (int)i;
  }
}

__global__ void k_item_gather(const WorkItem* __restrict__ in, const int* __restrict__ idx, long long cnt,
                              WorkItem* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cnt; i += (long long)gridDim.x * blockDim.x)
    out[i] = in[idx[i]];
}

static int grid_for(long long work) { return (int)std::max<long long>(1, std::min<long long>((work + 255) / 256, 148 * 8)); }

// ------------------------------------------------------------------ point sort (replaces the atomic scatter)
// key of (window w, point i) = its slot's key: a stable radix sort by key puts every window's points
// in bin-major order, inside a slot by increasing point index (deterministic, unlike cursor atomics)
__global__ void k_point_keys(long long n, const WinTable* __restrict__ tabp, BinLayout L,
                             const double* __restrict__ u_tmp, long long n_split, unsigned* __restrict__ keys,
                             int* __restrict__ vals) {
  const WinTable& tab = *tabp;
  const int w = blockIdx.y;
  const WinGeom& g = tab.w[w];
  const int m = tab.m;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    int c[3] = {0, 0, 0};
    for (int a = 3 - g.d; a < 3; ++a) c[a] = (int)floor(u_tmp[((long long)w * 3 + a) * n + i]) - (g.box_lo[a] + m - 1);
    long long bin;
    const long long key = slot_key(g, L, w, c, i >= n_split ? 1 : 0, bin);
    keys[(long long)w * n + i] = (unsigned)key;
    vals[(long long)w * n + i] = (int)i;
  }
}

// sorted index j: window order[j / n] (every window holds n points; windows in group order), position
// j % n; gathers the scaled coordinates into u_sorted and the point index into perm
// (fixed_w >= 0: the sorted sequence of that window alone, j = position)
__global__ void k_point_gather(long long n, int P, const WinTable* __restrict__ tabp, WinGroupMap order,
                               const int* __restrict__ vals, const double* __restrict__ u_tmp,
                               double* __restrict__ u_sorted, int* __restrict__ perm, int fixed_w) {
  const WinTable& tab = *tabp;
  const long long total = fixed_w >= 0 ? n : n * P;
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < total; j += (long long)gridDim.x * blockDim.x) {
    const int w = fixed_w >= 0 ? fixed_w : order.group[j / n];
    const long long pos = j % n;
    const WinGeom& g = tab.w[w];
    const int i = vals[j];
    perm[(long long)w * n + pos] = i;
    for (int a = 3 - g.d; a < 3; ++a) u_sorted[((long long)w * 3 + a) * n + pos] = u_tmp[((long long)w * 3 + a) * n + i];
  }
}

cudaError_t launch_slot_keys(const WinTable& tab, const WinTable* dtab, const int* hist, const long long* hist_off,
                             const BinLayout& L, long long* key_cnt, int* i0cnt, int* i1cnt, int ch_i, cudaStream_t s) {
  long long maxslots = 1;
  for (int w = 0; w < tab.P; ++w)
    maxslots = std::max(maxslots, 2LL * tab.w[w].ncell[0] * tab.w[w].ncell[1] * tab.w[w].ncell[2]);
  k_slot_keys<<<dim3(grid_for(maxslots), tab.P), 256, 0, s>>>(dtab, hist, hist_off, L, key_cnt, i0cnt, i1cnt, ch_i);
  return cudaGetLastError();
}

cudaError_t launch_slot_cursor(const WinTable& tab, const WinTable* dtab, const long long* hist_off, const BinLayout& L,
                               const long long* key_cnt, const long long* key_off, int* cursor, int2* cell_tab,
                               cudaStream_t s) {
  long long maxslots = 1;
  for (int w = 0; w < tab.P; ++w)
    maxslots = std::max(maxslots, 2LL * tab.w[w].ncell[0] * tab.w[w].ncell[1] * tab.w[w].ncell[2]);
  k_slot_cursor<<<dim3(grid_for(maxslots), tab.P), 256, 0, s>>>(dtab, hist_off, L, key_cnt, key_off, cursor, cell_tab);
  return cudaGetLastError();
}

cudaError_t launch_bin_pass(const WinTable& tab, const WinTable* dtab, const BinLayout& L, const long long* key_off,
                            long long n, long long ch_s, int ch_ib, int* bin_start, int* s0, int* b0, int* s1, int* b1,
                            cudaStream_t s) {
  long long maxb = 1;
  for (int w = 0; w < tab.P; ++w) maxb = std::max(maxb, (long long)tab.w[w].nbin[0] * tab.w[w].nbin[1] * tab.w[w].nbin[2]);
  k_bin_pass<<<dim3(grid_for(maxb), tab.P), 256, 0, s>>>(dtab, L, key_off, n, ch_s, ch_ib, bin_start, s0, b0, s1, b1);
  return cudaGetLastError();
}

cudaError_t launch_group_bounds(const ListScanParam& lp, int ngroups, int* bounds, cudaStream_t s) {
  k_group_bounds<<<1, 32, 0, s>>>(lp, ngroups, bounds);
  return cudaGetLastError();
}

cudaError_t launch_emit_items(const WinTable& tab, const WinTable* dtab, const BinLayout& L, const long long* key_cnt,
                              const long long* key_off, long long n, long long ch_s, int ch_i, int ch_ib,
                              const int* const off[6], WorkItem* const out[6], cudaStream_t s) {
  long long maxslots = 1, maxb = 1;
  for (int w = 0; w < tab.P; ++w) {
    maxslots = std::max(maxslots, 2LL * tab.w[w].ncell[0] * tab.w[w].ncell[1] * tab.w[w].ncell[2]);
    maxb = std::max(maxb, (long long)tab.w[w].nbin[0] * tab.w[w].nbin[1] * tab.w[w].nbin[2]);
  }
  // lists: 0 interp-cell set 0, 1 interp-cell set 1, 2 spread set 0, 3 bin set 0, 4 spread set 1, 5 bin set 1
  k_emit_cell_items<<<dim3(grid_for(maxslots), tab.P), 256, 0, s>>>(dtab, L, key_cnt, key_off, off[0], off[1], ch_i,
                                                                    out[0], out[1]);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_emit_bin_items<<<dim3(grid_for(maxb), tab.P), 256, 0, s>>>(dtab, L, key_off, n, ch_s, ch_ib, off[2], off[3], off[4],
                                                               off[5], out[2], out[3], out[4], out[5]);
  return cudaGetLastError();
}

// Exclusive sums with a caller-owned temporary (grown on demand through *temp / *temp_bytes).
template <class T>
static cudaError_t scan_excl(const T* in, T* out, long long len, void** temp, size_t* temp_bytes, cudaStream_t s) {
  if (len <= 0) return cudaSuccess;
  size_t need = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, need, in, out, (int)len, s);
  if (e != cudaSuccess) return e;
  if (need > *temp_bytes) {
    if (*temp) cudaFree(*temp);
    *temp = nullptr;
    *temp_bytes = 0;
    e = cudaMalloc(temp, need);
    if (e != cudaSuccess) return e;
    *temp_bytes = need;
  }
  return cub::DeviceScan::ExclusiveSum(*temp, need, in, out, (int)len, s);
}

cudaError_t scan_excl_ll(const long long* in, long long* out, long long len, void** temp, size_t* temp_bytes,
                         cudaStream_t s) {
  return scan_excl(in, out, len, temp, temp_bytes, s);
}
cudaError_t scan_excl_int(const int* in, int* out, long long len, void** temp, size_t* temp_bytes, cudaStream_t s) {
  return scan_excl(in, out, len, temp, temp_bytes, s);
}

// Stable sort of one list by (group, decreasing count), then gather into `out`.
cudaError_t sort_items_larger_first(const WorkItem* in, long long cnt, int maxc, const WinGroupMap& gm, int ngroups,
                                    unsigned* keys, unsigned* keys_alt, int* idx, int* idx_alt, void** temp,
                                    size_t* temp_bytes, WorkItem* out, cudaStream_t s) {
  if (cnt <= 0) return cudaSuccess;
  int cbits = 1;
  while ((1 << cbits) <= maxc) ++cbits;
  int gbits = 0;
  while ((1 << gbits) < ngroups) ++gbits;
  k_item_keys<<<grid_for(cnt), 256, 0, s>>>(in, cnt, maxc, cbits, gm, keys, idx);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  size_t need = 0;
  e = cub::DeviceRadixSort::SortPairs(nullptr, need, keys, keys_alt, idx, idx_alt, (int)cnt, 0, cbits + gbits, s);
  if (e != cudaSuccess) return e;
  if (need > *temp_bytes) {
    if (*temp) cudaFree(*temp);
    *temp = nullptr;
    *temp_bytes = 0;
    e = cudaMalloc(temp, need);
    if (e != cudaSuccess) return e;
    *temp_bytes = need;
  }
  e = cub::DeviceRadixSort::SortPairs(*temp, need, keys, keys_alt, idx, idx_alt, (int)cnt, 0, cbits + gbits, s);
  if (e != cudaSuccess) return e;
  k_item_gather<<<grid_for(cnt), 256, 0, s>>>(in, idx_alt, cnt, out);
  return cudaGetLastError();
}

cudaError_t sort_points(long long n, const WinTable& tab, const WinTable* dtab, const BinLayout& L, long long nkeys,
                        const WinGroupMap& order, const double* u_tmp, long long n_split, unsigned* keys,
                        unsigned* keys_alt, int* vals, int* vals_alt, void** temp, size_t* temp_bytes,
                        double* u_sorted, int* perm, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const long long total = n * tab.P;
  k_point_keys<<<dim3(grid_for(n), tab.P), 256, 0, s>>>(n, dtab, L, u_tmp, n_split, keys, vals);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  int bits = 1;
  while ((1LL << bits) < nkeys) ++bits;
  // one sort over every (window, point) while the count fits CUB's int sizes, else one per window
  // (AKM_SORT_PER_WINDOW=1 forces the per-window path: tests exercise it at small sizes)
  static const bool per_window_env = getenv("AKM_SORT_PER_WINDOW") && atoi(getenv("AKM_SORT_PER_WINDOW")) == 1;
  const bool whole = total < (1LL << 31) - 1 && !per_window_env;
  const long long len = whole ? total : n;
  size_t need = 0;
  e = cub::DeviceRadixSort::SortPairs(nullptr, need, keys, keys_alt, vals, vals_alt, (int)len, 0, bits, s);
  if (e != cudaSuccess) return e;
  if (need > *temp_bytes) {
    if (*temp) cudaFree(*temp);
    *temp = nullptr;
    *temp_bytes = 0;
    e = cudaMalloc(temp, need);
    if (e != cudaSuccess) return e;
    *temp_bytes = need;
  }
  if (whole) {
    e = cub::DeviceRadixSort::SortPairs(*temp, need, keys, keys_alt, vals, vals_alt, (int)total, 0, bits, s);
    if (e != cudaSuccess) return e;
    k_point_gather<<<grid_for(total), 256, 0, s>>>(n, tab.P, dtab, order, vals_alt, u_tmp, u_sorted, perm, -1);
    return cudaGetLastError();
  }
  for (int w = 0; w < tab.P; ++w) {
    const long long o = (long long)w * n;
    e = cub::DeviceRadixSort::SortPairs(*temp, need, keys + o, keys_alt + o, vals + o, vals_alt + o, (int)n, 0, bits,
                                        s);
    if (e != cudaSuccess) return e;
    k_point_gather<<<grid_for(n), 256, 0, s>>>(n, tab.P, dtab, order, vals_alt + o, u_tmp, u_sorted, perm, w);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace akm
