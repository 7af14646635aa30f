// trb_ccl.cu — north-star kernels (3) and (4): connected-component
// labelling as tile-local union-find + a boundary-merge pass + canonical
// relabelling, and per-blob area/bbox/centroid reduction.
//
// Reference: label_blocked / label_sequential (segmentation.hpp:183-264),
// label_window + UnionFind (:154-178, :58-75), finalize_labels (:88-149).
//
// Canonical output (segmentation.hpp:193-197): labels are dense 1..k in
// raster order of each component's first pixel, components with
// area < min_area dropped and the survivors compacted.  So the final label
// of a component is 1 + the number of surviving components whose minimum
// linear pixel index is smaller — computed here from a per-row survivor
// count (exclusive scan over rows) plus a per-row survivor bitmap
// (popcount of the bits to the left).  `n_blocks` never changes the output.
//
// Kernels (grid.z or grid.y = stream):
//   ccl_occupancy one warp per 32x32 tile: tiles holding foreground are
//                appended to a compact list
//   ccl_local    per listed tile (persistent CTAs): run-based union-find in
//                shared memory (root = smallest local index = raster-first
//                pixel), per tile component stats (area, bbox, sum x,
//                sum y), one global slot per tile component; labg[p] = slot
//                for foreground pixels
//   ccl_merge    unions across the seams of listed tiles (slot union-find)
//   ccl_resolve  slot -> set root; stats of non-root slots atomically
//                folded into their root
//   ccl_mark     surviving roots: bitmap bit + per-row count
//   ccl_scan     exclusive scan of the row counts (one CTA per stream)
//   ccl_assign   rank of every slot's component; Blob record per survivor
//   ccl_final    labels[p] = dense[labg[p]] (16 pixels per thread)
#include "trb_kernels.cuh"

namespace trb {

namespace {

// find with path halving: every visited node is re-pointed at its
// grandparent (values only move towards the root, so racing writers are
// harmless and later finds walk shorter chains)
__device__ __forceinline__ int sfind(int* lab, int i) {
  int p = lab[i];
  while (p != i) {
    const int gp = lab[p];
    if (gp != p) lab[i] = gp;
    i = p;
    p = gp;
  }
  return i;
}

// Playne & Hawick style lock-free union in shared memory: the larger root
// is pointed at the smaller with atomicMin until one attempt lands on a
// root.
__device__ __forceinline__ void sunion(int* lab, int a, int b) {
  bool done;
  do {
    a = sfind(lab, a);
    b = sfind(lab, b);
    if (a < b) {
      const int old = atomicMin(&lab[b], a);
      done = (old == b);
      b = old;
    } else if (b < a) {
      const int old = atomicMin(&lab[a], b);
      done = (old == a);
      a = old;
    } else {
      done = true;
    }
  } while (!done);
}

__device__ __forceinline__ int gfind(int* parent, int s) {
  int p = *reinterpret_cast<volatile int*>(&parent[s]);
  while (p != s) {
    const int gp = *reinterpret_cast<volatile int*>(&parent[p]);
    if (gp != p) atomicMin(&parent[s], gp);  // path halving; monotone, ancestors only
    s = p;
    p = gp;
  }
  return s;
}

__device__ __forceinline__ void gunion(int* parent, int a, int b) {
  bool done;
  do {
    a = gfind(parent, a);
    b = gfind(parent, b);
    if (a < b) {
      const int old = atomicMin(&parent[b], a);
      done = (old == b);
      b = old;
    } else if (b < a) {
      const int old = atomicMin(&parent[a], b);
      done = (old == a);
      a = old;
    } else {
      done = true;
    }
  } while (!done);
}

__device__ __forceinline__ SlotTable slot_base(const CclArgs& a, int s) {
  SlotTable t = a.slots;
  const int64_t o = static_cast<int64_t>(s) * a.slot_cap;
  t.parent += o, t.root += o, t.area += o, t.x0 += o, t.y0 += o, t.x1 += o, t.y1 += o;
  t.sx += o, t.sy += o, t.minpix += o, t.dense += o;
  return t;
}

}  // namespace

// ------------------------------------------------------------------ local
// Run-based: warp w loads rows w, w+8, w+16, w+24 (lane = column) and a
// ballot turns each row into a 32-bit mask; horizontal runs are bit runs.
// Only run-start pixels enter the union-find (a run's pixels share its
// start), and only vertical run adjacencies are unioned; statistics are
// accumulated per run (area = length, sum x = arithmetic series).
__device__ __forceinline__ int run_len(uint32_t m, int c) {  // ones from bit c up
  const uint32_t z = ~(m >> c);
  return z ? __ffs(z) - 1 : 32 - c;
}
__device__ __forceinline__ int run_start_at(uint32_t starts, int p) {  // start of the run covering bit p
  const uint32_t x = starts & (p == 31 ? 0xffffffffu : ((2u << p) - 1));
  return 31 - __clz(x);
}

// Tile-list entries carry (stream, tile x, tile y) packed, so the list
// walkers need no integer division: s < 2^11, tx, ty < 2^10 (checked on
// the host, CclState).
__device__ __forceinline__ int tile_pack(int s, int tx, int ty) { return (s << 20) | (ty << 10) | tx; }
__device__ __forceinline__ void tile_unpack(int v, int& s, int& tx, int& ty) {
  s = v >> 20, ty = (v >> 10) & 1023, tx = v & 1023;
}

// Tiles holding foreground: one warp per 32x32 tile (lane = row, 32 bytes
// per lane), appended to a compact list that the local and seam kernels
// walk — most of a frame is background (C5: ~8 % foreground).
__global__ void __launch_bounds__(256) ccl_occupancy_kernel(CclArgs a, int vec_ok) {
  const int n_tiles = a.tiles_x * a.tiles_y;
  const int s = blockIdx.y;
  {
    // per-frame resets of this stream's slot counter, row counts and
    // survivor bitmap (first used by ccl_local / ccl_mark, which wait for
    // this grid); the tile-list counter was reset by the previous frame's
    // ccl_final (this kernel appends to it)
    const int64_t gt = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t gn = static_cast<int64_t>(gridDim.x) * blockDim.x;
    if (gt == 0) a.nslots[s] = 0;
    int32_t* rc = a.rowcount + static_cast<int64_t>(s) * a.h;
    for (int64_t i = gt; i < a.h; i += gn) rc[i] = 0;
    uint32_t* bm = a.bitmap + static_cast<int64_t>(s) * a.h * a.wpr;
    for (int64_t i = gt; i < static_cast<int64_t>(a.h) * a.wpr; i += gn) bm[i] = 0u;
  }
  const int t = static_cast<int>((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= n_tiles) return;
  const int tile = s * n_tiles + t;
  const int tx = t % a.tiles_x, ty = t / a.tiles_x;
  const int gy = ty * kTileH + lane, gx0 = tx * kTileW;
  bool any = false;
  if (gy < a.h) {
    const uint8_t* row = a.mask + static_cast<int64_t>(s) * a.px + static_cast<int64_t>(gy) * a.w + gx0;
    if (vec_ok && gx0 + kTileW <= a.w) {
      const uint4 q0 = reinterpret_cast<const uint4*>(row)[0], q1 = reinterpret_cast<const uint4*>(row)[1];
      any = (q0.x | q0.y | q0.z | q0.w | q1.x | q1.y | q1.z | q1.w) != 0;
    } else {
      for (int c = 0; c < kTileW && gx0 + c < a.w; ++c) any |= row[c] != 0;
    }
  }
  const bool fg = __any_sync(0xffffffffu, any);
  if (lane == 0) {
    if (fg) a.tile_list[atomicAdd(a.tile_count, 1)] = tile_pack(s, tx, ty);
    a.tile_state[tile] = static_cast<uint8_t>((a.tile_state[tile] & 2u) | (fg ? 1u : 0u));
  }
}

__global__ void __launch_bounds__(256) ccl_local_kernel(CclArgs a) {
  pdl_wait();  // launched with launch_pdl: the previous kernel's results first
  __shared__ int lab[kTilePx];
  __shared__ int cid[kTilePx];  // compact component id of each local root
  __shared__ uint32_t rowm[kTileH], starts[kTileH];
  __shared__ int st_area[kMaxTileComps], st_x0[kMaxTileComps], st_y0[kMaxTileComps], st_x1[kMaxTileComps],
      st_y1[kMaxTileComps], st_sx[kMaxTileComps], st_sy[kMaxTileComps];
  __shared__ int n_comp, slot_base_id;

  const int n_list = *a.tile_count;
  const int w = threadIdx.x >> 5, c = threadIdx.x & 31;
  // this thread's 4 mask bytes of a listed tile (rows w, w+8, w+16, w+24)
  auto load_rows = [&](int it, uint32_t& bits) {
    bits = 0;
    if (it >= n_list) return;
    int s_, tx_, ty_;
    tile_unpack(a.tile_list[it], s_, tx_, ty_);
    const uint8_t* m_ = a.mask + static_cast<int64_t>(s_) * a.px;
    const int gx_ = tx_ * kTileW + c;
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      const int gy_ = ty_ * kTileH + w + 8 * rr;
      if (gy_ < a.h && gx_ < a.w && m_[static_cast<int64_t>(gy_) * a.w + gx_] != 0) bits |= 1u << rr;
    }
  };
  uint32_t next_bits;
  load_rows(blockIdx.x, next_bits);
  for (int it = blockIdx.x; it < n_list; it += gridDim.x) {
  int s, tx, ty;
  tile_unpack(a.tile_list[it], s, tx, ty);
  int32_t* labg = a.labg + static_cast<int64_t>(s) * a.px;
  const int tx0 = tx * kTileW, ty0 = ty * kTileH;
  const int gx = tx0 + c;
  // the next listed tile's mask bytes are requested before this one is
  // labelled (their latency overlaps the work below)
  const uint32_t cur_bits = next_bits;
  load_rows(it + gridDim.x, next_bits);
  __syncthreads();  // the previous tile is done with the shared arrays
  if (threadIdx.x == 0) n_comp = 0;

  // 1. rows as bit masks
  bool any = false;
  uint32_t mine = 0;  // bit rr: pixel (row w + 8*rr, column c) is foreground
#pragma unroll
  for (int rr = 0; rr < 4; ++rr) {
    const int r = w + 8 * rr;
    const bool fg = (cur_bits >> rr) & 1u;
    const uint32_t m = __ballot_sync(0xffffffffu, fg);
    if (c == 0) rowm[r] = m, starts[r] = m & ~(m << 1);
    mine |= static_cast<uint32_t>(fg) << rr;
    any |= fg;
  }
  if (!__syncthreads_or(any)) continue;  // (listed tiles hold foreground)

  // 2. run starts are the union-find nodes
#pragma unroll
  for (int rr = 0; rr < 4; ++rr) {
    const int r = w + 8 * rr;
    if ((starts[r] >> c) & 1u) lab[r * kTileW + c] = r * kTileW + c;
  }
  __syncthreads();
  // 3. union every run with the runs of the row above that touch it
  //    (label_window's up / up-left / up-right neighbours, segmentation.hpp:169-174)
#pragma unroll
  for (int rr = 0; rr < 4; ++rr) {
    const int r = w + 8 * rr;
    if (r == 0 || !((starts[r] >> c) & 1u)) continue;
    const uint32_t up = rowm[r - 1];
    if (!up) continue;
    const int b = c + run_len(rowm[r], c) - 1;
    const int lo = a.conn == TRB_CONN_EIGHT ? max(c - 1, 0) : c;
    const int hi = a.conn == TRB_CONN_EIGHT ? min(b + 1, 31) : b;
    uint32_t ov = up & ((hi == 31 ? 0xffffffffu : ((2u << hi) - 1)) & ~((1u << lo) - 1));
    const uint32_t sup = starts[r - 1];
    while (ov) {
      const int p = __ffs(ov) - 1;
      const int sa = run_start_at(sup, p);
      sunion(lab, r * kTileW + c, (r - 1) * kTileW + sa);
      const int ea = sa + run_len(up, sa) - 1;  // skip the rest of that run
      ov &= ea >= 31 ? 0u : ~((2u << ea) - 1);
    }
  }
  __syncthreads();

  // 4. flatten; number the local roots (root = smallest local index, the
  //    component's raster-first pixel)
  int root[4];
#pragma unroll
  for (int rr = 0; rr < 4; ++rr) {
    const int r = w + 8 * rr;
    root[rr] = ((starts[r] >> c) & 1u) ? sfind(lab, r * kTileW + c) : -1;
  }
  __syncthreads();
#pragma unroll
  for (int rr = 0; rr < 4; ++rr) {
    const int r = w + 8 * rr, i = r * kTileW + c;
    if (root[rr] < 0) continue;
    lab[i] = root[rr];
    if (root[rr] == i) {
      const int id = atomicAdd(&n_comp, 1);
      cid[i] = id;
      st_area[id] = 0;
      st_x0[id] = INT_MAX, st_y0[id] = INT_MAX, st_x1[id] = -1, st_y1[id] = -1;
      st_sx[id] = 0, st_sy[id] = 0;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && n_comp > 0) slot_base_id = atomicAdd(&a.nslots[s], n_comp);

  // 5. tile-component statistics per run (integer, order-free)
#pragma unroll
  for (int rr = 0; rr < 4; ++rr) {
    if (root[rr] < 0) continue;
    const int r = w + 8 * rr, gy = ty0 + r;
    const int len = run_len(rowm[r], c);
    const int id = cid[root[rr]];
    atomicAdd(&st_area[id], len);
    atomicMin(&st_x0[id], gx);
    atomicMin(&st_y0[id], gy);
    atomicMax(&st_x1[id], gx + len - 1);
    atomicMax(&st_y1[id], gy);
    atomicAdd(&st_sx[id], len * gx + len * (len - 1) / 2);
    atomicAdd(&st_sy[id], len * gy);
  }
  __syncthreads();
  const int base = slot_base_id;

  // 6. slot id per foreground pixel (its run start's root); slot records
#pragma unroll
  for (int rr = 0; rr < 4; ++rr) {
    if (!((mine >> rr) & 1u)) continue;
    const int r = w + 8 * rr, gy = ty0 + r;
    const int sc = run_start_at(starts[r], c);
    labg[static_cast<int64_t>(gy) * a.w + gx] = base + cid[lab[r * kTileW + sc]];
  }
  SlotTable t = slot_base(a, s);
#pragma unroll
  for (int rr = 0; rr < 4; ++rr) {
    const int r = w + 8 * rr, i = r * kTileW + c;
    if (root[rr] != i) continue;
    const int id = cid[i];
    const int slot = base + id;
    t.parent[slot] = slot;
    t.area[slot] = st_area[id];
    t.x0[slot] = st_x0[id];
    t.y0[slot] = st_y0[id];
    t.x1[slot] = st_x1[id];
    t.y1[slot] = st_y1[id];
    t.sx[slot] = static_cast<unsigned long long>(st_sx[id]);
    t.sy[slot] = static_cast<unsigned long long>(st_sy[id]);
    t.minpix[slot] = (ty0 + r) * a.w + gx;
  }
  }  // tile loop
}

// ------------------------------------------------------------------ merge
// One thread per tile-seam pixel: 32 top-seam + 32 left-seam per tile.
__device__ __forceinline__ void ccl_merge_one(const CclArgs& a, int s, int tx, int ty, int j) {
  const uint8_t* mask = a.mask + static_cast<int64_t>(s) * a.px;
  const int32_t* labg = a.labg + static_cast<int64_t>(s) * a.px;
  int* parent = a.slots.parent + static_cast<int64_t>(s) * a.slot_cap;
  const int w = a.w, h = a.h;
  auto fgat = [&](int x, int y) { return mask[static_cast<int64_t>(y) * w + x] != 0; };
  auto sl = [&](int x, int y) { return labg[static_cast<int64_t>(y) * w + x]; };
  if (j < 32) {  // top seam: (x, y) against row y-1
    if (ty == 0) return;
    const int x = tx * kTileW + j, y = ty * kTileH;
    if (x >= w || y >= h || !fgat(x, y)) return;
    const int me = sl(x, y);
    if (fgat(x, y - 1)) {
      gunion(parent, me, sl(x, y - 1));
    } else if (a.conn == TRB_CONN_EIGHT) {
      if (x > 0 && fgat(x - 1, y - 1)) gunion(parent, me, sl(x - 1, y - 1));
      if (x + 1 < w && fgat(x + 1, y - 1)) gunion(parent, me, sl(x + 1, y - 1));
    }
  } else {  // left seam: (x, y) against column x-1
    if (tx == 0) return;
    const int x = tx * kTileW, y = ty * kTileH + (j - 32);
    if (x >= w || y >= h || !fgat(x, y)) return;
    const int me = sl(x, y);
    if (fgat(x - 1, y)) gunion(parent, me, sl(x - 1, y));
    if (a.conn == TRB_CONN_EIGHT) {
      if (y > 0 && fgat(x - 1, y - 1)) gunion(parent, me, sl(x - 1, y - 1));
      if (y + 1 < h && fgat(x - 1, y + 1)) gunion(parent, me, sl(x - 1, y + 1));
    }
  }
}

// Only listed (foreground) tiles can own a seam union: the pixel below /
// right of the seam must be foreground.  Grid-stride over list x 64.
__global__ void __launch_bounds__(256) ccl_merge_kernel(CclArgs a) {
  pdl_wait();  // launched with launch_pdl: the previous kernel's results first
  const int64_t total = static_cast<int64_t>(*a.tile_count) * 64;
  for (int64_t gid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; gid < total;
       gid += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int s, tx, ty;
    tile_unpack(a.tile_list[gid >> 6], s, tx, ty);
    ccl_merge_one(a, s, tx, ty, static_cast<int>(gid & 63));
  }
}

// ---------------------------------------------------------------- resolve
__global__ void __launch_bounds__(256) ccl_resolve_kernel(CclArgs a) {
  pdl_wait();  // launched with launch_pdl: the previous kernel's results first
  const int s = blockIdx.y;
  const int n = a.nslots[s];
  SlotTable t = slot_base(a, s);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int r = gfind(t.parent, i);
    t.root[i] = r;
    if (r == i) continue;
    atomicAdd(&t.area[r], t.area[i]);
    atomicMin(&t.x0[r], t.x0[i]);
    atomicMin(&t.y0[r], t.y0[i]);
    atomicMax(&t.x1[r], t.x1[i]);
    atomicMax(&t.y1[r], t.y1[i]);
    atomicAdd(&t.sx[r], t.sx[i]);
    atomicAdd(&t.sy[r], t.sy[i]);
    atomicMin(&t.minpix[r], t.minpix[i]);
  }
}

// ------------------------------------------------------------------- mark
__global__ void __launch_bounds__(256) ccl_mark_kernel(CclArgs a) {
  pdl_wait();  // launched with launch_pdl: the previous kernel's results first
  const int s = blockIdx.y;
  const int n = a.nslots[s];
  SlotTable t = slot_base(a, s);
  int32_t* rowcount = a.rowcount + static_cast<int64_t>(s) * a.h;
  uint32_t* bitmap = a.bitmap + static_cast<int64_t>(s) * a.h * a.wpr;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (t.root[i] != i || t.area[i] < a.min_area) continue;
    const int pos = t.minpix[i];
    const int y = pos / a.w, x = pos - y * a.w;
    atomicOr(&bitmap[static_cast<int64_t>(y) * a.wpr + (x >> 5)], 1u << (x & 31));
    atomicAdd(&rowcount[y], 1);
  }
}

// ------------------------------------------------------------------- scan
// Exclusive scan of the per-row survivor counts; one 1024-thread CTA per
// stream, rows processed in chunks of 1024.
__global__ void __launch_bounds__(1024) ccl_scan_kernel(CclArgs a) {
  pdl_wait();  // launched with launch_pdl: the previous kernel's results first
  __shared__ int warp_sums[32];
  __shared__ int carry;
  const int s = blockIdx.x;
  int32_t* rc = a.rowcount + static_cast<int64_t>(s) * a.h;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < a.h; base += 1024) {
    const int i = base + threadIdx.x;
    const int v = i < a.h ? rc[i] : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int ws = warp_sums[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, ws, o);
        if (lane >= o) ws += y;
      }
      warp_sums[lane] = ws;
    }
    __syncthreads();
    const int incl = x + (wid > 0 ? warp_sums[wid - 1] : 0) + carry;
    if (i < a.h) rc[i] = incl - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry = incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) a.nblobs[s] = carry;
}

// ----------------------------------------------------------------- assign
__global__ void __launch_bounds__(256) ccl_assign_kernel(CclArgs a) {
  pdl_wait();  // launched with launch_pdl: the previous kernel's results first
  const int s = blockIdx.y;
  const int n = a.nslots[s];
  SlotTable t = slot_base(a, s);
  const int32_t* rowpre = a.rowcount + static_cast<int64_t>(s) * a.h;
  const uint32_t* bitmap = a.bitmap + static_cast<int64_t>(s) * a.h * a.wpr;
  trb_blob* blobs = a.blobs + static_cast<int64_t>(s) * a.blob_cap;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int r = t.root[i];
    const int area = t.area[r];
    if (area < a.min_area) {
      t.dense[i] = 0;
      continue;
    }
    const int pos = t.minpix[r];
    const int y = pos / a.w, x = pos - y * a.w;
    const uint32_t* row = bitmap + static_cast<int64_t>(y) * a.wpr;
    int rank = rowpre[y];
    for (int k = 0; k < (x >> 5); ++k) rank += __popc(row[k]);
    rank += __popc(row[x >> 5] & ((1u << (x & 31)) - 1u));
    const int label = rank + 1;
    t.dense[i] = label;
    if (r != i) continue;
    trb_blob b;
    b.label = label;
    b.area = area;
    b.x_min = t.x0[r];
    b.y_min = t.y0[r];
    b.x_max = t.x1[r];
    b.y_max = t.y1[r];
    // exact: integer sums < 2^53 converted to double, one IEEE division
    // (segmentation.hpp:139-147 accumulates the same integers in a double)
    b.cx = static_cast<double>(t.sx[r]) / static_cast<double>(area);
    b.cy = static_cast<double>(t.sy[r]) / static_cast<double>(area);
    blobs[rank] = b;
  }
}

// ------------------------------------------------------------------ final
// Final labels, tile by tile (one warp per 32x32 tile, lane = column, so
// every row is one coalesced 128-byte store): tiles holding foreground get
// their labels; tiles whose labels were written on an earlier frame but hold
// none now are cleared; untouched background tiles (most of a frame) are
// skipped — the plane stays zero there from the allocation on.
__global__ void __launch_bounds__(256) ccl_final_kernel(CclArgs a) {
  pdl_wait();  // launched with launch_pdl: the previous kernel's results first
  // the next frame's tile list starts empty (ccl_local / ccl_merge, its
  // readers, completed before this grid got past its PDL wait)
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *a.tile_count = 0;
  const int n_tiles = a.tiles_x * a.tiles_y;
  const int t = static_cast<int>((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= n_tiles) return;
  const int s = blockIdx.y;
  const int tile = s * n_tiles + t;
  const unsigned st = a.tile_state[tile];
  if (!(st & 3u)) return;
  const bool fg = st & 1u;
  const int tx = t % a.tiles_x, ty = t / a.tiles_x;
  const int gx = tx * kTileW + lane, gy0 = ty * kTileH;
  const uint8_t* mask = a.mask + static_cast<int64_t>(s) * a.px;
  const int32_t* labg = a.labg + static_cast<int64_t>(s) * a.px;
  int32_t* labels = a.labels + static_cast<int64_t>(s) * a.px;
  const int32_t* dense = a.slots.dense + static_cast<int64_t>(s) * a.slot_cap;
  const int y1 = min(a.h, gy0 + kTileH);
  if (gx < a.w) {
    for (int gy = gy0; gy < y1; ++gy) {
      const int64_t p = static_cast<int64_t>(gy) * a.w + gx;
      labels[p] = (fg && mask[p]) ? dense[labg[p]] : 0;
    }
  }
  if (lane == 0) a.tile_state[tile] = fg ? 3u : 0u;
}

int launch_ccl(const CclArgs& a, int S, cudaStream_t st) {
  const int64_t n_tiles = static_cast<int64_t>(a.tiles_x) * a.tiles_y;
  // per-frame resets happen inside the kernels (ccl_occupancy: slot
  // counters, row counts, survivor bitmap; ccl_final: the tile-list counter
  // for the next frame) — no memset launches on the chain
  const int vec_occ = (a.w % 16 == 0);
  ccl_occupancy_kernel<<<dim3(static_cast<unsigned>(ceil_div64(n_tiles * 32, 256)), S), 256, 0, st>>>(a, vec_occ);
  TRB_LAUNCH_CHECK("ccl_occupancy_kernel");
  // persistent CTAs over the foreground-tile list (count known on the device)
  const unsigned list_ctas = static_cast<unsigned>(std::min<int64_t>(n_tiles * S, 148 * 8));
  // the chain below overlaps each launch with its predecessor's drain (PDL)
  launch_pdl(ccl_local_kernel, dim3(list_ctas), dim3(256), 0, st, a);
  launch_pdl(ccl_merge_kernel, dim3(list_ctas), dim3(256), 0, st, a);
  // slot kernels: enough CTAs to cover a typical frame, grid-stride beyond
  const unsigned slot_blocks = static_cast<unsigned>(std::min<int64_t>(ceil_div64(a.slot_cap, 256), 64));
  launch_pdl(ccl_resolve_kernel, dim3(slot_blocks, S), dim3(256), 0, st, a);
  launch_pdl(ccl_mark_kernel, dim3(slot_blocks, S), dim3(256), 0, st, a);
  launch_pdl(ccl_scan_kernel, dim3(S), dim3(1024), 0, st, a);
  launch_pdl(ccl_assign_kernel, dim3(slot_blocks, S), dim3(256), 0, st, a);
  launch_pdl(ccl_final_kernel, dim3(static_cast<unsigned>(ceil_div64(n_tiles * 32, 256)), S), dim3(256), 0, st, a);
  return 8;
}


namespace {
__global__ void __launch_bounds__(128) pack_blobs_kernel(const trb_blob* blobs, int64_t stride, const int32_t* nblobs,
                                                         trb_blob* out, int bcap) {
  const int s = blockIdx.x, n = min(nblobs[s], bcap);
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[static_cast<int64_t>(s) * bcap + i] = blobs[s * stride + i];
}
}  // namespace

void launch_pack_blobs(const trb_blob* blobs, int64_t stride, const int32_t* nblobs, trb_blob* out, int bcap,
                       int n_streams, cudaStream_t st) {
  pack_blobs_kernel<<<n_streams, 128, 0, st>>>(blobs, stride, nblobs, out, bcap);
  TRB_LAUNCH_CHECK("pack_blobs_kernel");
}

}  // namespace trb
