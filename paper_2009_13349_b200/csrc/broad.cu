// GPU broad phase: the candidate pairs of the
// reference's broad_phase (pkg/src/ccdkit/scene.py:225-300) -- primitive
// pairs whose inflated swept boxes overlap, minus pairs sharing a mesh
// vertex, vertex-face pairs sorted by (vertex, triangle) then edge-edge
// pairs sorted by (edge_a, edge_b) with edge_a < edge_b -- written straight
// into the solver's [m][8][3] query layout on the device.
//
// Swept boxes are computed exactly as the reference (min / max over both
// snapshots, then -/+ inflation: one rounding each, scene.py:195-200).  The
// reference hashes boxes on a grid and then applies the exact closed-box
// test, so its pair set is exactly the overlap set; here:
//   1. boxes of vertices, triangles and edges; global bounds and the mean
//      box extent (-> grid cell size h) by a two-stage reduction;
//   2. every triangle / edge box enters the cells it covers as (cell, id)
//      entries, sorted by cell with a stable LSD radix sort, so each cell's
//      ids are ascending;
//   3. every vertex (edge) visits the cells its box covers, binary-searches
//      each cell's entry range and tests the candidates exactly; a pair is
//      counted only in its canonical cell (per axis the larger of the two
//      lower-corner cells: it contains max(lo_a, lo_b), a point of both
//      boxes), so each overlapping pair is found exactly once;
//   4. count -> scan -> emit (a, b) keys -> radix sort -> gather points.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>

#include "tccd.h"

namespace tccd_bp {

using u64 = unsigned long long;
using u32 = unsigned int;

constexpr int kT = 256;                 // threads per block
constexpr int kItems = 4;               // items per thread in scans / radix passes
constexpr int kTile = kT * kItems;      // items per block
constexpr int kMaxDimBits = 20;         // cells per axis <= 2^20

// ---------------------------------------------------------------- scans
__device__ __forceinline__ u64 block_excl_scan(u64 v, u64* sh, u64& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  u64 x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u64 y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[w] = x;
  __syncthreads();
  if (w == 0) {
    u64 s = lane < kT / 32 ? sh[lane] : 0ull;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u64 y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < kT / 32) sh[lane] = s;
  }
  __syncthreads();
  const u64 before = w ? sh[w - 1] : 0ull;
  total = sh[kT / 32 - 1];
  __syncthreads();
  return before + x - v;
}

// per-block sums of in[0, n)
__global__ void k_scan_partial(const u64* in, long long n, u64* bsum) {
  __shared__ u64 sh[kT / 32];
  const long long base = (long long)blockIdx.x * kTile + (long long)threadIdx.x * kItems;
  u64 s = 0;
#pragma unroll
  for (int j = 0; j < kItems; ++j)
    if (base + j < n) s += in[base + j];
  u64 tot;
  block_excl_scan(s, sh, tot);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

// exclusive scan of the nb block sums in place (one block); *total = sum
__global__ void k_scan_top(u64* bsum, long long nb, u64* total) {
  __shared__ u64 sh[kT / 32];
  u64 carry = 0;
  for (long long c = 0; c < nb; c += kT) {
    const long long i = c + threadIdx.x;
    const u64 v = i < nb ? bsum[i] : 0ull;
    u64 tot;
    const u64 ex = block_excl_scan(v, sh, tot);
    if (i < nb) bsum[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) *total = carry;
}

// out = exclusive prefix of in (may alias), using the scanned block sums
__global__ void k_scan_final(const u64* in, u64* out, long long n, const u64* bsum) {
  __shared__ u64 sh[kT / 32];
  const long long base = (long long)blockIdx.x * kTile + (long long)threadIdx.x * kItems;
  u64 v[kItems], s = 0;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    v[j] = base + j < n ? in[base + j] : 0ull;
    s += v[j];
  }
  u64 tot;
  u64 run = bsum[blockIdx.x] + block_excl_scan(s, sh, tot);
#pragma unroll
  for (int j = 0; j < kItems; ++j)
    if (base + j < n) {
      out[base + j] = run;
      run += v[j];
    }
}

// ---------------------------------------------------------- radix sort
// one stable LSD pass on one key bit: zeros first, then ones
__global__ void k_bit_count(const u64* keys, long long n, int bit, u64* bsum) {
  __shared__ u64 sh[kT / 32];
  const long long base = (long long)blockIdx.x * kTile + (long long)threadIdx.x * kItems;
  u64 z = 0;
#pragma unroll
  for (int j = 0; j < kItems; ++j)
    if (base + j < n) z += ((keys[base + j] >> bit) & 1ull) ? 0ull : 1ull;
  u64 tot;
  block_excl_scan(z, sh, tot);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

__global__ void k_bit_scatter(const u64* kin, const u32* vin, u64* kout, u32* vout, long long n,
                              int bit, const u64* zoff, const u64* zeros_total) {
  __shared__ u64 sh[kT / 32];
  const long long base = (long long)blockIdx.x * kTile + (long long)threadIdx.x * kItems;
  u64 k[kItems];
  u64 z = 0;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    k[j] = base + j < n ? kin[base + j] : 0ull;
    if (base + j < n && !((k[j] >> bit) & 1ull)) ++z;
  }
  u64 tot;
  u64 zb = zoff[blockIdx.x] + block_excl_scan(z, sh, tot);  // zeros before this thread's items
  const u64 Z = *zeros_total;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const long long i = base + j;
    if (i >= n) break;
    const bool one = (k[j] >> bit) & 1ull;
    const u64 pos = one ? Z + ((u64)i - zb) : zb;
    if (!one) ++zb;
    kout[pos] = k[j];
    if (vin) vout[pos] = vin[i];
  }
}

// ------------------------------------------------------------ geometry
// swept box of primitive i (k vertices, idx == nullptr: vertex i itself),
// scene.py:195-200: min / max over both snapshots, then -/+ inflation
__global__ void k_boxes(const double* x0, const double* x1, const int64_t* idx, int k, long long m,
                        double infl, double* lo, double* hi) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
#pragma unroll 1
  for (int ax = 0; ax < 3; ++ax) {
    double mn = INFINITY, mx = -INFINITY;
    for (int j = 0; j < k; ++j) {
      const long long v = idx ? idx[i * k + j] : i;
      const double a = x0[v * 3 + ax], b = x1[v * 3 + ax];
      mn = fmin(mn, fmin(a, b));
      mx = fmax(mx, fmax(a, b));
    }
    lo[i * 3 + ax] = mn - infl;
    hi[i * 3 + ax] = mx + infl;
  }
}

// partial reductions over boxes [0, N): min lo, max hi (all boxes) and the
// sum of the largest extent over boxes [sum_from, N)
struct Red {
  double mn[3], mx[3], ext;
};

__global__ void k_reduce_partial(const double* lo, const double* hi, long long N, long long sum_from,
                                 Red* part) {
  __shared__ Red sh[kT];
  Red r;
  for (int a = 0; a < 3; ++a) { r.mn[a] = INFINITY; r.mx[a] = -INFINITY; }
  r.ext = 0.0;
  for (long long i = (long long)blockIdx.x * kT + threadIdx.x; i < N; i += (long long)gridDim.x * kT) {
    double e = 0.0;
    for (int a = 0; a < 3; ++a) {
      r.mn[a] = fmin(r.mn[a], lo[i * 3 + a]);
      r.mx[a] = fmax(r.mx[a], hi[i * 3 + a]);
      e = fmax(e, hi[i * 3 + a] - lo[i * 3 + a]);
    }
    if (i >= sum_from) r.ext += e;
  }
  sh[threadIdx.x] = r;
  __syncthreads();
  for (int s = kT / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      Red& x = sh[threadIdx.x];
      const Red& y = sh[threadIdx.x + s];
      for (int a = 0; a < 3; ++a) { x.mn[a] = fmin(x.mn[a], y.mn[a]); x.mx[a] = fmax(x.mx[a], y.mx[a]); }
      x.ext += y.ext;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void k_reduce_final(Red* part, int nb) {
  if (threadIdx.x != 0) return;
  Red r = part[0];
  for (int b = 1; b < nb; ++b) {
    for (int a = 0; a < 3; ++a) { r.mn[a] = fmin(r.mn[a], part[b].mn[a]); r.mx[a] = fmax(r.mx[a], part[b].mx[a]); }
    r.ext += part[b].ext;
  }
  part[0] = r;
}

struct Grid {
  double g0[3];  // grid origin (global min corner)
  double h;      // cell size
  double inv_h;  // 1 / h: cells by multiplication (monotone; no division sequence)
  int bits[3];   // key bits per axis
  long long dim[3];
};

__device__ __forceinline__ long long cell_of(double x, double g0, double inv_h, long long dim) {
  long long c = (long long)floor((x - g0) * inv_h);  // monotone in x
  return c < 0 ? 0 : (c >= dim ? dim - 1 : c);
}

__device__ __forceinline__ u64 cell_key(const Grid& g, long long cx, long long cy, long long cz) {
  return ((u64)cx << (g.bits[1] + g.bits[2])) | ((u64)cy << g.bits[2]) | (u64)cz;
}

__device__ __forceinline__ void cell_range(const Grid& g, const double* lo, const double* hi,
                                           long long c0[3], long long c1[3]) {
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    c0[a] = cell_of(lo[a], g.g0[a], g.inv_h, g.dim[a]);
    c1[a] = cell_of(hi[a], g.g0[a], g.inv_h, g.dim[a]);
  }
}

// cells covered by each box of [first, first + m)
__global__ void k_entry_counts(Grid g, const double* lo, const double* hi, long long first, long long m,
                               u64* cnt) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  long long c0[3], c1[3];
  cell_range(g, lo + (first + i) * 3, hi + (first + i) * 3, c0, c1);
  cnt[i] = (u64)(c1[0] - c0[0] + 1) * (u64)(c1[1] - c0[1] + 1) * (u64)(c1[2] - c0[2] + 1);
}

__global__ void k_entry_fill(Grid g, const double* lo, const double* hi, long long first, long long m,
                             const u64* off, u64* key, u32* val) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  long long c0[3], c1[3];
  cell_range(g, lo + (first + i) * 3, hi + (first + i) * 3, c0, c1);
  u64 o = off[i];
  for (long long x = c0[0]; x <= c1[0]; ++x)
    for (long long y = c0[1]; y <= c1[1]; ++y)
      for (long long z = c0[2]; z <= c1[2]; ++z) {
        key[o] = cell_key(g, x, y, z);
        val[o] = (u32)i;
        ++o;
      }
}

__device__ __forceinline__ long long lower_bound(const u64* a, long long n, u64 k) {
  long long l = 0, h = n;
  while (l < h) {
    const long long m = (l + h) >> 1;
    if (a[m] < k) l = m + 1;
    else h = m;
  }
  return l;
}

__device__ __forceinline__ bool overlap(const double* la, const double* ha, const double* lb,
                                        const double* hb) {
  return la[0] <= hb[0] && lb[0] <= ha[0] && la[1] <= hb[1] && lb[1] <= ha[1] && la[2] <= hb[2] &&
         lb[2] <= ha[2];
}

// Pairs of A primitive a (boxes [a_first + a]) against the B grid (boxes
// [b_first + b]); EMIT = false counts, true writes (a << bbits | b) keys.
// kind 0: A = vertices, B = triangles; kind 1: A = B = edges, b > a.
template <bool EMIT>
__global__ void k_pairs(Grid g, const double* lo, const double* hi, int kind, long long a_first,
                        long long na, long long b_first, const u64* ekey, const u32* eval,
                        long long ne, const int64_t* tris, const int64_t* edges, u64* cnt,
                        const u64* off, u64* out, int bbits) {
  const long long a = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= na) return;
  const double* la = lo + (a_first + a) * 3;
  const double* ha = hi + (a_first + a) * 3;
  long long c0[3], c1[3];
  cell_range(g, la, ha, c0, c1);
  long long ea0 = 0, ea1 = 0;
  if (kind == 1) { ea0 = edges[2 * a]; ea1 = edges[2 * a + 1]; }
  u64 n = 0, o = EMIT ? off[a] : 0ull;
  for (long long x = c0[0]; x <= c1[0]; ++x)
    for (long long y = c0[1]; y <= c1[1]; ++y)
      for (long long z = c0[2]; z <= c1[2]; ++z) {
        const u64 ck = cell_key(g, x, y, z);
        for (long long e = lower_bound(ekey, ne, ck); e < ne && ekey[e] == ck; ++e) {
          const long long b = eval[e];
          if (kind == 1 && b <= a) continue;
          const double* lb = lo + (b_first + b) * 3;
          const double* hb = hi + (b_first + b) * 3;
          // canonical cell: per axis the larger lower-corner cell
          const long long bx = cell_of(lb[0], g.g0[0], g.inv_h, g.dim[0]);
          const long long by = cell_of(lb[1], g.g0[1], g.inv_h, g.dim[1]);
          const long long bz = cell_of(lb[2], g.g0[2], g.inv_h, g.dim[2]);
          if (x != (bx > c0[0] ? bx : c0[0]) || y != (by > c0[1] ? by : c0[1]) ||
              z != (bz > c0[2] ? bz : c0[2]))
            continue;
          if (!overlap(la, ha, lb, hb)) continue;
          if (kind == 0) {
            if (tris[3 * b] == a || tris[3 * b + 1] == a || tris[3 * b + 2] == a) continue;
          } else {
            const long long eb0 = edges[2 * b], eb1 = edges[2 * b + 1];
            if (ea0 == eb0 || ea0 == eb1 || ea1 == eb0 || ea1 == eb1) continue;
          }
          if (EMIT) out[o++] = ((u64)a << bbits) | (u64)b;
          else ++n;
        }
      }
  if (!EMIT) cnt[a] = n;
}

// sorted keys -> kind, index pairs and the [8][3] query points
__global__ void k_gather(const u64* keys, long long m, int kind, int bbits, const double* x0,
                         const double* x1, const int64_t* tris, const int64_t* edges,
                         uint8_t* okind, int64_t* opairs, double* opts) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  const u64 k = keys[r];
  const long long a = (long long)(k >> bbits), b = (long long)(k & ((1ull << bbits) - 1ull));
  long long v[4];
  if (kind == 0) {
    v[0] = a; v[1] = tris[3 * b]; v[2] = tris[3 * b + 1]; v[3] = tris[3 * b + 2];
  } else {
    v[0] = edges[2 * a]; v[1] = edges[2 * a + 1]; v[2] = edges[2 * b]; v[3] = edges[2 * b + 1];
  }
  okind[r] = (uint8_t)kind;
  opairs[2 * r] = a;
  opairs[2 * r + 1] = b;
  double* p = opts + r * 24;
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      p[3 * j + ax] = x0[v[j] * 3 + ax];
      p[12 + 3 * j + ax] = x1[v[j] * 3 + ax];
    }
}

}  // namespace tccd_bp

// ===========================================================================
// host side
// ===========================================================================
using namespace tccd_bp;

struct tccd_broad {
  cudaStream_t st;
  tccd_mesh mesh;
  Grid grid;
  double* lo;
  double* hi;
  // per kind (0 VF, 1 EE): sorted cell entries, per-A pair offsets, counts
  u64* ekey[2];
  u32* eval[2];
  long long nent[2];
  u64* poff[2];
  long long npairs[2];
  int abits[2], bbits[2];
};

namespace {

int bits_for(long long n) {  // bits to index [0, n)
  int b = 1;
  while (b < 62 && (1ll << b) < n) ++b;
  return b;
}

unsigned nblk(long long n, int t = kT) { return (unsigned)((n + t - 1) / t); }

// The broad phase allocates its temporaries stream-ordered and synchronizes
// a few times (candidate counts).  With the default pool's release threshold
// of 0 every synchronization hands the freed blocks back to the driver, and
// the next allocation maps them again (tens of ms for a million-triangle
// mesh).  The device's default pool keeps up to this much freed memory
// instead (set once per device; the caller's own allocator is not affected).
constexpr unsigned long long kPoolKeep = 4ull << 30;

cudaError_t keep_pool() {
  static bool done[64] = {false};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess || dev < 0 || dev >= 64 || done[dev]) return e;
  cudaMemPool_t pool;
  if ((e = cudaDeviceGetDefaultMemPool(&pool, dev)) != cudaSuccess) return e;
  unsigned long long keep = kPoolKeep;
  if ((e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep)) != cudaSuccess)
    return e;
  done[dev] = true;
  return cudaSuccess;
}

template <class T>
cudaError_t dalloc(T** p, long long count, cudaStream_t st) {
  return cudaMallocAsync((void**)p, (size_t)(count > 0 ? count : 1) * sizeof(T), st);
}

// exclusive scan of in[0, n) into out (may alias); returns the total on the host
cudaError_t scan(const u64* in, u64* out, long long n, u64* tmp, cudaStream_t st, u64* total) {
  const long long nb = (n + kTile - 1) / kTile;
  u64* bsum = tmp;       // [nb]
  u64* dtot = tmp + nb;  // [1]
  if (n > 0) {
    k_scan_partial<<<(unsigned)nb, kT, 0, st>>>(in, n, bsum);
    k_scan_top<<<1, kT, 0, st>>>(bsum, nb, dtot);
    k_scan_final<<<(unsigned)nb, kT, 0, st>>>(in, out, n, bsum);
  } else {
    cudaMemsetAsync(dtot, 0, sizeof(u64), st);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  e = cudaMemcpyAsync(total, dtot, sizeof(u64), cudaMemcpyDeviceToHost, st);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(st);
}

// stable LSD radix sort of keys (and optional values) on bits [0, nbits);
// the result ends in the buffers passed as k0 / v0 (k1 / v1 are scratch)
cudaError_t radix_sort(u64* k0, u32* v0, u64* k1, u32* v1, long long n, int nbits, u64* tmp,
                       cudaStream_t st) {
  if (n <= 1) return cudaSuccess;
  const long long nb = (n + kTile - 1) / kTile;
  u64* bsum = tmp;
  u64* dz = tmp + nb;
  for (int bit = 0; bit < nbits; ++bit) {
    k_bit_count<<<(unsigned)nb, kT, 0, st>>>(k0, n, bit, bsum);
    k_scan_top<<<1, kT, 0, st>>>(bsum, nb, dz);
    k_bit_scatter<<<(unsigned)nb, kT, 0, st>>>(k0, v0, k1, v1, n, bit, bsum, dz);
    u64* tk = k0; k0 = k1; k1 = tk;
    u32* tv = v0; v0 = v1; v1 = tv;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (nbits & 1) {  // odd pass count: the result sits in the scratch buffers
    e = cudaMemcpyAsync(k1, k0, n * sizeof(u64), cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess && v0) e = cudaMemcpyAsync(v1, v0, n * sizeof(u32), cudaMemcpyDeviceToDevice, st);
  }
  return e;
}

#define TRY(x)                                  \
  do {                                          \
    if ((x) != cudaSuccess) return TCCD_E_CUDA; \
  } while (0)

}  // namespace

extern "C" {

int tccd_broad_create(const tccd_mesh* m, double inflation, tccd_broad** out, int64_t* n_vf,
                      int64_t* n_ee, void* stream) {
  if (!m || !out || !n_vf || !n_ee) return TCCD_E_NULL;
  *out = nullptr;
  if (m->struct_size != sizeof(tccd_mesh)) return TCCD_E_STRUCT;
  if (!(inflation >= 0.0 && inflation < INFINITY)) return TCCD_E_SEPARATION;
  const long long nv = m->n_vertices, nt = m->n_triangles, ne = m->n_edges;
  if (nv < 0 || nt < 0 || ne < 0) return TCCD_E_N;
  if (nv > 0 && (!m->x0 || !m->x1)) return TCCD_E_NULL;
  if ((nt > 0 && !m->triangles) || (ne > 0 && !m->edges)) return TCCD_E_NULL;
  if (nv >= (1ll << 31) || nt >= (1ll << 31) || ne >= (1ll << 31)) return TCCD_E_CAPACITY;
  if (keep_pool() != cudaSuccess) return TCCD_E_CUDA;
  tccd_broad* h = new tccd_broad;
  memset(h, 0, sizeof(*h));
  h->st = (cudaStream_t)stream;
  h->mesh = *m;
  cudaStream_t st = h->st;
  *out = h;
  *n_vf = *n_ee = 0;
  if (nv == 0) return TCCD_OK;

  // 1. boxes: vertices [0, nv), triangles [nv, nv + nt), edges [nv + nt, N)
  const long long N = nv + nt + ne;
  TRY(dalloc(&h->lo, 3 * N, st));
  TRY(dalloc(&h->hi, 3 * N, st));
  k_boxes<<<nblk(nv), kT, 0, st>>>(m->x0, m->x1, nullptr, 1, nv, inflation, h->lo, h->hi);
  if (nt) k_boxes<<<nblk(nt), kT, 0, st>>>(m->x0, m->x1, m->triangles, 3, nt, inflation,
                                           h->lo + 3 * nv, h->hi + 3 * nv);
  if (ne) k_boxes<<<nblk(ne), kT, 0, st>>>(m->x0, m->x1, m->edges, 2, ne, inflation,
                                           h->lo + 3 * (nv + nt), h->hi + 3 * (nv + nt));
  const int rb = (int)(N < 256 * kT ? nblk(N) : 256);
  Red* part;
  TRY(dalloc(&part, rb, st));
  k_reduce_partial<<<rb, kT, 0, st>>>(h->lo, h->hi, N, nv, part);
  k_reduce_final<<<1, 32, 0, st>>>(part, rb);
  Red r;
  TRY(cudaGetLastError());
  TRY(cudaMemcpyAsync(&r, part, sizeof(Red), cudaMemcpyDeviceToHost, st));
  TRY(cudaStreamSynchronize(st));
  TRY(cudaFreeAsync(part, st));
  // cell size: the mean largest extent of the triangle / edge boxes (the
  // reference uses the mean swept-box diagonal, scene.py:245-247; any
  // positive size gives the same pair set), at most 2^20 cells per axis
  Grid& g = h->grid;
  double hh = nt + ne > 0 ? r.ext / (double)(nt + ne) : 0.0;
  for (int a = 0; a < 3; ++a) {
    const double span = r.mx[a] - r.mn[a];
    const double lim = span / (double)(1 << kMaxDimBits) * 1.0001;
    if (hh < lim) hh = lim;
  }
  if (!(hh > 0.0 && hh < INFINITY)) hh = 1.0;
  g.h = hh;
  g.inv_h = 1.0 / hh;
  for (int a = 0; a < 3; ++a) {
    g.g0[a] = r.mn[a];
    double d = floor((r.mx[a] - r.mn[a]) * g.inv_h) + 1.0;
    if (!(d >= 1.0)) d = 1.0;
    if (d > (double)(1 << kMaxDimBits)) d = (double)(1 << kMaxDimBits);
    g.dim[a] = (long long)d;
    g.bits[a] = g.dim[a] > 1 ? bits_for(g.dim[a]) : 0;
  }
  const int cbits = g.bits[0] + g.bits[1] + g.bits[2];

  // scratch for scans / radix passes
  const long long nmax = (N > 1 ? N : 1);
  u64* tmp;
  TRY(dalloc(&tmp, (nmax + kTile - 1) / kTile + 2, st));

  for (int kind = 0; kind < 2; ++kind) {
    const long long nb_ = kind == 0 ? nt : ne;    // grid side
    const long long na = kind == 0 ? nv : ne;     // query side
    const long long b_first = kind == 0 ? nv : nv + nt;
    const long long a_first = kind == 0 ? 0 : nv + nt;
    h->abits[kind] = bits_for(na);
    h->bbits[kind] = bits_for(nb_);
    if (nb_ == 0 || na == 0) continue;
    // 2. cell entries of the grid side, sorted by cell (ids ascending per cell)
    u64* cnt;
    TRY(dalloc(&cnt, nb_, st));
    k_entry_counts<<<nblk(nb_), kT, 0, st>>>(g, h->lo, h->hi, b_first, nb_, cnt);
    u64* tmp2;
    TRY(dalloc(&tmp2, (nb_ + kTile - 1) / kTile + 2, st));
    u64 nent = 0;
    TRY(scan(cnt, cnt, nb_, tmp2, st, &nent));
    TRY(cudaFreeAsync(tmp2, st));
    h->nent[kind] = (long long)nent;
    u64* k1;
    u32* v1;
    TRY(dalloc(&h->ekey[kind], nent, st));
    TRY(dalloc(&h->eval[kind], nent, st));
    TRY(dalloc(&k1, nent, st));
    TRY(dalloc(&v1, nent, st));
    k_entry_fill<<<nblk(nb_), kT, 0, st>>>(g, h->lo, h->hi, b_first, nb_, cnt, h->ekey[kind],
                                           h->eval[kind]);
    TRY(cudaGetLastError());
    TRY(cudaFreeAsync(cnt, st));
    u64* tmp3;
    TRY(dalloc(&tmp3, ((long long)nent + kTile - 1) / kTile + 2, st));
    TRY(radix_sort(h->ekey[kind], h->eval[kind], k1, v1, (long long)nent, cbits, tmp3, st));
    TRY(cudaFreeAsync(tmp3, st));
    TRY(cudaFreeAsync(k1, st));
    TRY(cudaFreeAsync(v1, st));
    // 3. pair counts per query-side primitive -> offsets
    TRY(dalloc(&h->poff[kind], na, st));
    k_pairs<false><<<nblk(na), kT, 0, st>>>(g, h->lo, h->hi, kind, a_first, na, b_first,
                                            h->ekey[kind], h->eval[kind], (long long)nent,
                                            m->triangles, m->edges, h->poff[kind], nullptr,
                                            nullptr, h->bbits[kind]);
    TRY(cudaGetLastError());
    u64* tmp4;
    TRY(dalloc(&tmp4, (na + kTile - 1) / kTile + 2, st));
    u64 np = 0;
    TRY(scan(h->poff[kind], h->poff[kind], na, tmp4, st, &np));
    TRY(cudaFreeAsync(tmp4, st));
    h->npairs[kind] = (long long)np;
  }
  TRY(cudaFreeAsync(tmp, st));
  TRY(cudaStreamSynchronize(st));
  *n_vf = h->npairs[0];
  *n_ee = h->npairs[1];
  return TCCD_OK;
}

int tccd_broad_emit(tccd_broad* h, uint8_t* kind, int64_t* pairs, double* points) {
  if (!h) return TCCD_E_NULL;
  const long long m = h->npairs[0] + h->npairs[1];
  if (m == 0) return TCCD_OK;
  if (!kind || !pairs || !points) return TCCD_E_NULL;
  cudaStream_t st = h->st;
  const tccd_mesh& me = h->mesh;
  const Grid& g = h->grid;
  const long long nv = me.n_vertices, nt = me.n_triangles, ne = me.n_edges;
  long long row = 0;
  for (int k = 0; k < 2; ++k) {
    const long long np = h->npairs[k];
    if (np == 0) continue;
    const long long na = k == 0 ? nv : ne;
    const long long a_first = k == 0 ? 0 : nv + nt;
    const long long b_first = k == 0 ? nv : nv + nt;
    u64 *k0, *k1, *tmp;
    TRY(dalloc(&k0, np, st));
    TRY(dalloc(&k1, np, st));
    TRY(dalloc(&tmp, (np + kTile - 1) / kTile + 2, st));
    k_pairs<true><<<nblk(na), kT, 0, st>>>(g, h->lo, h->hi, k, a_first, na, b_first, h->ekey[k],
                                           h->eval[k], h->nent[k], me.triangles, me.edges,
                                           nullptr, h->poff[k], k0, h->bbits[k]);
    TRY(cudaGetLastError());
    const int nbits = h->abits[k] + h->bbits[k];
    TRY(radix_sort(k0, nullptr, k1, nullptr, np, nbits, tmp, st));
    k_gather<<<nblk(np), kT, 0, st>>>(k0, np, k, h->bbits[k], me.x0, me.x1, me.triangles,
                                      me.edges, kind + row, pairs + 2 * row,
                                      points + 24 * row);
    TRY(cudaGetLastError());
    TRY(cudaFreeAsync(k0, st));
    TRY(cudaFreeAsync(k1, st));
    TRY(cudaFreeAsync(tmp, st));
    row += np;
  }
  return TCCD_OK;
}

void tccd_broad_destroy(tccd_broad* h) {
  if (!h) return;
  cudaStream_t st = h->st;
  cudaFreeAsync(h->lo, st);
  cudaFreeAsync(h->hi, st);
  for (int k = 0; k < 2; ++k) {
    cudaFreeAsync(h->ekey[k], st);
    cudaFreeAsync(h->eval[k], st);
    cudaFreeAsync(h->poff[k], st);
  }
  delete h;
}

}  // extern "C"
