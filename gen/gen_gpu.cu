// gen_gpu.cu — device fill kernels over gen/sxgen.h (libsxgen_gpu.so).
// Generates the synthetic TPC-H-shaped tables straight into HBM (the repo
// snapshot stays small; SF100 is ~36 GB).  Byte-identical to gen_cpu.c by
// construction (same value functions) and by test (tests/test_gen_gpu.py).
// Untimed: bench.py fills tables before the timed region (hot runs).
#include "sxgen.h"
#include <cuda_runtime.h>
#include <stdint.h>

#define EXPORT extern "C" __attribute__((visibility("default")))

namespace {

constexpr int kThreads = 256;

inline unsigned grid_for(int64_t n) {
  int64_t g = (n + kThreads - 1) / kThreads;
  if (g > (1ll << 30)) g = 1ll << 30;
  return (unsigned)(g < 1 ? 1 : g);
}

__global__ void k_supplier(uint64_t seed, int64_t k0, int64_t n, int32_t* suppkey, int32_t* nationkey) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t k = k0 + t;
    if (suppkey) suppkey[t] = (int32_t)k;
    if (nationkey) nationkey[t] = sxg_s_nationkey(seed, k);
  }
}

__global__ void k_customer(uint64_t seed, int64_t k0, int64_t n, int32_t* custkey, uint8_t* seg, int32_t* nat) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t k = k0 + t;
    if (custkey) custkey[t] = (int32_t)k;
    if (seg) seg[t] = sxg_c_mktsegment(seed, k);
    if (nat) nat[t] = sxg_c_nationkey(seed, k);
  }
}

__global__ void k_part_len(uint64_t seed, int64_t k0, int64_t n, int64_t* len) {
  char buf[SXG_PNAME_MAXLEN];
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    len[t] = sxg_p_name(seed, k0 + t, buf);
}

__global__ void k_part(uint64_t seed, int64_t k0, int64_t n, int32_t* partkey, const int64_t* offsets, char* chars,
                       int64_t* retail) {
  char buf[SXG_PNAME_MAXLEN];
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t k = k0 + t;
    if (partkey) partkey[t] = (int32_t)k;
    if (retail) retail[t] = sxg_p_retailprice(k);
    if (chars) {
      int len = sxg_p_name(seed, k, buf);
      char* dst = chars + offsets[t];
      for (int c = 0; c < len; ++c) dst[c] = buf[c];
    }
  }
}

__global__ void k_partsupp(uint64_t seed, int64_t S, int64_t p0, int64_t nrows, int32_t* pk, int32_t* sk, int64_t* cost) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = p0 + r / 4, i = r % 4;
    if (pk) pk[r] = (int32_t)p;
    if (sk) sk[r] = (int32_t)sxg_ps_suppkey(p, i, S);
    if (cost) cost[r] = sxg_ps_supplycost(seed, p, i);
  }
}

__global__ void k_nlines(uint64_t seed, int64_t i0, int64_t n, int64_t* out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    out[t] = sxg_o_nlines(seed, i0 + t);
}

// ---- exclusive scan of int64 (generator-internal; three simple phases) ----
constexpr int kScanBlock = 1024;

__global__ void k_scan_local(int64_t* a, int64_t n, int64_t* block_sums) {
  __shared__ int64_t warp_tot[32];
  int64_t i = blockIdx.x * (int64_t)kScanBlock + threadIdx.x;
  int64_t v = i < n ? a[i] : 0;
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t x = v;
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  if (w == 0) {
    int64_t t = warp_tot[lane];
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    warp_tot[lane] = t;
  }
  __syncthreads();
  int64_t incl = x + (w ? warp_tot[w - 1] : 0);
  if (i < n) a[i] = incl - v;  // exclusive within block
  if (threadIdx.x == kScanBlock - 1) block_sums[blockIdx.x] = incl;
}

__global__ void k_scan_sums(int64_t* sums, int64_t nb, int64_t* total) {
  // single thread: nb is small (n / 1024)
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    int64_t run = 0;
    for (int64_t b = 0; b < nb; ++b) {
      int64_t s = sums[b];
      sums[b] = run;
      run += s;
    }
    *total = run;
  }
}

__global__ void k_scan_add(int64_t* a, int64_t n, const int64_t* sums) {
  int64_t i = blockIdx.x * (int64_t)kScanBlock + threadIdx.x;
  if (i < n) a[i] += sums[blockIdx.x];
}

// a[0..n) -> exclusive scan in place, a[n] = total. `tmp` has >= n/1024+1 int64.
void exclusive_scan(int64_t* a, int64_t n, int64_t* tmp, cudaStream_t s) {
  int64_t nb = (n + kScanBlock - 1) / kScanBlock;
  if (nb == 0) {
    cudaMemsetAsync(a, 0, sizeof(int64_t), s);
    return;
  }
  k_scan_local<<<(unsigned)nb, kScanBlock, 0, s>>>(a, n, tmp);
  k_scan_sums<<<1, 32, 0, s>>>(tmp, nb, a + n);
  k_scan_add<<<(unsigned)nb, kScanBlock, 0, s>>>(a, n, tmp);
}

template <typename K>
__global__ void k_orders_lineitem(uint64_t seed, int64_t P, int64_t S, int64_t C, int64_t i0, int64_t n,
                                  const int64_t* offsets, K* o_orderkey, int32_t* o_custkey, int32_t* o_orderdate,
                                  int32_t* o_shippriority, int64_t* o_totalprice, K* l_orderkey, int32_t* l_partkey,
                                  int32_t* l_suppkey, int64_t* l_quantity, int64_t* l_ext, int64_t* l_disc,
                                  int64_t* l_tax, uint8_t* l_rf, uint8_t* l_ls, int32_t* l_ship) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = i0 + t;
    int64_t ok = sxg_o_orderkey(i);
    int32_t od = sxg_o_orderdate(seed, i);
    int32_t nl = sxg_o_nlines(seed, i);
    if (o_orderkey) o_orderkey[t] = (K)ok;
    if (o_custkey) o_custkey[t] = (int32_t)sxg_o_custkey(seed, i, C);
    if (o_orderdate) o_orderdate[t] = od;
    if (o_shippriority) o_shippriority[t] = 0;
    int64_t r = offsets[t], total = 0;
    for (int32_t j = 1; j <= nl; ++j, ++r) {
      sxg_line L;
      sxg_l_line(seed, i, j, od, P, S, &L);
      total += sxg_line_price_term(&L);
      if (l_orderkey) l_orderkey[r] = (K)ok;
      if (l_partkey) l_partkey[r] = L.partkey;
      if (l_suppkey) l_suppkey[r] = L.suppkey;
      if (l_quantity) l_quantity[r] = L.quantity;
      if (l_ext) l_ext[r] = L.extendedprice;
      if (l_disc) l_disc[r] = L.discount;
      if (l_tax) l_tax[r] = L.tax;
      if (l_rf) l_rf[r] = L.returnflag;
      if (l_ls) l_ls[r] = L.linestatus;
      if (l_ship) l_ship[r] = L.shipdate;
    }
    if (o_totalprice) o_totalprice[t] = total;
  }
}

}  // namespace

EXPORT int sxg_gpu_fill_supplier(uint64_t seed, int64_t k0, int64_t k1, int32_t* suppkey, int32_t* nationkey,
                                 cudaStream_t s) {
  int64_t n = k1 - k0;
  if (n > 0) k_supplier<<<grid_for(n), kThreads, 0, s>>>(seed, k0, n, suppkey, nationkey);
  return (int)cudaGetLastError();
}

EXPORT int sxg_gpu_fill_customer(uint64_t seed, int64_t k0, int64_t k1, int32_t* custkey, uint8_t* seg, int32_t* nat,
                                 cudaStream_t s) {
  int64_t n = k1 - k0;
  if (n > 0) k_customer<<<grid_for(n), kThreads, 0, s>>>(seed, k0, n, custkey, seg, nat);
  return (int)cudaGetLastError();
}

// offsets: int64[n+1] (device); tmp: int64[n/1024+2] (device). After this call offsets[n] = total chars
// (caller reads it, allocates chars, then calls sxg_gpu_fill_part).
EXPORT int sxg_gpu_part_offsets(uint64_t seed, int64_t k0, int64_t k1, int64_t* offsets, int64_t* tmp, cudaStream_t s) {
  int64_t n = k1 - k0;
  if (n > 0) k_part_len<<<grid_for(n), kThreads, 0, s>>>(seed, k0, n, offsets);
  exclusive_scan(offsets, n, tmp, s);
  return (int)cudaGetLastError();
}

EXPORT int sxg_gpu_fill_part(uint64_t seed, int64_t k0, int64_t k1, int32_t* partkey, const int64_t* offsets,
                             char* chars, int64_t* retail, cudaStream_t s) {
  int64_t n = k1 - k0;
  if (n > 0) k_part<<<grid_for(n), kThreads, 0, s>>>(seed, k0, n, partkey, offsets, chars, retail);
  return (int)cudaGetLastError();
}

EXPORT int sxg_gpu_fill_partsupp(uint64_t seed, int64_t sf_milli, int64_t p0, int64_t p1, int32_t* pk, int32_t* sk,
                                 int64_t* cost, cudaStream_t s) {
  int64_t nrows = 4 * (p1 - p0);
  if (nrows > 0) k_partsupp<<<grid_for(nrows), kThreads, 0, s>>>(seed, sxg_n_supplier(sf_milli), p0, nrows, pk, sk, cost);
  return (int)cudaGetLastError();
}

// line offsets for orders [i0, i1): offsets int64[n+1] (device), offsets[n] = lineitem rows.
EXPORT int sxg_gpu_line_offsets(uint64_t seed, int64_t i0, int64_t i1, int64_t* offsets, int64_t* tmp, cudaStream_t s) {
  int64_t n = i1 - i0;
  if (n > 0) k_nlines<<<grid_for(n), kThreads, 0, s>>>(seed, i0, n, offsets);
  exclusive_scan(offsets, n, tmp, s);
  return (int)cudaGetLastError();
}

EXPORT int sxg_gpu_fill_orders_lineitem(uint64_t seed, int64_t sf_milli, int64_t i0, int64_t i1, int key_bytes,
                                        const int64_t* offsets, void* o_orderkey, int32_t* o_custkey,
                                        int32_t* o_orderdate, int32_t* o_shippriority, int64_t* o_totalprice,
                                        void* l_orderkey, int32_t* l_partkey, int32_t* l_suppkey, int64_t* l_quantity,
                                        int64_t* l_ext, int64_t* l_disc, int64_t* l_tax, uint8_t* l_rf, uint8_t* l_ls,
                                        int32_t* l_ship, cudaStream_t s) {
  int64_t n = i1 - i0;
  if (n <= 0) return 0;
  int64_t P = sxg_n_part(sf_milli), S = sxg_n_supplier(sf_milli), C = sxg_n_customer(sf_milli);
  if (key_bytes == 8)
    k_orders_lineitem<int64_t><<<grid_for(n), kThreads, 0, s>>>(
        seed, P, S, C, i0, n, offsets, (int64_t*)o_orderkey, o_custkey, o_orderdate, o_shippriority, o_totalprice,
        (int64_t*)l_orderkey, l_partkey, l_suppkey, l_quantity, l_ext, l_disc, l_tax, l_rf, l_ls, l_ship);
  else
    k_orders_lineitem<int32_t><<<grid_for(n), kThreads, 0, s>>>(
        seed, P, S, C, i0, n, offsets, (int32_t*)o_orderkey, o_custkey, o_orderdate, o_shippriority, o_totalprice,
        (int32_t*)l_orderkey, l_partkey, l_suppkey, l_quantity, l_ext, l_disc, l_tax, l_rf, l_ls, l_ship);
  return (int)cudaGetLastError();
}

// ---- operator micro-benchmarks (rows [r0, r1)) ----
namespace {
__global__ void k_mb_build(int64_t r0, int64_t n, int64_t* key, int64_t* payload) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    if (key) key[t] = (int64_t)sxg_mb_build_key(r0 + t);
    if (payload) payload[t] = r0 + t;
  }
}
__global__ void k_mb_probe(uint64_t seed, int64_t nb, int zipf, int64_t r0, int64_t n, int64_t* key, int64_t* payload) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    if (key) key[t] = (int64_t)sxg_mb_probe_key(seed, r0 + t, nb, zipf);
    if (payload) payload[t] = r0 + t;
  }
}
__global__ void k_mb_groupby(uint64_t seed, int64_t G, int64_t r0, int64_t n, int64_t* key, int64_t* value) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    if (key) key[t] = (int64_t)sxg_mix64((uint64_t)sxg_mb_gb_group(seed, r0 + t, G));
    if (value) value[t] = sxg_mb_gb_value(seed, r0 + t);
  }
}
__global__ void k_mb_sort(uint64_t seed, int64_t r0, int64_t n, int64_t* key, int32_t* payload) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    if (key) key[t] = sxg_mb_sort_key(seed, r0 + t);
    if (payload) payload[t] = (int32_t)(r0 + t);
  }
}
}  // namespace

EXPORT int sxg_gpu_fill_mb_build(int64_t r0, int64_t r1, int64_t* key, int64_t* payload, cudaStream_t s) {
  if (r1 > r0) k_mb_build<<<grid_for(r1 - r0), kThreads, 0, s>>>(r0, r1 - r0, key, payload);
  return (int)cudaGetLastError();
}
EXPORT int sxg_gpu_fill_mb_probe(uint64_t seed, int64_t nb, int zipf, int64_t r0, int64_t r1, int64_t* key,
                                 int64_t* payload, cudaStream_t s) {
  if (r1 > r0) k_mb_probe<<<grid_for(r1 - r0), kThreads, 0, s>>>(seed, nb, zipf, r0, r1 - r0, key, payload);
  return (int)cudaGetLastError();
}
EXPORT int sxg_gpu_fill_mb_groupby(uint64_t seed, int64_t G, int64_t r0, int64_t r1, int64_t* key, int64_t* value,
                                   cudaStream_t s) {
  if (r1 > r0) k_mb_groupby<<<grid_for(r1 - r0), kThreads, 0, s>>>(seed, G, r0, r1 - r0, key, value);
  return (int)cudaGetLastError();
}
EXPORT int sxg_gpu_fill_mb_sort(uint64_t seed, int64_t r0, int64_t r1, int64_t* key, int32_t* payload, cudaStream_t s) {
  if (r1 > r0) k_mb_sort<<<grid_for(r1 - r0), kThreads, 0, s>>>(seed, r0, r1 - r0, key, payload);
  return (int)cudaGetLastError();
}
