// ctx.cu — context lifecycle, stream-ordered pool, errors, profiling, sx_gather.
#include <cstdlib>

#include "common.cuh"

using namespace sx;

SX_EXPORT sx_status sx_ctx_create(int device, void* stream, sx_ctx** out) {
  sx_ctx* ctx = nullptr;
  if (!out) return SX_EINVAL;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return SX_ECUDA;  // no device: there is no CPU fallback
  }
  if (device < 0 || device >= ndev) return SX_EINVAL;
  ctx = new sx_ctx();
  ctx->device = device;
  ctx->stream = (cudaStream_t)stream;
  SX_CUDA(cudaSetDevice(device));
  SX_CUDA(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device));
  int l2 = 0;
  SX_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device));
  ctx->l2_bytes = (size_t)l2;
  // Keep freed blocks in the device's default pool (no trim between queries).
  cudaMemPool_t pool;
  SX_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t thresh = UINT64_MAX;
  SX_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh));
  // Reserve the processing region up front ("pre-allocated in advance"): growing the pool
  // later maps physical memory on the host timeline, inside whatever query first needs it.
  {
    const char* env = getenv("SX_POOL_RESERVE_GB");
    double gb = env ? atof(env) : 48.0;
    size_t freeb = 0, totalb = 0;
    cudaMemGetInfo(&freeb, &totalb);
    size_t want = (size_t)(gb * (1ull << 30));
    if (want > freeb / 2) want = freeb / 2;
    uint64_t reserved = 0;
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
    if (want > reserved) {
      void* p = nullptr;
      if (cudaMallocAsync(&p, want - reserved, ctx->stream) == cudaSuccess) cudaFreeAsync(p, ctx->stream);
      cudaGetLastError();
      cudaStreamSynchronize(ctx->stream);
    }
  }
  // L2 fetch granularity (bytes per DRAM fetch on an L2 miss; SX_L2_FETCH = 32 / 64 / 128): the
  // hot path's sparse gathers (K10w's green rows, probe lookups) touch one 32-byte sector per
  // line, so a larger fetch moves bytes nobody reads.  Unset: the driver default.
  if (const char* fe = getenv("SX_L2_FETCH")) {
    const size_t g = (size_t)atoi(fe);
    if (g == 32 || g == 64 || g == 128) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, g);
    cudaGetLastError();
  }
  SX_CUDA(cudaMalloc((void**)&ctx->d_flags, 64 * sizeof(int)));
  SX_CUDA(cudaMemset(ctx->d_flags, 0, 64 * sizeof(int)));
  SX_CUDA(cudaMalloc((void**)&ctx->d_counters, 64 * sizeof(unsigned int)));
  SX_CUDA(cudaMallocHost((void**)&ctx->h_pinned, 64 * sizeof(int64_t)));
  *out = ctx;
  return SX_OK;
}

SX_EXPORT void sx_ctx_destroy(sx_ctx* ctx) {
  if (!ctx) return;
  cudaStreamSynchronize(ctx->stream);
  for (auto& p : ctx->prof) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  cudaFree(ctx->d_flags);
  cudaFree(ctx->d_counters);
  cudaFreeHost(ctx->h_pinned);
  if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
  delete ctx;
}

SX_EXPORT const char* sx_last_error(const sx_ctx* ctx) { return ctx ? ctx->err.c_str() : "null ctx"; }

SX_EXPORT sx_status sx_free(sx_ctx* ctx, void* p) {
  if (!ctx) return SX_EINVAL;
  if (p) SX_CUDA(cudaFreeAsync(p, ctx->stream));
  return SX_OK;
}

SX_EXPORT sx_status sx_sync(sx_ctx* ctx) {
  if (!ctx) return SX_EINVAL;
  SX_CUDA(cudaStreamSynchronize(ctx->stream));
  return SX_OK;
}

SX_EXPORT sx_status sx_profile_enable(sx_ctx* ctx, int on) {
  if (!ctx) return SX_EINVAL;
  ctx->profile = on != 0;
  return SX_OK;
}

SX_EXPORT sx_status sx_profile_read(sx_ctx* ctx, char (*names)[32], float* ms, double* bytes, int cap, int* n) {
  if (!ctx || !n) return SX_EINVAL;
  SX_CUDA(cudaStreamSynchronize(ctx->stream));
  int k = 0;
  for (auto& p : ctx->prof) {
    if (k < cap) {
      float t = 0.f;
      cudaEventElapsedTime(&t, p.a, p.b);
      if (names) snprintf(names[k], 32, "%s", p.name);
      if (ms) ms[k] = t;
      if (bytes) bytes[k] = p.bytes;
      ++k;
    }
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  ctx->prof.clear();
  *n = k;
  return SX_OK;
}

namespace {
template <typename T>
__global__ void k_gather(const T* __restrict__ src, const int32_t* __restrict__ sel, int64_t n, T* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[sel[i]];
}
}  // namespace

SX_EXPORT sx_status sx_gather(sx_ctx* ctx, const sx_col* col, const sx_sel* sel, sx_col* out) {
  if (!ctx || !col || !sel || !out) return SX_EINVAL;
  *out = sx_col{};
  ProfScope ps(ctx, "gather");
  int w = type_width(col->type);
  if (w == 0) return set_err(ctx, SX_ETYPE, "sx_gather: type %d is not fixed-width", col->type);
  if (col->validity) return set_err(ctx, SX_EUNSUPPORTED, "validity bitmaps unsupported");
  if (sel->len > INT32_MAX) return set_err(ctx, SX_EINDEX, "selection too long");
  void* dst;
  SX_TRY(alloc(ctx, (char**)&dst, (size_t)sel->len * w));
  int64_t n = sel->len;
  unsigned grid = persistent_grid(ctx, 8, (n + kBlock - 1) / kBlock);
  if (n > 0) {
    switch (w) {
      case 1: k_gather<uint8_t><<<grid, kBlock, 0, SX_STREAM(ctx)>>>((const uint8_t*)col->data, sel->idx, n, (uint8_t*)dst); break;
      case 4: k_gather<int32_t><<<grid, kBlock, 0, SX_STREAM(ctx)>>>((const int32_t*)col->data, sel->idx, n, (int32_t*)dst); break;
      case 8: k_gather<long long><<<grid, kBlock, 0, SX_STREAM(ctx)>>>((const long long*)col->data, sel->idx, n, (long long*)dst); break;
      default: k_gather<longlong2><<<grid, kBlock, 0, SX_STREAM(ctx)>>>((const longlong2*)col->data, sel->idx, n, (longlong2*)dst); break;
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    dfree(ctx, dst);
    return set_err(ctx, SX_ECUDA, "gather launch: %s", cudaGetErrorString(e));
  }
  *out = *col;
  out->len = n;
  out->data = dst;
  ps.set_bytes((4.0 + 2.0 * w) * n);  // selection + referenced rows read + output written
  return SX_OK;
}

// Stream-ordered copy between any two pointers (device or host); used by the Python binding
// to move library-owned outputs into caller-owned tensors/arrays.
SX_EXPORT sx_status sx_memcpy(sx_ctx* ctx, void* dst, const void* src, size_t bytes) {
  if (!ctx) return SX_EINVAL;
  if (bytes) SX_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, ctx->stream));
  return SX_OK;
}

SX_EXPORT int64_t sx_launch_count(sx_ctx* ctx, int reset) {
  if (!ctx) return -1;
  int64_t n = ctx->launches;
  if (reset) ctx->launches = 0;
  return n;
}
