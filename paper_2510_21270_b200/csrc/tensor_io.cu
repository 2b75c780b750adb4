// tensor_io.cu -- the reference's PBST tensor files (tensor_io.hpp) straight to
// and from device memory.
//
// File layout (tensor_io.hpp:23-29): "PBST", u32 version 1, u32 dtype
// (0 = f32, 1 = f64), u32 ndim (2 or 3), ndim x u64 shape, row-major
// little-endian payload.  A 3-D file is a [heads, rows, cols] stack, the
// [H, N, d] layout every device entry point takes.
//
// Loading streams the payload through two pinned chunks: while the host reads
// chunk i + 1 from the file, chunk i is copied to the device and widened /
// narrowed there into the destination dtype (bf16 or f32), and the conversion
// kernel records the first non-finite element (parse_payload's check,
// tensor_io.hpp:80-81).  Saving runs the same pipeline backwards.  Header
// validation and error texts follow read_tensor (tensor_io.hpp:98-146) and
// write_tensor (155-186) so callers see the reference's E_IO / E_FORMAT /
// E_SHAPE lines.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <sys/stat.h>

#include <cstring>
#include <mutex>
#include <string>

#include "common.cuh"
#include "pbs_cabi.h"

namespace pbs_b200 {
namespace {

constexpr size_t kChunkBytes = size_t(64) << 20;  // per pinned / device staging chunk

int format_error(const std::string& msg, uint64_t offset) {
  return fail(PBS_ERR_IO, "E_FORMAT", msg + " (byte offset " + std::to_string(offset) + ")");
}

struct Staging {
  std::mutex mu;
  int device = -1;
  void* host[2] = {nullptr, nullptr};
  void* dev[2] = {nullptr, nullptr};
  unsigned long long* bad = nullptr;  // first non-finite element index (load)
  cudaEvent_t done[2] = {nullptr, nullptr};
};
Staging g_stage;

int staging_ready(Staging& S) {
  int dev = 0;
  PBS_CUDA_CHECK(cudaGetDevice(&dev));
  if (S.device == dev && S.host[0]) return PBS_OK;
  for (int i = 0; i < 2; ++i) {
    if (!S.host[i]) PBS_CUDA_CHECK(cudaMallocHost(&S.host[i], kChunkBytes));
    PBS_CUDA_CHECK(cudaMalloc(&S.dev[i], kChunkBytes));
    PBS_CUDA_CHECK(cudaEventCreateWithFlags(&S.done[i], cudaEventDisableTiming));
  }
  PBS_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&S.bad), sizeof(unsigned long long)));
  S.device = dev;
  return PBS_OK;
}

__device__ __forceinline__ bool finite_val(double x) { return isfinite(x); }

// file element type F -> device element type D, recording the first non-finite index
template <typename F, typename D>
__global__ void load_convert_kernel(const F* __restrict__ src, D* __restrict__ dst, int64_t count, uint64_t base,
                                    unsigned long long* __restrict__ bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const F x = src[i];
    if (!finite_val((double)x)) atomicMin(bad, (unsigned long long)(base + i));
    if constexpr (sizeof(D) == 2) dst[i] = __float2bfloat16_rn((float)x);
    else dst[i] = (D)x;
  }
}

template <typename S, typename F>
__global__ void save_convert_kernel(const S* __restrict__ src, F* __restrict__ dst, int64_t count) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    if constexpr (sizeof(S) == 2) dst[i] = (F)__bfloat162float(src[i]);
    else dst[i] = (F)src[i];
  }
}

unsigned grid_of(int64_t count) {
  const int64_t b = (count + 255) / 256;
  return (unsigned)(b < 4096 ? (b > 0 ? b : 1) : 4096);
}

struct Header {
  pbs_tensor_info info;
  uint64_t header_size;
  uint64_t payload_bytes;
};

// read_tensor's header checks (tensor_io.hpp:98-146), in the same order
int parse_header(const char* path, FILE* f, uint64_t file_size, Header* h) {
  unsigned char b[40];
  const size_t got = fread(b, 1, file_size < 40 ? (size_t)file_size : 40, f);
  if (got != (file_size < 40 ? file_size : 40)) return fail(PBS_ERR_IO, "E_IO", std::string("failed reading '") + path + "'");
  auto u32 = [&](size_t off) {
    uint32_t v;
    memcpy(&v, b + off, 4);
    return v;
  };
  if (file_size < 4 || memcmp(b, "PBST", 4) != 0) return format_error("bad magic, expected \"PBST\"", 0);
  if (file_size < 8) return format_error("truncated before version field", file_size);
  const uint32_t version = u32(4);
  if (version != 1) return format_error("unsupported version " + std::to_string(version), 4);
  if (file_size < 12) return format_error("truncated before dtype field", file_size);
  const uint32_t dtype = u32(8);
  if (dtype > 1) return format_error("unknown dtype code " + std::to_string(dtype), 8);
  if (file_size < 16) return format_error("truncated before ndim field", file_size);
  const uint32_t ndim = u32(12);
  if (ndim != 2 && ndim != 3) return format_error("ndim must be 2 or 3, got " + std::to_string(ndim), 12);
  const uint64_t header_size = 16 + (uint64_t)ndim * 8;
  if (file_size < header_size) return format_error("truncated shape header", file_size);
  uint64_t dims[3] = {1, 0, 0};
  for (uint32_t i = 0; i < ndim; ++i) memcpy(&dims[i + (3 - ndim)], b + 16 + i * 8, 8);
  const uint64_t heads = ndim == 3 ? dims[0] : 1, rows = dims[1], cols = dims[2];
  const uint64_t esize = dtype == 0 ? 4 : 8;
  uint64_t elems = heads;
  for (uint64_t dim : {rows, cols}) {
    if (dim != 0 && elems > UINT64_MAX / dim) return format_error("shape product overflows", 16);
    elems *= dim;
  }
  if (elems > (uint64_t(1) << 40)) return format_error("shape product exceeds supported tensor size", 16);
  const uint64_t payload = elems * esize;
  if (file_size < header_size + payload)
    return format_error("payload truncated, expected " + std::to_string(payload) + " bytes", file_size);
  if (file_size > header_size + payload) return format_error("trailing bytes after payload", header_size + payload);
  h->info.file_dtype = (int32_t)dtype;
  h->info.ndim = (int32_t)ndim;
  h->info.heads = (int64_t)heads;
  h->info.rows = (int64_t)rows;
  h->info.cols = (int64_t)cols;
  h->info.payload_offset = (int64_t)header_size;
  h->header_size = header_size;
  h->payload_bytes = payload;
  return PBS_OK;
}

int open_and_parse(const char* path, FILE** fp, Header* h) {
  if (!path) return fail(PBS_ERR_CONFIG, "E_CONFIG", "null path");
  struct stat st;
  FILE* f = fopen(path, "rb");
  if (!f || stat(path, &st) != 0) {
    if (f) fclose(f);
    return fail(PBS_ERR_IO, "E_IO", std::string("cannot open '") + path + "' for reading");
  }
  if (int rc = parse_header(path, f, (uint64_t)st.st_size, h)) {
    fclose(f);
    return rc;
  }
  *fp = f;
  return PBS_OK;
}

}  // namespace
}  // namespace pbs_b200

using namespace pbs_b200;

extern "C" {

int pbs_tensor_info_read(const char* path, pbs_tensor_info* info) {
  if (!info) return fail(PBS_ERR_CONFIG, "E_CONFIG", "null info");
  FILE* f = nullptr;
  Header h;
  if (int rc = open_and_parse(path, &f, &h)) return rc;
  fclose(f);
  *info = h.info;
  return PBS_OK;
}

int pbs_tensor_load(const char* path, void* dst, int32_t dst_dtype, void* stream) {
  if (dst_dtype != PBS_DTYPE_F32 && dst_dtype != PBS_DTYPE_BF16)
    return fail(PBS_ERR_CONFIG, "E_CONFIG", "load dtype must be f32 or bf16");
  FILE* f = nullptr;
  Header h;
  if (int rc = open_and_parse(path, &f, &h)) return rc;
  struct Closer {
    FILE* f;
    ~Closer() { fclose(f); }
  } closer{f};
  if (h.payload_bytes == 0) return PBS_OK;
  if (!dst) return fail(PBS_ERR_CONFIG, "E_CONFIG", "null destination");
  Staging& S = g_stage;
  std::lock_guard<std::mutex> lk(S.mu);
  if (int rc = staging_ready(S)) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint64_t esize = h.info.file_dtype == 0 ? 4 : 8;
  const uint64_t chunk_elems = kChunkBytes / esize;
  const uint64_t elems = h.payload_bytes / esize;
  const size_t dsize = dst_dtype == PBS_DTYPE_BF16 ? 2 : 4;
  PBS_CUDA_CHECK(cudaMemsetAsync(S.bad, 0xff, sizeof(unsigned long long), st));
  if (fseek(f, (long)h.header_size, SEEK_SET) != 0)
    return fail(PBS_ERR_IO, "E_IO", std::string("failed reading '") + path + "'");
  int i = 0;
  for (uint64_t e0 = 0; e0 < elems; e0 += chunk_elems, i ^= 1) {
    const uint64_t cnt = elems - e0 < chunk_elems ? elems - e0 : chunk_elems;
    // the H2D that last read this pinned chunk is done (the device chunk is
    // reused in stream order after its conversion kernel)
    PBS_CUDA_CHECK(cudaEventSynchronize(S.done[i]));
    if (fread(S.host[i], esize, cnt, f) != cnt)
      return fail(PBS_ERR_IO, "E_IO", std::string("failed reading '") + path + "'");
    PBS_CUDA_CHECK(cudaMemcpyAsync(S.dev[i], S.host[i], cnt * esize, cudaMemcpyHostToDevice, st));
    PBS_CUDA_CHECK(cudaEventRecord(S.done[i], st));
    char* d = static_cast<char*>(dst) + e0 * dsize;
    if (h.info.file_dtype == 0) {
      if (dst_dtype == PBS_DTYPE_BF16)
        load_convert_kernel<float, __nv_bfloat16><<<grid_of(cnt), 256, 0, st>>>(
            static_cast<const float*>(S.dev[i]), reinterpret_cast<__nv_bfloat16*>(d), (int64_t)cnt, e0, S.bad);
      else
        load_convert_kernel<float, float><<<grid_of(cnt), 256, 0, st>>>(
            static_cast<const float*>(S.dev[i]), reinterpret_cast<float*>(d), (int64_t)cnt, e0, S.bad);
    } else {
      if (dst_dtype == PBS_DTYPE_BF16)
        load_convert_kernel<double, __nv_bfloat16><<<grid_of(cnt), 256, 0, st>>>(
            static_cast<const double*>(S.dev[i]), reinterpret_cast<__nv_bfloat16*>(d), (int64_t)cnt, e0, S.bad);
      else
        load_convert_kernel<double, float><<<grid_of(cnt), 256, 0, st>>>(
            static_cast<const double*>(S.dev[i]), reinterpret_cast<float*>(d), (int64_t)cnt, e0, S.bad);
    }
    PBS_LAUNCH_CHECK("load_convert_kernel");
  }
  unsigned long long bad = 0;
  PBS_CUDA_CHECK(cudaMemcpyAsync(&bad, S.bad, sizeof(bad), cudaMemcpyDeviceToHost, st));
  PBS_CUDA_CHECK(cudaStreamSynchronize(st));
  if (bad != ~0ull) return format_error("non-finite element in tensor payload", h.header_size + bad * esize);
  return PBS_OK;
}

int pbs_tensor_save(const char* path, const void* src, int32_t src_dtype, int64_t heads, int64_t rows, int64_t cols,
                    int32_t file_dtype, int32_t as_stack, void* stream) {
  if (src_dtype != PBS_DTYPE_F32 && src_dtype != PBS_DTYPE_BF16)
    return fail(PBS_ERR_CONFIG, "E_CONFIG", "save source dtype must be f32 or bf16");
  if (file_dtype != 0 && file_dtype != 1) return fail(PBS_ERR_CONFIG, "E_CONFIG", "file dtype must be 0 (f32) or 1 (f64)");
  if (heads <= 0) return fail(PBS_ERR_CONFIG, "E_SHAPE", "write_tensor: empty head list");
  if (rows < 0 || cols < 0) return fail(PBS_ERR_CONFIG, "E_SHAPE", "write_tensor: negative shape");
  if (!as_stack && heads != 1) return fail(PBS_ERR_CONFIG, "E_SHAPE", "write_tensor: multiple heads require a 3-D stack");
  if (!path) return fail(PBS_ERR_CONFIG, "E_CONFIG", "null path");
  const uint64_t elems = (uint64_t)heads * (uint64_t)rows * (uint64_t)cols;
  if (elems && !src) return fail(PBS_ERR_CONFIG, "E_CONFIG", "null source");
  FILE* f = fopen(path, "wb");
  if (!f) return fail(PBS_ERR_IO, "E_IO", std::string("cannot open '") + path + "' for writing");
  struct Closer {
    FILE* f;
    ~Closer() {
      if (f) fclose(f);
    }
  } closer{f};
  unsigned char hdr[40];
  const uint32_t version = 1, dt = (uint32_t)file_dtype, ndim = as_stack ? 3 : 2;
  memcpy(hdr, "PBST", 4);
  memcpy(hdr + 4, &version, 4);
  memcpy(hdr + 8, &dt, 4);
  memcpy(hdr + 12, &ndim, 4);
  size_t off = 16;
  const uint64_t dims[3] = {(uint64_t)heads, (uint64_t)rows, (uint64_t)cols};
  for (uint32_t k = 3 - ndim; k < 3; ++k, off += 8) memcpy(hdr + off, &dims[k], 8);
  if (fwrite(hdr, 1, off, f) != off) return fail(PBS_ERR_IO, "E_IO", std::string("short write to '") + path + "'");
  if (elems) {
    Staging& S = g_stage;
    std::lock_guard<std::mutex> lk(S.mu);
    if (int rc = staging_ready(S)) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const uint64_t esize = file_dtype == 0 ? 4 : 8;
    const uint64_t chunk_elems = kChunkBytes / esize;
    const size_t ssize = src_dtype == PBS_DTYPE_BF16 ? 2 : 4;
    // chunk i converts + copies out while the host writes chunk i - 1
    uint64_t prev_cnt = 0;
    int i = 0;
    for (uint64_t e0 = 0; e0 < elems + chunk_elems; e0 += chunk_elems, i ^= 1) {
      if (e0 < elems) {
        const uint64_t cnt = elems - e0 < chunk_elems ? elems - e0 : chunk_elems;
        const char* s = static_cast<const char*>(src) + e0 * ssize;
        if (file_dtype == 0) {
          if (src_dtype == PBS_DTYPE_BF16)
            save_convert_kernel<__nv_bfloat16, float><<<grid_of(cnt), 256, 0, st>>>(
                reinterpret_cast<const __nv_bfloat16*>(s), static_cast<float*>(S.dev[i]), (int64_t)cnt);
          else
            save_convert_kernel<float, float><<<grid_of(cnt), 256, 0, st>>>(
                reinterpret_cast<const float*>(s), static_cast<float*>(S.dev[i]), (int64_t)cnt);
        } else {
          if (src_dtype == PBS_DTYPE_BF16)
            save_convert_kernel<__nv_bfloat16, double><<<grid_of(cnt), 256, 0, st>>>(
                reinterpret_cast<const __nv_bfloat16*>(s), static_cast<double*>(S.dev[i]), (int64_t)cnt);
          else
            save_convert_kernel<float, double><<<grid_of(cnt), 256, 0, st>>>(
                reinterpret_cast<const float*>(s), static_cast<double*>(S.dev[i]), (int64_t)cnt);
        }
        PBS_LAUNCH_CHECK("save_convert_kernel");
        PBS_CUDA_CHECK(cudaMemcpyAsync(S.host[i], S.dev[i], cnt * esize, cudaMemcpyDeviceToHost, st));
        PBS_CUDA_CHECK(cudaEventRecord(S.done[i], st));
      }
      if (e0 > 0) {  // write the previous chunk
        const int j = i ^ 1;
        PBS_CUDA_CHECK(cudaEventSynchronize(S.done[j]));
        if (fwrite(S.host[j], esize, prev_cnt, f) != prev_cnt)
          return fail(PBS_ERR_IO, "E_IO", std::string("short write to '") + path + "'");
      }
      prev_cnt = e0 < elems ? (elems - e0 < chunk_elems ? elems - e0 : chunk_elems) : 0;
    }
  }
  const int rc = fclose(f);
  closer.f = nullptr;
  if (rc != 0) return fail(PBS_ERR_IO, "E_IO", std::string("short write to '") + path + "'");
  return PBS_OK;
}

}  // extern "C"
