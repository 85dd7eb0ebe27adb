// SOFC / SOFG containers streamed between files and device memory (row 8(f).2; reference
// core.py:179-225).  Format (the reference's, byte for byte): 4-byte magic "SOFC" (coefficients)
// or "SOFG" (samples), little-endian u32 format version (1) and u32 bandwidth, then the payload
// as little-endian complex128 in the reference's order (coefficients l-major; samples
// [i = alpha][j = beta][k = gamma]).
//
// The reference reads a whole file into one bytes object and converts it (two copies of a
// 17 GB grid at B = 512).  Here a beta slab [jbase, jbase + J) of a grid -- the whole grid for
// J = 2B, one rank's slab for a sharded plan -- is read with pread() in pieces of whole
// [i][jj][k] rows into two pinned bounce buffers and copied to the device while the next piece
// is read, so host staging stays at 2 x `staging` bytes.  The reference rejects non-finite
// payloads on read and write; that check runs on the device (one pass over the slab) instead
// of on the host.
#pragma once
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cerrno>
#include <cstring>
#include <thread>
#include <vector>

namespace so3io {

constexpr int kHeader = 12;
constexpr uint32_t kVersion = 1;

struct Header {
  int kind;          // 0 = SOFC, 1 = SOFG
  int bandwidth;
  int64_t elements;  // payload complex128 elements
};

inline int64_t expected_elements(int kind, int b) {
  return kind == 0 ? (int64_t)b * (4LL * b * b - 1) / 3 : (int64_t)(2LL * b) * (2LL * b) * (2LL * b);
}

// 0 on success; otherwise an SO3_ERR_* code with the message in *why
// want: 0 = SOFC, 1 = SOFG, -1 = either (messages as the reference's core.py:190-198)
inline int parse_header(int fd, const char* path, Header* h, std::string* why, int want = -1) {
  unsigned char buf[kHeader];
  const ssize_t got = pread(fd, buf, kHeader, 0);
  struct stat st;
  if (fstat(fd, &st) != 0) { *why = std::string(path) + ": " + strerror(errno); return SO3_ERR_INVALID; }
  const bool sofc = got == kHeader && memcmp(buf, "SOFC", 4) == 0, sofg = got == kHeader && memcmp(buf, "SOFG", 4) == 0;
  if ((want == 0 && !sofc) || (want == 1 && !sofg) || (!sofc && !sofg)) {
    *why = std::string(path) + ": not a " + (want == 0 ? "SOFC" : want == 1 ? "SOFG" : "SOFC/SOFG") + " container";
    return SO3_ERR_INVALID;
  }
  uint32_t version, b;
  memcpy(&version, buf + 4, 4);
  memcpy(&b, buf + 8, 4);
  if (version != kVersion) {
    *why = std::string(path) + ": unsupported format version " + std::to_string(version);
    return SO3_ERR_INVALID;
  }
  h->kind = memcmp(buf, "SOFG", 4) == 0 ? 1 : 0;
  h->bandwidth = (int)b;
  const int64_t payload = (int64_t)st.st_size - kHeader;
  if (payload % 16) { *why = std::string(path) + ": truncated payload"; return SO3_ERR_INVALID; }
  h->elements = payload / 16;
  if (b < 1 || h->elements != expected_elements(h->kind, (int)b)) {
    *why = std::string(path) + ": payload length " + std::to_string(h->elements) + " does not match bandwidth " +
           std::to_string(b);
    return SO3_ERR_INVALID;
  }
  return SO3_OK;
}

inline bool pread_all(int fd, void* dst, size_t bytes, off_t off) {
  char* p = static_cast<char*>(dst);
  while (bytes) {
    const ssize_t r = pread(fd, p, bytes, off);
    if (r <= 0) {
      if (r < 0 && errno == EINTR) continue;
      return false;
    }
    p += r;
    off += r;
    bytes -= (size_t)r;
  }
  return true;
}

inline bool pwrite_all(int fd, const void* src, size_t bytes, off_t off) {
  const char* p = static_cast<const char*>(src);
  while (bytes) {
    const ssize_t r = pwrite(fd, p, bytes, off);
    if (r <= 0) {
      if (r < 0 && errno == EINTR) continue;
      return false;
    }
    p += r;
    off += r;
    bytes -= (size_t)r;
  }
  return true;
}

// count of non-finite doubles (reference: "payload contains non-finite values")
__global__ void count_nonfinite_kernel(const double* v, long long count, unsigned long long* bad) {
  unsigned long long local = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x)
    local += !isfinite(v[i]);
  for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(bad, local);
}

inline int device_nonfinite(const void* dev, long long doubles, cudaStream_t st, unsigned long long* out) {
  unsigned long long* d_bad = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&d_bad, sizeof(unsigned long long), st);
  e = e ? e : cudaMemsetAsync(d_bad, 0, sizeof(unsigned long long), st);
  if (e) return SO3_ERR_CUDA;
  int dev_id = 0, sms = 148;
  cudaGetDevice(&dev_id);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev_id);
  count_nonfinite_kernel<<<sms * 8, 256, 0, st>>>(static_cast<const double*>(dev), doubles, d_bad);
  e = cudaGetLastError();
  e = e ? e : cudaMemcpyAsync(out, d_bad, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st);
  e = e ? e : cudaStreamSynchronize(st);
  cudaFreeAsync(d_bad, st);
  return e ? SO3_ERR_CUDA : SO3_OK;
}

// A run of `rows` file rows of `row_bytes`, row r at file offset off0 + r * file_stride and at
// device offset r * row_bytes (contiguous device destination / source).
struct Rows {
  off_t off0;
  off_t file_stride;
  size_t row_bytes;
  long long rows;
};

// file -> device, double-buffered through pinned staging
inline int stream_in(int fd, const Rows& rw, char* dev, size_t staging, cudaStream_t st, std::string* why) {
  const long long per = std::max<long long>(1, (long long)(staging / rw.row_bytes));
  const size_t buf_bytes = (size_t)std::min<long long>(per, rw.rows) * rw.row_bytes;
  char* host[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  int rc = SO3_OK;
  for (int k = 0; k < 2 && rc == SO3_OK; ++k) {
    if (cudaHostAlloc((void**)&host[k], buf_bytes, cudaHostAllocDefault) != cudaSuccess ||
        cudaEventCreateWithFlags(&done[k], cudaEventDisableTiming) != cudaSuccess) {
      *why = "pinned staging allocation failed";
      rc = SO3_ERR_NOMEM;
    }
  }
  long long r0 = 0;
  for (int k = 0; rc == SO3_OK && r0 < rw.rows; ++k, r0 += per) {
    const int s = k & 1;
    const long long nr = std::min(per, rw.rows - r0);
    if (k >= 2 && cudaEventSynchronize(done[s]) != cudaSuccess) { rc = SO3_ERR_CUDA; break; }
    bool ok = true;
    if (rw.file_stride == (off_t)rw.row_bytes) {
      ok = pread_all(fd, host[s], (size_t)nr * rw.row_bytes, rw.off0 + (off_t)r0 * rw.file_stride);
    } else {
      for (long long r = 0; ok && r < nr; ++r)
        ok = pread_all(fd, host[s] + r * rw.row_bytes, rw.row_bytes, rw.off0 + (off_t)(r0 + r) * rw.file_stride);
    }
    if (!ok) { *why = std::string("read failed: ") + strerror(errno); rc = SO3_ERR_INVALID; break; }
    if (cudaMemcpyAsync(dev + r0 * rw.row_bytes, host[s], (size_t)nr * rw.row_bytes, cudaMemcpyHostToDevice, st) !=
            cudaSuccess ||
        cudaEventRecord(done[s], st) != cudaSuccess) {
      rc = SO3_ERR_CUDA;
      break;
    }
  }
  if (cudaStreamSynchronize(st) != cudaSuccess && rc == SO3_OK) rc = SO3_ERR_CUDA;
  for (int k = 0; k < 2; ++k) {
    if (host[k]) cudaFreeHost(host[k]);
    if (done[k]) cudaEventDestroy(done[k]);
  }
  return rc;
}

// device -> file, double-buffered: the copy of piece k+1 overlaps the write of piece k
inline int stream_out(int fd, const Rows& rw, const char* dev, size_t staging, cudaStream_t st, std::string* why) {
  const long long per = std::max<long long>(1, (long long)(staging / rw.row_bytes));
  const size_t buf_bytes = (size_t)std::min<long long>(per, rw.rows) * rw.row_bytes;
  char* host[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  int rc = SO3_OK;
  for (int k = 0; k < 2 && rc == SO3_OK; ++k) {
    if (cudaHostAlloc((void**)&host[k], buf_bytes, cudaHostAllocDefault) != cudaSuccess ||
        cudaEventCreateWithFlags(&done[k], cudaEventDisableTiming) != cudaSuccess) {
      *why = "pinned staging allocation failed";
      rc = SO3_ERR_NOMEM;
    }
  }
  const long long pieces = (rw.rows + per - 1) / per;
  auto issue = [&](long long k) {
    const long long a = k * per, nr = std::min(per, rw.rows - a);
    return cudaMemcpyAsync(host[k & 1], dev + a * rw.row_bytes, (size_t)nr * rw.row_bytes, cudaMemcpyDeviceToHost,
                           st) == cudaSuccess &&
           cudaEventRecord(done[k & 1], st) == cudaSuccess;
  };
  if (rc == SO3_OK && pieces > 0 && !issue(0)) rc = SO3_ERR_CUDA;
  for (long long k = 0; rc == SO3_OK && k < pieces; ++k) {
    if (cudaEventSynchronize(done[k & 1]) != cudaSuccess) { rc = SO3_ERR_CUDA; break; }
    if (k + 1 < pieces && !issue(k + 1)) { rc = SO3_ERR_CUDA; break; }
    const long long a = k * per, nr = std::min(per, rw.rows - a);
    bool ok = true;
    if (rw.file_stride == (off_t)rw.row_bytes) {
      ok = pwrite_all(fd, host[k & 1], (size_t)nr * rw.row_bytes, rw.off0 + (off_t)a * rw.file_stride);
    } else {
      for (long long r = 0; ok && r < nr; ++r)
        ok = pwrite_all(fd, host[k & 1] + r * rw.row_bytes, rw.row_bytes, rw.off0 + (off_t)(a + r) * rw.file_stride);
    }
    if (!ok) { *why = std::string("write failed: ") + strerror(errno); rc = SO3_ERR_INVALID; }
  }
  cudaStreamSynchronize(st);
  for (int k = 0; k < 2; ++k) {
    if (host[k]) cudaFreeHost(host[k]);
    if (done[k]) cudaEventDestroy(done[k]);
  }
  return rc;
}

// The rows of a container that hold beta slab [jbase, jbase + J) of a grid (kind 1), or the
// whole coefficient payload (kind 0): one row per alpha index i of J * 2B elements.
inline Rows slab_rows(int kind, int b, int jbase, int J) {
  if (kind == 0) return Rows{kHeader, 16, 16, expected_elements(0, b)};   // contiguous elements
  const long long n = 2LL * b;
  return Rows{(off_t)(kHeader + (long long)jbase * n * 16), (off_t)(n * n * 16), (size_t)(J * n * 16), n};
}

// host-side check for host buffers, split over the host's cores
inline long long host_nonfinite(const double* v, long long count) {
  const unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  std::vector<long long> bad(nt, 0);
  std::vector<std::thread> th;
  const long long per = (count + nt - 1) / nt;
  for (unsigned t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      const long long a = t * per, e = std::min(count, a + per);
      long long k = 0;
      for (long long i = a; i < e; ++i) k += !std::isfinite(v[i]);
      bad[t] = k;
    });
  long long total = 0;
  for (unsigned t = 0; t < nt; ++t) {
    th[t].join();
    total += bad[t];
  }
  return total;
}

}  // namespace so3io
