// rbd_io.cu — the RBD1 model container (reference
// proj/src/io.cpp:527-622, proj/include/rbd/io.hpp:51-64).
//
// Layout, all little-endian (io.hpp:51-56):
//   "RBD1" | u64 m, n, d | u8 weight tag (0 identity, 1 diagonal, 2 sparse SPD
//   held externally) | f64 Y column-major (m x d) | f64 T row-major (d x n) |
//   f64 eps_R | f64 residual_history[d] | (tag 1) f64 diag[m]
// The header is 29 bytes (io.cpp:554,589; test_io.cpp:303-309).
//
// Y and T are the decompose outputs as the library keeps them in HBM (Y
// column-major with leading dimension ldy, T row-major), i.e. already in file
// order. Device-resident Y/T stream through two pinned staging buffers: the
// copy of chunk i+1 overlaps the write (or read) of chunk i. Host pointers are
// written/read directly. Writes go to path + ".tmp" and are renamed into place
// (io.cpp:60-73).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cerrno>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "rbd_cuda.h"
#include "rbd_internal.h"

namespace {

constexpr char kMagic[4] = {'R', 'B', 'D', '1'};
constexpr size_t kHeader = 29;
constexpr size_t kStage = size_t(32) << 20;   // bytes per staging buffer

int err(int code, const std::string& msg) { return rbd_internal_set_error(code, msg); }
int parse_err(const char* path, const std::string& what) {   // ParseError(path, 0, what)
  return err(RBD_ERR_PARSE, std::string(path) + ":0: " + what);
}

bool on_device(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

void put_u64(unsigned char* o, uint64_t v) {   // little-endian (x86-64 and aarch64 hosts)
  std::memcpy(o, &v, 8);
}

struct File {
  FILE* f = nullptr;
  ~File() {
    if (f) fclose(f);
  }
};

// Two pinned staging buffers + events, allocated on first use and kept per
// host thread (page-locking 64 MiB costs more than streaming a model through it).
struct Pinned {
  void* p[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  int device = -1;
  ~Pinned() { reset(); }
  void reset() {
    for (int i = 0; i < 2; ++i) {
      if (ev[i]) cudaEventDestroy(ev[i]);
      if (p[i]) cudaFreeHost(p[i]);
      ev[i] = nullptr;
      p[i] = nullptr;
    }
  }
  int init(size_t bytes) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (p[0] && device == dev) return RBD_OK;
    reset();
    device = dev;
    for (int i = 0; i < 2; ++i) {
      if (cudaHostAlloc(&p[i], bytes, cudaHostAllocDefault) != cudaSuccess ||
          cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming) != cudaSuccess) {
        reset();
        return err(RBD_ERR_OUT_OF_MEMORY, "model container: pinned staging allocation failed");
      }
    }
    return RBD_OK;
  }
};

Pinned& staging() {
  thread_local Pinned pin;
  return pin;
}

// One contiguous run of doubles in file order: `cols` runs of `rows` doubles,
// the run c starting at base + c * ld (Y: rows = m, ld = ldy; T/other: cols = 1).
struct Span {
  double* base;
  int64_t rows, cols, ld;
  bool dev;
};

// Streams the spans to the file (device spans through the staging buffers).
int write_spans(FILE* f, const char* path, const std::vector<Span>& spans, cudaStream_t st) {
  Pinned& pin = staging();
  bool any_dev = false;
  for (const Span& s : spans) any_dev = any_dev || s.dev;
  if (any_dev) {
    const int rc = pin.init(kStage);
    if (rc) return rc;
  }
  const size_t per = kStage / sizeof(double);
  int slot = 0;
  // pending chunk waiting to be written: (slot, doubles)
  int pend_slot = -1;
  size_t pend_n = 0;
  auto flush_pending = [&]() -> int {
    if (pend_slot < 0) return RBD_OK;
    if (cudaEventSynchronize(pin.ev[pend_slot]) != cudaSuccess)
      return err(RBD_ERR_CUDA, "model container: device-to-host copy failed");
    if (fwrite(pin.p[pend_slot], sizeof(double), pend_n, f) != pend_n)
      return err(RBD_ERR_IO, std::string("write failed: ") + path);
    pend_slot = -1;
    return RBD_OK;
  };
  for (const Span& s : spans) {
    for (int64_t c = 0; c < s.cols; ++c) {
      const double* col = s.base + c * s.ld;
      int64_t off = 0;
      while (off < s.rows) {
        if (!s.dev) {
          int rc = flush_pending();
          if (rc) return rc;
          const size_t cnt = (size_t)(s.rows - off);
          if (fwrite(col + off, sizeof(double), cnt, f) != cnt)
            return err(RBD_ERR_IO, std::string("write failed: ") + path);
          off = s.rows;
          continue;
        }
        const size_t cnt = (size_t)std::min<int64_t>(s.rows - off, (int64_t)per);
        // the slot we are about to fill must not be the pending one
        if (slot == pend_slot) {
          int rc = flush_pending();
          if (rc) return rc;
        }
        if (cudaMemcpyAsync(pin.p[slot], col + off, cnt * sizeof(double), cudaMemcpyDeviceToHost,
                            st) != cudaSuccess ||
            cudaEventRecord(pin.ev[slot], st) != cudaSuccess)
          return err(RBD_ERR_CUDA, "model container: device-to-host copy failed");
        int rc = flush_pending();   // write the previous chunk while this one copies
        if (rc) return rc;
        pend_slot = slot;
        pend_n = cnt;
        slot ^= 1;
        off += (int64_t)cnt;
      }
    }
  }
  return flush_pending();
}

// Reads the spans from the file (device spans through the staging buffers).
int read_spans(FILE* f, const char* path, const std::vector<Span>& spans, cudaStream_t st) {
  Pinned& pin = staging();
  bool any_dev = false;
  for (const Span& s : spans) any_dev = any_dev || s.dev;
  if (any_dev) {
    const int rc = pin.init(kStage);
    if (rc) return rc;
  }
  const size_t per = kStage / sizeof(double);
  int slot = 0;
  bool used[2] = {false, false};
  for (const Span& s : spans) {
    for (int64_t c = 0; c < s.cols; ++c) {
      double* col = s.base + c * s.ld;
      int64_t off = 0;
      while (off < s.rows) {
        if (!s.dev) {
          const size_t cnt = (size_t)(s.rows - off);
          if (fread(col + off, sizeof(double), cnt, f) != cnt)
            return parse_err(path, "unexpected end of file");
          off = s.rows;
          continue;
        }
        const size_t cnt = (size_t)std::min<int64_t>(s.rows - off, (int64_t)per);
        // the staging slot is free once its previous upload finished
        if (used[slot] && cudaEventSynchronize(pin.ev[slot]) != cudaSuccess)
          return err(RBD_ERR_CUDA, "model container: host-to-device copy failed");
        if (fread(pin.p[slot], sizeof(double), cnt, f) != cnt)
          return parse_err(path, "unexpected end of file");
        if (cudaMemcpyAsync(col + off, pin.p[slot], cnt * sizeof(double), cudaMemcpyHostToDevice,
                            st) != cudaSuccess ||
            cudaEventRecord(pin.ev[slot], st) != cudaSuccess)
          return err(RBD_ERR_CUDA, "model container: host-to-device copy failed");
        used[slot] = true;
        slot ^= 1;
        off += (int64_t)cnt;
      }
    }
  }
  if (any_dev && cudaStreamSynchronize(st) != cudaSuccess)
    return err(RBD_ERR_CUDA, "model container: host-to-device copy failed");
  return RBD_OK;
}

// io.cpp:595-596 with overflow-checked arithmetic: header values come from an
// untrusted file, so a product that does not fit in 64 bits is "no size" (the
// file cannot match it) rather than a wrapped number.
bool expected_size(int64_t m, int64_t n, int64_t d, int tag, uint64_t* out) {
  uint64_t md, dn, s;
  if (__builtin_mul_overflow((uint64_t)m, (uint64_t)d, &md) ||
      __builtin_mul_overflow((uint64_t)d, (uint64_t)n, &dn) ||
      __builtin_add_overflow(md, dn, &s) || __builtin_add_overflow(s, (uint64_t)(1 + d), &s) ||
      (tag == 1 && __builtin_add_overflow(s, (uint64_t)m, &s)) ||
      __builtin_mul_overflow(s, (uint64_t)8, &s) || __builtin_add_overflow(s, (uint64_t)kHeader, &s))
    return false;
  *out = s;
  return true;
}

}  // namespace

int rbd_model_write(rbd_ctx_t ctx, const char* path, int64_t m, int64_t n, int64_t d,
                    const double* Y, int64_t ldy, const double* T, double eps_r,
                    const double* h_history, int weight_kind, const double* h_diag) {
  if (!path) return err(RBD_ERR_INVALID_ARGUMENT, "write_model: null path");
  if (m < 1 || n < 1 || d < 1 || d > n || ldy < m || !Y || !T || !h_history)
    return err(RBD_ERR_DIMENSION_MISMATCH, "write_model: inconsistent model shapes");
  if (weight_kind < 0 || weight_kind > 2)
    return err(RBD_ERR_INVALID_ARGUMENT, "write_model: unknown weight kind");
  if (weight_kind == RBD_WEIGHT_DIAGONAL && !h_diag)
    return err(RBD_ERR_INVALID_ARGUMENT, "write_model: diagonal weight without values");
  cudaStream_t st = ctx ? (cudaStream_t)rbd_ctx_stream(ctx) : (cudaStream_t)0;
  const std::string tmp = std::string(path) + ".tmp";
  unsigned char head[kHeader];
  std::memcpy(head, kMagic, 4);                              // io.cpp:556
  put_u64(head + 4, (uint64_t)m);                            // :557-559
  put_u64(head + 12, (uint64_t)n);
  put_u64(head + 20, (uint64_t)d);
  head[28] = (unsigned char)weight_kind;                     // :560
  double tail1[1] = {eps_r};
  std::vector<Span> spans;
  spans.push_back({const_cast<double*>(Y), m, d, ldy, on_device(Y)});           // :561-562
  spans.push_back({const_cast<double*>(T), d * n, 1, d * n, on_device(T)});     // :563-564
  spans.push_back({tail1, 1, 1, 1, false});                                     // :565
  spans.push_back({const_cast<double*>(h_history), d, 1, d, false});            // :566-567
  if (weight_kind == RBD_WEIGHT_DIAGONAL)
    spans.push_back({const_cast<double*>(h_diag), m, 1, m, on_device(h_diag)});  // :568-569
  {
    File fo;
    fo.f = fopen(tmp.c_str(), "wb");
    if (!fo.f) return err(RBD_ERR_IO, "cannot open " + tmp + " for writing");
    setvbuf(fo.f, nullptr, _IONBF, 0);   // large writes go straight to write(2)
    if (fwrite(head, 1, kHeader, fo.f) != kHeader) return err(RBD_ERR_IO, "write failed: " + tmp);
    const int rc = write_spans(fo.f, tmp.c_str(), spans, st);
    if (rc) {
      fclose(fo.f);
      fo.f = nullptr;
      std::remove(tmp.c_str());
      return rc;
    }
    const int cl = fclose(fo.f);
    fo.f = nullptr;
    if (cl != 0) return err(RBD_ERR_IO, "write failed: " + tmp);
  }
  if (std::rename(tmp.c_str(), path) != 0)                   // write_file_atomic, io.cpp:69-72
    return err(RBD_ERR_IO, std::string("rename to ") + path + " failed: " + std::strerror(errno));
  return RBD_OK;
}

int rbd_model_read_header(const char* path, int64_t* m, int64_t* n, int64_t* d, int* weight_kind) {
  if (!path) return err(RBD_ERR_INVALID_ARGUMENT, "read_model: null path");
  File fi;
  fi.f = fopen(path, "rb");
  if (!fi.f) return err(RBD_ERR_IO, std::string("cannot open ") + path);   // read_file, io.cpp:52
  unsigned char head[kHeader];
  const size_t got = fread(head, 1, kHeader, fi.f);
  if (got < kHeader || std::memcmp(head, kMagic, 4) != 0)                 // io.cpp:580-581
    return parse_err(path, "not a model file (bad magic)");
  uint64_t mm, nn, dd;
  std::memcpy(&mm, head + 4, 8);
  std::memcpy(&nn, head + 12, 8);
  std::memcpy(&dd, head + 20, 8);
  const int64_t M = (int64_t)mm, N = (int64_t)nn, D = (int64_t)dd;
  if (M < 1 || N < 1 || D < 1 || D > N)                                  // :587-588
    return parse_err(path, "implausible model dimensions");
  const int tag = head[28];
  if (tag > 2) return parse_err(path, "unknown weight tag");             // :590
  if (fseeko(fi.f, 0, SEEK_END) != 0) return err(RBD_ERR_IO, std::string("read failed: ") + path);
  const off_t size = ftello(fi.f);
  uint64_t want = 0;
  if (size < 0 || !expected_size(M, N, D, tag, &want) || (uint64_t)size != want)   // :592-596
    return parse_err(path, "model file size does not match header");
  if (m) *m = M;
  if (n) *n = N;
  if (d) *d = D;
  if (weight_kind) *weight_kind = tag;
  return RBD_OK;
}

int rbd_model_read(rbd_ctx_t ctx, const char* path, double* Y, int64_t ldy, double* T,
                   double* eps_r, double* h_history, double* h_diag) {
  int64_t m, n, d;
  int tag;
  const int rc0 = rbd_model_read_header(path, &m, &n, &d, &tag);
  if (rc0) return rc0;
  if (!Y || !T || !h_history || ldy < m)
    return err(RBD_ERR_DIMENSION_MISMATCH, "read_model: output buffers do not match the header");
  if (tag == RBD_WEIGHT_DIAGONAL && !h_diag)
    return err(RBD_ERR_INVALID_ARGUMENT, "read_model: diagonal weight needs an output buffer");
  cudaStream_t st = ctx ? (cudaStream_t)rbd_ctx_stream(ctx) : (cudaStream_t)0;
  File fi;
  fi.f = fopen(path, "rb");
  if (!fi.f) return err(RBD_ERR_IO, std::string("cannot open ") + path);
  setvbuf(fi.f, nullptr, _IONBF, 0);
  if (fseeko(fi.f, (off_t)kHeader, SEEK_SET) != 0)
    return err(RBD_ERR_IO, std::string("read failed: ") + path);
  double e = 0.0;
  std::vector<Span> spans;
  spans.push_back({Y, m, d, ldy, on_device(Y)});                 // io.cpp:601-603
  spans.push_back({T, d * n, 1, d * n, on_device(T)});           // :604-606
  spans.push_back({&e, 1, 1, 1, false});                         // :607
  spans.push_back({h_history, d, 1, d, false});                  // :608-610
  if (tag == RBD_WEIGHT_DIAGONAL) spans.push_back({h_diag, m, 1, m, on_device(h_diag)});   // :617
  const int rc = read_spans(fi.f, path, spans, st);
  if (rc) return rc;
  if (tag == RBD_WEIGHT_DIAGONAL) {   // WeightSpec::diagonal(values), io.cpp:617-618 (weight.cpp:11-17)
    std::vector<double> dh((size_t)m);
    if (on_device(h_diag)) {
      if (cudaMemcpyAsync(dh.data(), h_diag, sizeof(double) * m, cudaMemcpyDeviceToHost, st) ||
          cudaStreamSynchronize(st))
        return err(RBD_ERR_CUDA, "read_model: diagonal D2H failed");
    } else {
      std::memcpy(dh.data(), h_diag, sizeof(double) * m);
    }
    for (double v : dh)
      if (!(v > 0.0) || !std::isfinite(v))
        return err(RBD_ERR_INVALID_ARGUMENT,
                   "diagonal weight entries must be strictly positive and finite");
  }
  if (eps_r) *eps_r = e;
  return RBD_OK;
}
