// Test shim: a libnccl-compatible P2P library for TWO processes on ONE GPU
// (test infrastructure, not product code).
//
// The round-end GPU boxes have one B200, and real NCCL refuses two ranks on the
// same device, so libzb.so's NCCL transport (csrc/comm.cu: ncclGetUniqueId,
// ncclCommInitRank, ncclSend, ncclRecv, ncclAllReduce, ncclCommDestroy, ncclGetErrorString,
// dlopen'ed; ZB_NCCL_LIB selects this file instead) is exercised across real
// processes through this shim: every 2-rank communicator owns, per receiving
// rank, a device staging ring (NSLOT x CAP bytes) plus two 32-bit counters
// (produced, consumed), shared with the peer through CUDA IPC.  Send / recv are
// fully stream-ordered and never block the host, like NCCL's:
//   send chunk k:  wait(consumed >= k+1-NSLOT); memcpy -> peer slot k % NSLOT;
//                  write(produced = k+1)
//   recv chunk k:  wait(produced >= k+1); memcpy slot -> user buffer;
//                  write(consumed = k+1)
// with cuStreamWaitValue32 / cuStreamWriteValue32 (front-end semaphore waits: a
// blocked stream does not occupy SMs, so the two processes' contexts keep
// time-slicing the GPU).  Messages on a communicator match in order; a message
// larger than CAP is cut into chunks identically on both sides.
// The rendezvous is a pair of files /dev/shm/zbnccl_<id>_<rank> carrying the
// cudaIpcMemHandle of each rank's receive region.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <thread>

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

extern "C" {
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
}

namespace {
constexpr int NSLOT = 2;
constexpr ncclResult_t kOk = 0, kUnhandled = 1, kSystem = 2, kInternal = 3, kInvalid = 4;

size_t cap_bytes() {
  static const size_t c = [] {
    const char* e = std::getenv("ZB_SHIM_CAP_MB");
    const long v = e ? std::atol(e) : 0;
    return static_cast<size_t>(v > 0 ? v : 64) << 20;
  }();
  return c;
}

struct Comm {
  int rank = 0;
  std::string files[2];
  char* in_base = nullptr;   // my receive region: NSLOT * CAP staging + counters
  char* out_base = nullptr;  // the peer's receive region (IPC-mapped)
  uint32_t send_seq = 0, recv_seq = 0;
  size_t cap = 0;
  uint32_t* ctr(char* base) const { return reinterpret_cast<uint32_t*>(base + NSLOT * cap); }
};

thread_local std::string g_err;

ncclResult_t fail(ncclResult_t r, const std::string& m) {
  g_err = m;
  std::fprintf(stderr, "zbnccl shim: %s\n", m.c_str());
  return r;
}

bool cu_ok(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return true;
  const char* s = nullptr;
  cuGetErrorString(r, &s);
  fail(kSystem, std::string(what) + ": " + (s ? s : "?"));
  return false;
}

size_t dtype_size(int dt) {
  switch (dt) {
    case 0: case 1: return 1;                    // int8, uint8
    case 2: case 3: case 7: return 4;            // int32, uint32, float32
    case 4: case 5: case 8: return 8;            // int64, uint64, float64
    case 6: case 9: return 2;                    // float16, bfloat16
    default: return 0;
  }
}
}  // namespace

extern "C" {

const char* ncclGetErrorString(ncclResult_t r) {
  static thread_local std::string s;
  s = "shim error " + std::to_string(r) + (g_err.empty() ? "" : (": " + g_err));
  return s.c_str();
}

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
  std::memset(id, 0, sizeof(*id));
  std::random_device rd;
  const uint64_t a = (static_cast<uint64_t>(rd()) << 32) ^ rd() ^ static_cast<uint64_t>(getpid());
  std::snprintf(id->internal, sizeof(id->internal), "zbshim%016llx", static_cast<unsigned long long>(a));
  return kOk;
}

ncclResult_t ncclCommInitRank(void** comm, int nranks, ncclUniqueId id, int rank) {
  if (nranks != 2 || rank < 0 || rank > 1) return fail(kInvalid, "the shim supports 2-rank communicators only");
  auto* c = new Comm();
  c->rank = rank;
  c->cap = cap_bytes();
  const std::string key(id.internal, strnlen(id.internal, sizeof(id.internal)));
  for (int r = 0; r < 2; ++r) c->files[r] = "/dev/shm/zbnccl_" + key + "_" + std::to_string(r);
  void* base = nullptr;
  if (cudaMalloc(&base, NSLOT * c->cap + 256) != cudaSuccess) return fail(kSystem, "cudaMalloc of the staging ring");
  c->in_base = static_cast<char*>(base);
  if (cudaMemset(c->ctr(c->in_base), 0, 256) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess)
    return fail(kSystem, "counter init");
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, base) != cudaSuccess) return fail(kSystem, "cudaIpcGetMemHandle");
  {  // publish atomically (write then rename)
    const std::string tmp = c->files[rank] + ".tmp";
    FILE* f = std::fopen(tmp.c_str(), "wb");
    if (!f || std::fwrite(&h, sizeof(h), 1, f) != 1) return fail(kSystem, "cannot write " + tmp);
    std::fclose(f);
    if (std::rename(tmp.c_str(), c->files[rank].c_str()) != 0) return fail(kSystem, "rename " + tmp);
  }
  const std::string& peer = c->files[1 - rank];
  const auto t0 = std::chrono::steady_clock::now();
  cudaIpcMemHandle_t ph;
  for (;;) {
    FILE* f = std::fopen(peer.c_str(), "rb");
    if (f) {
      const size_t n = std::fread(&ph, sizeof(ph), 1, f);
      std::fclose(f);
      if (n == 1) break;
    }
    if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(300))
      return fail(kSystem, "peer never published " + peer);
    std::this_thread::sleep_for(std::chrono::milliseconds(2));
  }
  void* pb = nullptr;
  if (cudaIpcOpenMemHandle(&pb, ph, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
    return fail(kSystem, "cudaIpcOpenMemHandle");
  c->out_base = static_cast<char*>(pb);
  *comm = c;
  return kOk;
}

ncclResult_t ncclCommDestroy(void* comm) {
  auto* c = static_cast<Comm*>(comm);
  if (!c) return kOk;
  cudaDeviceSynchronize();
  if (c->out_base) cudaIpcCloseMemHandle(c->out_base);
  if (c->in_base) cudaFree(c->in_base);
  std::remove(c->files[c->rank].c_str());
  delete c;
  return kOk;
}

ncclResult_t ncclSend(const void* buf, size_t count, int dtype, int peer, void* comm, cudaStream_t st) {
  auto* c = static_cast<Comm*>(comm);
  const size_t es = dtype_size(dtype);
  if (!c || !es || peer != 1 - c->rank) return fail(kInvalid, "ncclSend: bad arguments");
  const size_t bytes = count * es;
  uint32_t* ctr = c->ctr(c->out_base);  // [0] produced (written here), [1] consumed (by the peer)
  for (size_t off = 0; off < bytes || (bytes == 0 && off == 0); off += c->cap) {
    const uint32_t k = c->send_seq++;
    const size_t n = bytes - off < c->cap ? bytes - off : c->cap;
    if (k + 1 > static_cast<uint32_t>(NSLOT) &&
        !cu_ok(cuStreamWaitValue32(st, reinterpret_cast<CUdeviceptr>(ctr + 1), k + 1 - NSLOT,
                                   CU_STREAM_WAIT_VALUE_GEQ), "cuStreamWaitValue32"))
      return kSystem;
    if (n && cudaMemcpyAsync(c->out_base + (k % NSLOT) * c->cap, static_cast<const char*>(buf) + off, n,
                             cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return fail(kSystem, "ncclSend: copy");
    if (!cu_ok(cuStreamWriteValue32(st, reinterpret_cast<CUdeviceptr>(ctr + 0), k + 1,
                                    CU_STREAM_WRITE_VALUE_DEFAULT), "cuStreamWriteValue32"))
      return kSystem;
    if (bytes == 0) break;
  }
  return kOk;
}

ncclResult_t ncclRecv(void* buf, size_t count, int dtype, int peer, void* comm, cudaStream_t st) {
  auto* c = static_cast<Comm*>(comm);
  const size_t es = dtype_size(dtype);
  if (!c || !es || peer != 1 - c->rank) return fail(kInvalid, "ncclRecv: bad arguments");
  const size_t bytes = count * es;
  uint32_t* ctr = c->ctr(c->in_base);
  for (size_t off = 0; off < bytes || (bytes == 0 && off == 0); off += c->cap) {
    const uint32_t k = c->recv_seq++;
    const size_t n = bytes - off < c->cap ? bytes - off : c->cap;
    if (!cu_ok(cuStreamWaitValue32(st, reinterpret_cast<CUdeviceptr>(ctr + 0), k + 1, CU_STREAM_WAIT_VALUE_GEQ),
               "cuStreamWaitValue32"))
      return kSystem;
    if (n && cudaMemcpyAsync(static_cast<char*>(buf) + off, c->in_base + (k % NSLOT) * c->cap, n,
                             cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return fail(kSystem, "ncclRecv: copy");
    if (!cu_ok(cuStreamWriteValue32(st, reinterpret_cast<CUdeviceptr>(ctr + 1), k + 1,
                                    CU_STREAM_WRITE_VALUE_DEFAULT), "cuStreamWriteValue32"))
      return kSystem;
    if (bytes == 0) break;
  }
  return kOk;
}

}  // extern "C"

// ncclAllReduce (sum, 2 ranks): per chunk, my data goes to the peer's staging slot (as a send)
// and the peer's chunk, once produced, is added into my buffer straight from my staging slot.
// Rank 0 computes a + b, rank 1 b + a: IEEE addition is commutative, so both ranks hold the
// same bits.  In place is allowed (the chunk is sent before it is overwritten, stream order).
namespace {
template <typename T>
__global__ void k_add(T* out, const T* a, const T* b, size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    out[i] = a[i] + b[i];
}
}  // namespace

extern "C" ncclResult_t ncclAllReduce(const void* sendbuf, void* recvbuf, size_t count, int dtype, int op, void* comm,
                                      cudaStream_t st) {
  auto* c = static_cast<Comm*>(comm);
  if (!c || op != 0 || (dtype != 7 && dtype != 8)) return fail(kInvalid, "ncclAllReduce: only f32 / f64 sum");
  const size_t es = dtype_size(dtype);
  const size_t bytes = count * es;
  uint32_t* out_ctr = c->ctr(c->out_base);
  uint32_t* in_ctr = c->ctr(c->in_base);
  for (size_t off = 0; off < bytes || (bytes == 0 && off == 0); off += c->cap) {
    const size_t n = bytes - off < c->cap ? bytes - off : c->cap;
    const uint32_t k = c->send_seq++;
    if (k + 1 > static_cast<uint32_t>(NSLOT) &&
        !cu_ok(cuStreamWaitValue32(st, reinterpret_cast<CUdeviceptr>(out_ctr + 1), k + 1 - NSLOT,
                                   CU_STREAM_WAIT_VALUE_GEQ), "cuStreamWaitValue32"))
      return kSystem;
    if (n && cudaMemcpyAsync(c->out_base + (k % NSLOT) * c->cap, static_cast<const char*>(sendbuf) + off, n,
                             cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return fail(kSystem, "ncclAllReduce: copy");
    if (!cu_ok(cuStreamWriteValue32(st, reinterpret_cast<CUdeviceptr>(out_ctr + 0), k + 1,
                                    CU_STREAM_WRITE_VALUE_DEFAULT), "cuStreamWriteValue32"))
      return kSystem;
    const uint32_t r = c->recv_seq++;
    if (!cu_ok(cuStreamWaitValue32(st, reinterpret_cast<CUdeviceptr>(in_ctr + 0), r + 1, CU_STREAM_WAIT_VALUE_GEQ),
               "cuStreamWaitValue32"))
      return kSystem;
    if (n) {
      const size_t ne = n / es;
      const int grid = static_cast<int>(std::min<size_t>((ne + 255) / 256, 1184));
      const char* a = static_cast<const char*>(sendbuf) + off;
      const char* b = c->in_base + (r % NSLOT) * c->cap;
      char* o = static_cast<char*>(recvbuf) + off;
      if (dtype == 7)
        k_add<float><<<grid, 256, 0, st>>>(reinterpret_cast<float*>(o), reinterpret_cast<const float*>(a),
                                           reinterpret_cast<const float*>(b), ne);
      else
        k_add<double><<<grid, 256, 0, st>>>(reinterpret_cast<double*>(o), reinterpret_cast<const double*>(a),
                                            reinterpret_cast<const double*>(b), ne);
      if (cudaGetLastError() != cudaSuccess) return fail(kSystem, "ncclAllReduce: add kernel");
    }
    if (!cu_ok(cuStreamWriteValue32(st, reinterpret_cast<CUdeviceptr>(in_ctr + 1), r + 1,
                                    CU_STREAM_WRITE_VALUE_DEFAULT), "cuStreamWriteValue32"))
      return kSystem;
    if (bytes == 0) break;
  }
  return kOk;
}
