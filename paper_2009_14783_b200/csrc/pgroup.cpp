// NcclProcessGroup: the reference's ProcessGroup contract
// (include/hetpar/comm.hpp:16-49) over the engine's NCCL communicator, plus
// a TCP rendezvous that ships the ncclUniqueId (the role comm_tcp.cpp:154-237
// plays for the reference's TCP backend), so a world can be formed without
// any Python control plane.  Control-plane only: every call is host-staged
// and blocking, off the training hot path.
//
// Contract details kept from comm.hpp:
// - broadcast: every rank returns the root's exact bytes (length first);
// - all_reduce_sum: the rank-ordered left fold 0 -> world-1, identical bytes
//   on every rank (contributions all-gathered, folded on the host -- an NCCL
//   sum's order is not rank order); a length mismatch is a comm_error;
// - gather_scalars: the master gets [v_0 .. v_{w-1}], others nothing;
// - barrier: no rank returns before all entered.
#include <arpa/inet.h>
#include <netinet/in.h>
#include <netinet/tcp.h>
#include <poll.h>
#include <sys/socket.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "engine.h"
#include "hp_common.h"

namespace hp {
namespace {

// ---- TCP rendezvous: rank 0 listens, every other rank connects and reads
// the 128-byte id; retries until timeout_ms.
void send_all(int fd, const void* p, size_t n) {
  const char* c = static_cast<const char*>(p);
  while (n) {
    const ssize_t k = ::send(fd, c, n, MSG_NOSIGNAL);
    if (k <= 0) fail(HP_ECOMM, "tcp rendezvous: send failed");
    c += k;
    n -= static_cast<size_t>(k);
  }
}
void recv_all(int fd, void* p, size_t n, int timeout_ms) {
  char* c = static_cast<char*>(p);
  while (n) {
    pollfd pf{fd, POLLIN, 0};
    if (::poll(&pf, 1, timeout_ms) <= 0) fail(HP_ECOMM, "tcp rendezvous: receive timed out");
    const ssize_t k = ::recv(fd, c, n, 0);
    if (k <= 0) fail(HP_ECOMM, "tcp rendezvous: peer closed the connection");
    c += k;
    n -= static_cast<size_t>(k);
  }
}

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) ::close(fd);
  }
};

void tcp_share_id(const std::string& host, uint16_t port, int world, int rank, int timeout_ms,
                  uint8_t id[128]) {
  sockaddr_in addr{};
  addr.sin_family = AF_INET;
  addr.sin_port = htons(port);
  if (::inet_pton(AF_INET, host.c_str(), &addr.sin_addr) != 1)
    fail(HP_ECOMM, "tcp rendezvous: bad IPv4 address " + host);
  const auto deadline = std::chrono::steady_clock::now() + std::chrono::milliseconds(timeout_ms);
  const uint32_t magic = 0x48504231;  // "HPB1"
  if (rank == 0) {
    Fd ls;
    ls.fd = ::socket(AF_INET, SOCK_STREAM, 0);
    if (ls.fd < 0) fail(HP_ECOMM, "tcp rendezvous: socket failed");
    int one = 1;
    ::setsockopt(ls.fd, SOL_SOCKET, SO_REUSEADDR, &one, sizeof(one));
    if (::bind(ls.fd, reinterpret_cast<sockaddr*>(&addr), sizeof(addr)) != 0)
      fail(HP_ECOMM, "tcp rendezvous: cannot bind " + host + ":" + std::to_string(port));
    if (::listen(ls.fd, world) != 0) fail(HP_ECOMM, "tcp rendezvous: listen failed");
    for (int joined = 1; joined < world; ++joined) {
      pollfd pf{ls.fd, POLLIN, 0};
      const int left = static_cast<int>(std::chrono::duration_cast<std::chrono::milliseconds>(
                                            deadline - std::chrono::steady_clock::now())
                                            .count());
      if (left <= 0 || ::poll(&pf, 1, left) <= 0)
        fail(HP_ECOMM, "tcp rendezvous: only " + std::to_string(joined) + " of " +
                           std::to_string(world) + " ranks joined before the timeout");
      Fd c;
      c.fd = ::accept(ls.fd, nullptr, nullptr);
      if (c.fd < 0) fail(HP_ECOMM, "tcp rendezvous: accept failed");
      uint32_t hello[3];  // magic, world, rank
      recv_all(c.fd, hello, sizeof(hello), timeout_ms);
      if (hello[0] != magic || static_cast<int>(hello[1]) != world)
        fail(HP_ECOMM, "tcp rendezvous: a peer disagrees on the world size");
      send_all(c.fd, id, 128);
    }
  } else {
    for (;;) {
      Fd c;
      c.fd = ::socket(AF_INET, SOCK_STREAM, 0);
      if (c.fd < 0) fail(HP_ECOMM, "tcp rendezvous: socket failed");
      if (::connect(c.fd, reinterpret_cast<sockaddr*>(&addr), sizeof(addr)) == 0) {
        const uint32_t hello[3] = {magic, static_cast<uint32_t>(world), static_cast<uint32_t>(rank)};
        send_all(c.fd, hello, sizeof(hello));
        recv_all(c.fd, id, 128, timeout_ms);
        return;
      }
      if (std::chrono::steady_clock::now() > deadline)
        fail(HP_ECOMM, "tcp rendezvous: cannot reach rank 0 at " + host + ":" + std::to_string(port));
      std::this_thread::sleep_for(std::chrono::milliseconds(20));
    }
  }
}

// device scratch of the control-plane collectives (owned by the hp_comm)
struct PgScratch {
  cudaStream_t s;
  hp_comm* c;
};
PgScratch scratch(hp_comm* c) {
  HP_CUDA(cudaSetDevice(c->device));
  if (!c->pg_stream) HP_CUDA(cudaStreamCreateWithFlags(&c->pg_stream, cudaStreamNonBlocking));
  return PgScratch{c->pg_stream, c};
}
void* ensure(const PgScratch& p, size_t bytes) {
  if (p.c->pg_cap < bytes) {
    if (p.c->pg_buf) HP_CUDA(cudaFree(p.c->pg_buf));
    p.c->pg_buf = nullptr;
    HP_CUDA(cudaMalloc(&p.c->pg_buf, bytes));
    p.c->pg_cap = bytes;
  }
  return p.c->pg_buf;
}

void check_nccl(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(HP_ECOMM, std::string(what) + ": " + ncclGetErrorString(r));
}

// every rank's `count` doubles, rank-major
std::vector<double> all_gather(hp_comm* c, const double* v, size_t count) {
  const PgScratch p = scratch(c);
  double* d = static_cast<double*>(ensure(p, sizeof(double) * count * (c->world + 1)));
  double* mine = d + count * c->world;
  if (count) HP_CUDA(cudaMemcpyAsync(mine, v, sizeof(double) * count, cudaMemcpyHostToDevice, p.s));
  check_nccl(ncclAllGather(mine, d, count, ncclDouble, c->nccl, p.s), "ncclAllGather");
  std::vector<double> out(count * c->world);
  if (!out.empty())
    HP_CUDA(cudaMemcpyAsync(out.data(), d, sizeof(double) * out.size(), cudaMemcpyDeviceToHost, p.s));
  HP_CUDA(cudaStreamSynchronize(p.s));
  return out;
}

}  // namespace
}  // namespace hp

extern "C" {

hp_status hp_comm_create_tcp(const char* host, uint16_t port, int world, int rank, int device,
                             int timeout_ms, hp_comm** out) {
  HP_API_BEGIN
  if (!host || !out) hp::fail(HP_ECONFIG, "hp_comm_create_tcp: null argument");
  if (world < 1 || rank < 0 || rank >= world)
    hp::fail(HP_ECOMM, "rank " + std::to_string(rank) + " out of range for world_size " +
                           std::to_string(world));
  uint8_t id[128] = {};
  if (rank == 0) {
    const hp_status st = hp_comm_unique_id(id);
    if (st != HP_OK) return st;
  }
  if (world > 1) hp::tcp_share_id(host, port, world, rank, timeout_ms, id);
  return hp_comm_create(world, rank, device, id, out);
  HP_API_END
}

hp_status hp_pg_broadcast(hp_comm* c, const void* payload, uint64_t len, uint64_t root, void* out,
                          uint64_t cap, uint64_t* out_len) {
  HP_API_BEGIN
  if (!c || !out_len) hp::fail(HP_ECONFIG, "hp_pg_broadcast: null argument");
  if (root >= static_cast<uint64_t>(c->world))
    hp::fail(HP_ECOMM, "broadcast root " + std::to_string(root) + " out of range");
  // the root's length and every rank's capacity first (non-root lengths are
  // ignored): a capacity short of the root's length fails on EVERY rank,
  // before any of them enters the broadcast
  const double mine[2] = {c->rank == static_cast<int>(root) ? static_cast<double>(len) : 0.0,
                          static_cast<double>(cap)};
  const std::vector<double> lens = hp::all_gather(c, mine, 2);
  const uint64_t n = static_cast<uint64_t>(lens[2 * root]);
  *out_len = n;
  for (int r = 0; r < c->world; ++r)
    if (static_cast<uint64_t>(lens[2 * r + 1]) < n)
      hp::fail(HP_ECONFIG, "broadcast: rank " + std::to_string(r) + "'s output buffer holds " +
                               std::to_string(static_cast<uint64_t>(lens[2 * r + 1])) +
                               " bytes, the root sent " + std::to_string(n));
  const hp::PgScratch p = hp::scratch(c);
  void* d = hp::ensure(p, n ? n : 1);
  if (c->rank == static_cast<int>(root) && n)
    HP_CUDA(cudaMemcpyAsync(d, payload, n, cudaMemcpyHostToDevice, p.s));
  hp::check_nccl(ncclBroadcast(d, d, n, ncclUint8, static_cast<int>(root), c->nccl, p.s), "ncclBroadcast");
  if (n) HP_CUDA(cudaMemcpyAsync(out, d, n, cudaMemcpyDeviceToHost, p.s));
  HP_CUDA(cudaStreamSynchronize(p.s));
  HP_API_END
}

hp_status hp_pg_all_reduce_sum(hp_comm* c, const double* v, uint64_t n, double* out) {
  HP_API_BEGIN
  if (!c || (n && (!v || !out))) hp::fail(HP_ECONFIG, "hp_pg_all_reduce_sum: null argument");
  const double dn = static_cast<double>(n);
  const std::vector<double> lens = hp::all_gather(c, &dn, 1);
  for (int r = 1; r < c->world; ++r)
    if (lens[r] != lens[0])
      hp::fail(HP_ECOMM, "all_reduce length mismatch: rank " + std::to_string(r) + " sent " +
                             std::to_string(static_cast<uint64_t>(lens[r])) + " values, rank 0 sent " +
                             std::to_string(static_cast<uint64_t>(lens[0])));
  const std::vector<double> all = hp::all_gather(c, v, n);
  // fold_rank_ordered (comm.hpp:55-69)
  for (uint64_t i = 0; i < n; ++i) out[i] = all[i];
  for (int r = 1; r < c->world; ++r)
    for (uint64_t i = 0; i < n; ++i) out[i] += all[static_cast<size_t>(r) * n + i];
  HP_API_END
}

hp_status hp_pg_gather_scalars(hp_comm* c, double v, double* out) {
  HP_API_BEGIN
  if (!c) hp::fail(HP_ECONFIG, "hp_pg_gather_scalars: null argument");
  const std::vector<double> all = hp::all_gather(c, &v, 1);
  if (c->rank == 0) {
    if (!out) hp::fail(HP_ECONFIG, "hp_pg_gather_scalars: the master needs an output buffer");
    std::memcpy(out, all.data(), sizeof(double) * all.size());
  }
  HP_API_END
}

hp_status hp_comm_allreduce_bench(hp_comm* c, uint64_t bytes, double bucket_mb, int iters,
                                  int warmup, double* ms) {
  HP_API_BEGIN
  if (!c || !ms) hp::fail(HP_ECONFIG, "hp_comm_allreduce_bench: null argument");
  if (bytes < 4 || iters < 1 || warmup < 0 || !(bucket_mb > 0))
    hp::fail(HP_ECONFIG, "hp_comm_allreduce_bench: bad sizes");
  HP_CUDA(cudaSetDevice(c->device));
  const size_t n = bytes / 4;
  const size_t cap = std::max<size_t>(1, static_cast<size_t>(bucket_mb * 1048576.0) / 4);
  float* buf = nullptr;
  cudaStream_t s = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  HP_CUDA(cudaMalloc(&buf, n * 4));
  try {
    HP_CUDA(cudaMemsetAsync(buf, 0, n * 4));
    HP_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    HP_CUDA(cudaEventCreate(&e0));
    HP_CUDA(cudaEventCreate(&e1));
    HP_CUDA(cudaDeviceSynchronize());
    // buckets walk the buffer from its end (the engine's order: bucket 0
    // holds the last parameters, the first gradients backward produces)
    auto one = [&]() {
      for (size_t hi = n; hi > 0;) {
        const size_t lo = hi > cap ? hi - cap : 0;
        hp::check_nccl(ncclAllReduce(buf + lo, buf + lo, hi - lo, ncclFloat, ncclSum, c->nccl, s),
                       "ncclAllReduce");
        hi = lo;
      }
    };
    for (int i = 0; i < warmup; ++i) one();
    HP_CUDA(cudaStreamSynchronize(s));
    HP_CUDA(cudaEventRecord(e0, s));
    for (int i = 0; i < iters; ++i) one();
    HP_CUDA(cudaEventRecord(e1, s));
    HP_CUDA(cudaEventSynchronize(e1));
    float t = 0.f;
    HP_CUDA(cudaEventElapsedTime(&t, e0, e1));
    *ms = static_cast<double>(t) / iters;
  } catch (...) {
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (s) cudaStreamDestroy(s);
    cudaFree(buf);
    throw;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaStreamDestroy(s);
  cudaFree(buf);
  HP_API_END
}

hp_status hp_pg_barrier(hp_comm* c) {
  HP_API_BEGIN
  if (!c) hp::fail(HP_ECONFIG, "hp_pg_barrier: null argument");
  const double one = 1.0;
  (void)hp::all_gather(c, &one, 1);
  HP_API_END
}

}  // extern "C"
