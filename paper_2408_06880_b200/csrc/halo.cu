// Halo exchange between block engines (exchange.py:125-374).
//
// The Python host derives every edge's message layout exactly as
// EdgePlan._build does (exchange.py:148-219) and registers, per phase:
//   local edge   both engines in this process: one fused gather-scatter
//                dst.pdf[tgt[k]] = src.pdf[send[take[k]]]; all local edges of
//                a phase run as ONE kernel (no intermediate buffer);
//   remote send  entries gathered into the per-peer section of one send
//                buffer (one pack kernel for all peers);
//   remote recv  the peer's message lands in its section of one receive
//                buffer; stored entries are scattered by one unpack kernel.
// Messages travel as one ncclSend/ncclRecv pair per peer per phase inside
// an NCCL group, on the halo's own comm stream, so the interior sweep on the
// compute stream overlaps pack -> NVLink -> unpack (the interior
// sweep touches none of the exchanged slots).
//
// Peer transport (slbm_halo_use_peer + slbm_halo_connect): no NCCL.  Every
// rank maps its peers' receive buffers and flag words through CUDA IPC; the
// pack kernel gathers from the local PDFs and stores each message straight
// into the peer's receive buffer over NVLink (gather and transfer are one
// kernel), then a release store of the step's epoch into the peer's flag
// tells it the message is complete.  The receiver's unpack waits (acquire
// spin) on that flag and acknowledges into the sender's ack word, which the
// sender waits on before overwriting the buffer one exchange later:
//   comm stream:  wait acks(e-1) -> remote pack -> signal(e) -> local edges
//                 -> wait data(e) -> unpack -> ack(e) -> e += 1
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <vector>

#include "engine.cuh"

namespace slbm {
namespace {

constexpr int kMaxEngines = kMaxHaloEngines;

__global__ void k_local(PdfTable t, const uint16_t* se, const uint32_t* ss, const uint16_t* de,
                        const uint32_t* ds, int64_t n) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) t.p[de[i]][ds[i]] = t.p[se[i]][ss[i]];
}

__global__ void k_pack(PdfTable t, const uint16_t* e, const uint32_t* s, int64_t n,
                       double* buf) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) buf[i] = t.p[e[i]][s[i]];
}

__global__ void k_unpack(PdfTable t, const uint64_t* pos, const uint16_t* e, const uint32_t* s,
                         int64_t n, const double* buf) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) t.p[e[i]][s[i]] = buf[pos[i]];
}

// ---- peer transport: epoch flags with system-scope release / acquire ----
constexpr int kMaxPeers = 64;

struct FlagPtrs {
  uint64_t* p[kMaxPeers];
  int n;
};

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// a peer that never arrives is a fatal error (trap after 120 s), not a hang
__device__ __forceinline__ void spin_until(const uint64_t* flag, uint64_t want) {
  const uint64_t t0 = globaltimer();
  while (ld_acquire_sys(flag) < want) {
    __nanosleep(100);
    if (globaltimer() - t0 > 120ull * 1000000000ull) __trap();
  }
}

__global__ void k_epoch_advance(uint64_t* epoch) { *epoch += 1; }

// Peer unpack: every CTA waits (one thread) for all senders' epoch flags,
// scatters its entries; the CTA that finishes last acknowledges to every
// sender (they may overwrite this buffer again) and advances the epoch.
__global__ void k_unpack_ack(PdfTable t, const uint64_t* pos, const uint16_t* e,
                             const uint32_t* s, int64_t n, const double* buf, FlagPtrs data,
                             FlagPtrs acks, unsigned int* done, uint64_t* epoch) {
  const uint64_t ep = *epoch;
  if (threadIdx.x == 0)
    for (int k = 0; k < data.n; ++k) spin_until(data.p[k], ep);
  __syncthreads();
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) t.p[e[i]][s[i]] = buf[pos[i]];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int prev = atomicAdd(done, 1u);
    if (prev == gridDim.x - 1) {
      __threadfence_system();
      for (int k = 0; k < acks.n; ++k) st_release_sys(acks.p[k], ep);
      *done = 0;
      *epoch = ep + 1;
    }
  }
}

// Peer pack: gather this rank's entries for one peer and store them straight
// into the peer's receive buffer over NVLink; the CTA that finishes last
// publishes the epoch in the peer's flag word.  Every CTA fences its remote
// stores at system scope before it counts itself done, so the release store
// of the last one orders all of them (the "last block" pattern; no reliance
// on kernel-boundary visibility of peer writes).
// Every CTA first waits (one thread) until the peer acknowledged the
// previous exchange through this buffer (`ack` >= epoch - 1).
__global__ void k_pack_signal(PdfTable t, const uint16_t* e, const uint32_t* s, int64_t n,
                              double* remote, unsigned int* done, uint64_t* remote_flag,
                              const uint64_t* ack, const uint64_t* epoch) {
  if (threadIdx.x == 0) spin_until(ack, *epoch - 1);
  __syncthreads();
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) remote[i] = t.p[e[i]][s[i]];
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int prev = atomicAdd(done, 1u);
    if (prev == gridDim.x - 1) {
      __threadfence_system();
      st_release_sys(remote_flag, *epoch);
      *done = 0;  // every CTA has counted: reset for the next exchange
    }
  }
}

inline unsigned grid_for(int64_t n) { return unsigned(std::max<int64_t>((n + 255) / 256, 1)); }

template <class T>
int upload(const std::vector<T>& h, T** d) {
  if (h.empty()) return SLBM_OK;
  SLBM_CUDA_TRY(cudaMalloc(d, h.size() * sizeof(T)));
  SLBM_CUDA_TRY(cudaMemcpy(*d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  return SLBM_OK;
}

struct PeerRecv {
  int64_t n_wire = 0;
  std::vector<uint64_t> pos;  // position within this peer's message
  std::vector<uint16_t> eng;
  std::vector<uint32_t> slot;
};

struct PeerSend {
  std::vector<uint16_t> eng;
  std::vector<uint32_t> slot;
};

struct PhaseProg {
  std::vector<uint16_t> l_se, l_de;
  std::vector<uint32_t> l_ss, l_ds;
  std::map<int, PeerSend> sends;
  std::map<int, PeerRecv> recvs;
  // committed
  uint16_t *d_lse = nullptr, *d_lde = nullptr, *d_pe = nullptr, *d_ue = nullptr;
  uint32_t *d_lss = nullptr, *d_lds = nullptr, *d_ps = nullptr, *d_us = nullptr;
  uint64_t* d_upos = nullptr;
  int64_t n_local = 0, n_pack = 0, n_unpack = 0;
  std::vector<int> send_peer, recv_peer;
  std::vector<int64_t> send_off, send_cnt, recv_off, recv_cnt;
  int64_t send_total = 0, recv_total = 0;
  // unpack entries per peer (for the host-staged path)
  std::vector<int64_t> unpack_off, unpack_cnt;
  // peer transport: where each send section lands in its peer's receive buffer
  std::vector<double*> remote_dst;
};

}  // namespace
}  // namespace slbm

using namespace slbm;

struct SlbmHalo {
  int device = 0;
  cudaStream_t comm = nullptr;
  cudaEvent_t ev_ready = nullptr, ev_done = nullptr;
  std::vector<SlbmEngine*> engines;
  PhaseProg ph[2];
  double* d_send = nullptr;
  double* d_recv = nullptr;
  ncclComm_t nccl = nullptr;
  bool committed = false;
  // peer transport
  bool peer = false;
  int rank = 0;
  uint64_t* d_flags = nullptr;  // [0, kMaxPeers): data epoch per sender; [kMaxPeers, 2k): ack per receiver
  uint64_t* d_epoch = nullptr;
  unsigned int* d_done = nullptr;       // per send slot: CTAs finished in k_pack_signal
  std::map<int, double*> peer_recv;    // peer -> its receive buffer (mapped)
  std::map<int, uint64_t*> peer_flags; // peer -> its flag words (mapped)
  std::vector<void*> opened;           // IPC mappings to close

  int engine_id(SlbmEngine* e, uint16_t* id) {
    auto it = std::find(engines.begin(), engines.end(), e);
    if (it != engines.end()) {
      *id = uint16_t(it - engines.begin());
      return SLBM_OK;
    }
    if (int(engines.size()) >= kMaxEngines)
      return fail(SLBM_ECONFIG, "too many engines in one halo");
    engines.push_back(e);
    *id = uint16_t(engines.size() - 1);
    return SLBM_OK;
  }
  PdfTable table() const {
    PdfTable t{};
    for (size_t i = 0; i < engines.size(); ++i) t.p[i] = engines[i]->pdf;
    return t;
  }
};

namespace {

int check_slots(const SlbmEngine* e, const int64_t* s, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (s[i] < 0 || s[i] >= e->total_slots)
      return fail(SLBM_EPROTOCOL, "halo slot outside the engine's slot range");
  return SLBM_OK;
}

int check_phase(const SlbmHalo* h, int phase) {
  if (!h) return fail(SLBM_ECONFIG, "null halo");
  if (phase != 0 && phase != 1) return fail(SLBM_ECONFIG, "bad exchange phase");
  return SLBM_OK;
}

#define NCCL_TRY(expr)                                                                  \
  do {                                                                                  \
    ncclResult_t _r = (expr);                                                           \
    if (_r != ncclSuccess)                                                              \
      return fail(SLBM_ECUDA, std::string("NCCL error: ") + ncclGetErrorString(_r) +   \
                                  " at " #expr);                                        \
  } while (0)

}  // namespace

namespace {

FlagPtrs flag_ptrs(SlbmHalo* h, const std::vector<int>& peers, bool remote, int base) {
  FlagPtrs f{};
  f.n = int(peers.size());
  for (size_t i = 0; i < peers.size(); ++i) {
    // remote: the peer's word for this rank; local: this rank's word for the peer
    f.p[i] = remote ? h->peer_flags[peers[i]] + base + h->rank : h->d_flags + base + peers[i];
  }
  return f;
}

int nccl_start(SlbmHalo* h, PhaseProg& p, int phase, const PdfTable& t);

int peer_start(SlbmHalo* h, PhaseProg& p, int phase) {
  const PdfTable t = h->table();
  cudaStream_t s = h->comm;
  if (!p.send_peer.empty()) {
    const FlagPtrs data = flag_ptrs(h, p.send_peer, true, 0);      // peers' words for us
    const FlagPtrs acks = flag_ptrs(h, p.send_peer, false, kMaxPeers);  // their acks to us
    for (size_t i = 0; i < p.send_peer.size(); ++i) {
      if (!p.remote_dst[i]) return fail(SLBM_ECONFIG, "peer transport: halo not connected");
      { k_pack_signal<<<grid_for(p.send_cnt[i]), 256, 0, s>>>(
          t, p.d_pe + p.send_off[i], p.d_ps + p.send_off[i], p.send_cnt[i], p.remote_dst[i],
          h->d_done + phase * kMaxPeers + i, data.p[i], acks.p[i], h->d_epoch); slbm::count_launch(); }
    }
    SLBM_CUDA_TRY(cudaGetLastError());
  }
  SLBM_TRY(slbm_halo_local(h, phase));
  if (!p.recv_peer.empty()) {
    { k_unpack_ack<<<grid_for(p.n_unpack), 256, 0, s>>>(
        t, p.d_upos, p.d_ue, p.d_us, p.n_unpack, h->d_recv, flag_ptrs(h, p.recv_peer, false, 0),
        flag_ptrs(h, p.recv_peer, true, kMaxPeers), h->d_done + 2 * kMaxPeers + phase,
        h->d_epoch); slbm::count_launch(); }
  } else {
    { k_epoch_advance<<<1, 1, 0, s>>>(h->d_epoch); slbm::count_launch(); }
  }
  SLBM_CUDA_TRY(cudaGetLastError());
  SLBM_CUDA_TRY(cudaEventRecord(h->ev_done, s));
  return SLBM_OK;
}

}  // namespace

extern "C" {

int slbm_halo_create(int device, SlbmHalo** out) {
  if (!out) return fail(SLBM_ECONFIG, "null out");
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  SlbmHalo* h = new SlbmHalo();
  h->device = device;
  cudaError_t e1 = cudaStreamCreateWithFlags(&h->comm, cudaStreamNonBlocking);
  cudaError_t e2 = cudaEventCreateWithFlags(&h->ev_ready, cudaEventDisableTiming);
  cudaError_t e3 = cudaEventCreateWithFlags(&h->ev_done, cudaEventDisableTiming);
  cudaSetDevice(prev);
  if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess) {
    delete h;
    return fail(SLBM_ECUDA, "halo stream/event creation failed");
  }
  *out = h;
  return SLBM_OK;
}

int slbm_halo_destroy(SlbmHalo* h) {
  if (!h) return SLBM_OK;
  cudaSetDevice(h->device);
  cudaStreamSynchronize(h->comm);
  for (auto& p : h->ph) {
    void* ptrs[] = {p.d_lse, p.d_lde, p.d_pe, p.d_ue, p.d_lss, p.d_lds, p.d_ps, p.d_us, p.d_upos};
    for (void* x : ptrs)
      if (x) cudaFree(x);
  }
  if (h->d_send) cudaFree(h->d_send);
  if (h->d_recv) cudaFree(h->d_recv);
  for (void* m : h->opened) cudaIpcCloseMemHandle(m);
  if (h->d_flags) cudaFree(h->d_flags);
  if (h->d_epoch) cudaFree(h->d_epoch);
  if (h->d_done) cudaFree(h->d_done);
  cudaEventDestroy(h->ev_ready);
  cudaEventDestroy(h->ev_done);
  cudaStreamDestroy(h->comm);
  delete h;
  return SLBM_OK;
}

int slbm_halo_add_local(SlbmHalo* h, int phase, SlbmEngine* src, SlbmEngine* dst,
                        const int64_t* send, int64_t n_send, const int64_t* take,
                        const int64_t* tgt, int64_t n_tgt) {
  SLBM_TRY(check_phase(h, phase));
  if (h->committed) return fail(SLBM_ECONFIG, "halo already committed");
  if (!src || !dst) return fail(SLBM_ECONFIG, "null engine");
  SLBM_TRY(check_slots(src, send, n_send));
  SLBM_TRY(check_slots(dst, tgt, n_tgt));
  uint16_t si, di;
  SLBM_TRY(h->engine_id(src, &si));
  SLBM_TRY(h->engine_id(dst, &di));
  PhaseProg& p = h->ph[phase];
  for (int64_t k = 0; k < n_tgt; ++k) {
    if (take[k] < 0 || take[k] >= n_send)
      return fail(SLBM_EPROTOCOL, "take index outside the message");
    p.l_se.push_back(si);
    p.l_ss.push_back(uint32_t(src->phys_slot(send[take[k]])));
    p.l_de.push_back(di);
    p.l_ds.push_back(uint32_t(dst->phys_slot(tgt[k])));
  }
  return SLBM_OK;
}

int slbm_halo_add_send(SlbmHalo* h, int phase, SlbmEngine* src, int peer, const int64_t* send,
                       int64_t n) {
  SLBM_TRY(check_phase(h, phase));
  if (h->committed) return fail(SLBM_ECONFIG, "halo already committed");
  SLBM_TRY(check_slots(src, send, n));
  uint16_t si;
  SLBM_TRY(h->engine_id(src, &si));
  PeerSend& ps = h->ph[phase].sends[peer];
  for (int64_t k = 0; k < n; ++k) {
    ps.eng.push_back(si);
    ps.slot.push_back(uint32_t(src->phys_slot(send[k])));
  }
  return SLBM_OK;
}

int slbm_halo_add_recv(SlbmHalo* h, int phase, SlbmEngine* dst, int peer, int64_t n_wire,
                       const int64_t* take, const int64_t* tgt, int64_t n_tgt) {
  SLBM_TRY(check_phase(h, phase));
  if (h->committed) return fail(SLBM_ECONFIG, "halo already committed");
  SLBM_TRY(check_slots(dst, tgt, n_tgt));
  uint16_t di;
  SLBM_TRY(h->engine_id(dst, &di));
  PeerRecv& pr = h->ph[phase].recvs[peer];
  for (int64_t k = 0; k < n_tgt; ++k) {
    if (take[k] < 0 || take[k] >= n_wire)
      return fail(SLBM_EPROTOCOL, "take index outside the message");
    pr.pos.push_back(uint64_t(pr.n_wire + take[k]));
    pr.eng.push_back(di);
    pr.slot.push_back(uint32_t(dst->phys_slot(tgt[k])));
  }
  pr.n_wire += n_wire;
  return SLBM_OK;
}

int slbm_halo_commit(SlbmHalo* h, void* nccl_comm) {
  if (!h) return fail(SLBM_ECONFIG, "null halo");
  if (h->committed) return SLBM_OK;
  cudaSetDevice(h->device);
  h->nccl = (ncclComm_t)nccl_comm;
  int64_t max_send = 0, max_recv = 0;
  for (auto& p : h->ph) {
    {
      // local entries in (destination engine, destination slot) order: each
      // entry writes a distinct slot, so the order is free, and sorted the
      // warp's writes are consecutive slots of one direction group and its
      // reads (the same face cells upwind) follow them -- coalesced on both
      // sides instead of cell-major x direction (C4: ~1.4 M entries a step)
      const size_t n = p.l_se.size();
      std::vector<size_t> ord(n);
      for (size_t k = 0; k < n; ++k) ord[k] = k;
      std::sort(ord.begin(), ord.end(), [&](size_t a, size_t b) {
        return p.l_de[a] != p.l_de[b] ? p.l_de[a] < p.l_de[b] : p.l_ds[a] < p.l_ds[b];
      });
      auto perm = [&](auto& v) {
        auto w = v;
        for (size_t k = 0; k < n; ++k) w[k] = v[ord[k]];
        v.swap(w);
      };
      perm(p.l_se);
      perm(p.l_ss);
      perm(p.l_de);
      perm(p.l_ds);
    }
    SLBM_TRY(upload(p.l_se, &p.d_lse));
    SLBM_TRY(upload(p.l_ss, &p.d_lss));
    SLBM_TRY(upload(p.l_de, &p.d_lde));
    SLBM_TRY(upload(p.l_ds, &p.d_lds));
    p.n_local = int64_t(p.l_se.size());
    std::vector<uint16_t> pe, ue;
    std::vector<uint32_t> ps, us;
    std::vector<uint64_t> upos;
    for (auto& kv : p.sends) {
      p.send_peer.push_back(kv.first);
      p.send_off.push_back(int64_t(pe.size()));
      p.send_cnt.push_back(int64_t(kv.second.eng.size()));
      pe.insert(pe.end(), kv.second.eng.begin(), kv.second.eng.end());
      ps.insert(ps.end(), kv.second.slot.begin(), kv.second.slot.end());
    }
    int64_t roff = 0;
    for (auto& kv : p.recvs) {
      p.recv_peer.push_back(kv.first);
      p.recv_off.push_back(roff);
      p.recv_cnt.push_back(kv.second.n_wire);
      p.unpack_off.push_back(int64_t(ue.size()));
      p.unpack_cnt.push_back(int64_t(kv.second.eng.size()));
      for (size_t k = 0; k < kv.second.eng.size(); ++k) {
        upos.push_back(uint64_t(roff) + kv.second.pos[k]);
        ue.push_back(kv.second.eng[k]);
        us.push_back(kv.second.slot[k]);
      }
      roff += kv.second.n_wire;
    }
    if ((!p.sends.empty() || !p.recvs.empty()) && !h->nccl) {
      // allowed: host-staged transport (slbm_halo_pack_host / unpack_host)
    }
    p.send_total = int64_t(pe.size());
    p.recv_total = roff;
    p.n_pack = int64_t(pe.size());
    p.n_unpack = int64_t(ue.size());
    SLBM_TRY(upload(pe, &p.d_pe));
    SLBM_TRY(upload(ps, &p.d_ps));
    SLBM_TRY(upload(ue, &p.d_ue));
    SLBM_TRY(upload(us, &p.d_us));
    SLBM_TRY(upload(upos, &p.d_upos));
    max_send = std::max(max_send, p.send_total);
    max_recv = std::max(max_recv, p.recv_total);
  }
  if (max_send && !h->peer) SLBM_CUDA_TRY(cudaMalloc(&h->d_send, max_send * sizeof(double)));
  if (max_recv || h->peer)
    SLBM_CUDA_TRY(cudaMalloc(&h->d_recv, std::max<int64_t>(max_recv, 1) * sizeof(double)));
  if (h->peer) {
    SLBM_CUDA_TRY(cudaMalloc(&h->d_flags, 2 * kMaxPeers * sizeof(uint64_t)));
    SLBM_CUDA_TRY(cudaMemset(h->d_flags, 0, 2 * kMaxPeers * sizeof(uint64_t)));
    SLBM_CUDA_TRY(cudaMalloc(&h->d_epoch, sizeof(uint64_t)));
    SLBM_CUDA_TRY(cudaMalloc(&h->d_done, (2 * kMaxPeers + 2) * sizeof(unsigned int)));
    SLBM_CUDA_TRY(cudaMemset(h->d_done, 0, (2 * kMaxPeers + 2) * sizeof(unsigned int)));
    const uint64_t one = 1;
    SLBM_CUDA_TRY(cudaMemcpy(h->d_epoch, &one, sizeof(one), cudaMemcpyHostToDevice));
    for (auto& p : h->ph) p.remote_dst.assign(p.send_peer.size(), nullptr);
  }
  h->committed = true;
  return SLBM_OK;
}

}  // extern "C"

namespace slbm {
int halo_local_program(SlbmHalo* h, int phase, std::vector<SlbmEngine*>* engines,
                       std::vector<uint16_t>* se, std::vector<uint32_t>* ss,
                       std::vector<uint16_t>* de, std::vector<uint32_t>* ds) {
  if (!h || (phase != 0 && phase != 1)) return fail(SLBM_ECONFIG, "bad halo or phase");
  if (!h->committed) return fail(SLBM_ECONFIG, "halo not committed");
  const PhaseProg& p = h->ph[phase];
  *engines = h->engines;
  *se = p.l_se;
  *ss = p.l_ss;
  *de = p.l_de;
  *ds = p.l_ds;
  return SLBM_OK;
}

void halo_disable_local(SlbmHalo* h) {
  for (auto& p : h->ph) p.n_local = 0;
}

int halo_local_edges(SlbmHalo* h, int phase, PdfTable* table, LocalEdges* edges) {
  if (!h || (phase != 0 && phase != 1)) return fail(SLBM_ECONFIG, "bad halo or phase");
  *table = h->table();
  *edges = LocalEdges{};
  if (!h->committed) return SLBM_OK;  // no edges registered yet
  const PhaseProg& p = h->ph[phase];
  edges->se = p.d_lse;
  edges->ss = p.d_lss;
  edges->de = p.d_lde;
  edges->ds = p.d_lds;
  edges->n = p.n_local;
  edges->n_eng = int(h->engines.size());
  return SLBM_OK;
}
}  // namespace slbm

extern "C" {

int slbm_halo_local(SlbmHalo* h, int phase) {
  SLBM_TRY(check_phase(h, phase));
  if (!h->committed) return fail(SLBM_ECONFIG, "halo not committed");
  PhaseProg& p = h->ph[phase];
  if (p.n_local) {
    { k_local<<<grid_for(p.n_local), 256, 0, h->comm>>>(h->table(), p.d_lse, p.d_lss, p.d_lde,
                                                       p.d_lds, p.n_local); slbm::count_launch(); }
    SLBM_CUDA_TRY(cudaGetLastError());
  }
  SLBM_CUDA_TRY(cudaEventRecord(h->ev_done, h->comm));
  return SLBM_OK;
}

int slbm_halo_local_on(SlbmHalo* h, int phase, void* stream) {
  SLBM_TRY(check_phase(h, phase));
  if (!h->committed) return fail(SLBM_ECONFIG, "halo not committed");
  cudaSetDevice(h->device);
  PhaseProg& p = h->ph[phase];
  if (p.n_local) {
    { k_local<<<grid_for(p.n_local), 256, 0, (cudaStream_t)stream>>>(h->table(), p.d_lse, p.d_lss,
                                                                    p.d_lde, p.d_lds, p.n_local); slbm::count_launch(); }
    SLBM_CUDA_TRY(cudaGetLastError());
  }
  return SLBM_OK;
}

int slbm_halo_start_ex(SlbmHalo* h, int phase, void* after_stream, int with_local) {
  SLBM_TRY(check_phase(h, phase));
  if (!h->committed) return fail(SLBM_ECONFIG, "halo not committed");
  cudaSetDevice(h->device);
  if (after_stream) {
    SLBM_CUDA_TRY(cudaEventRecord(h->ev_ready, (cudaStream_t)after_stream));
    SLBM_CUDA_TRY(cudaStreamWaitEvent(h->comm, h->ev_ready, 0));
  }
  PhaseProg& p = h->ph[phase];
  const PdfTable t = h->table();
  const int64_t n_local = p.n_local;
  if (!with_local) p.n_local = 0;  // local edges run elsewhere (slbm_halo_local_on)
  int st;
  if (h->peer) {
    st = peer_start(h, p, phase);
  } else {
    st = nccl_start(h, p, phase, t);
  }
  p.n_local = n_local;
  return st;
}

int slbm_halo_start(SlbmHalo* h, int phase, void* after_stream) {
  return slbm_halo_start_ex(h, phase, after_stream, 1);
}

}  // extern "C"

namespace {
int nccl_start(SlbmHalo* h, PhaseProg& p, int phase, const PdfTable& t) {
  if (p.n_pack) {
    { k_pack<<<grid_for(p.n_pack), 256, 0, h->comm>>>(t, p.d_pe, p.d_ps, p.n_pack, h->d_send); slbm::count_launch(); }
    SLBM_CUDA_TRY(cudaGetLastError());
  }
  SLBM_TRY(slbm_halo_local(h, phase));
  if (!p.send_peer.empty() || !p.recv_peer.empty()) {
    if (!h->nccl) return fail(SLBM_ECONFIG, "halo has remote edges but no NCCL communicator");
    NCCL_TRY(ncclGroupStart());
    for (size_t i = 0; i < p.send_peer.size(); ++i)
      NCCL_TRY(ncclSend(h->d_send + p.send_off[i], size_t(p.send_cnt[i]), ncclFloat64,
                        p.send_peer[i], h->nccl, h->comm));
    for (size_t i = 0; i < p.recv_peer.size(); ++i)
      NCCL_TRY(ncclRecv(h->d_recv + p.recv_off[i], size_t(p.recv_cnt[i]), ncclFloat64,
                        p.recv_peer[i], h->nccl, h->comm));
    NCCL_TRY(ncclGroupEnd());
  }
  if (p.n_unpack) {
    { k_unpack<<<grid_for(p.n_unpack), 256, 0, h->comm>>>(t, p.d_upos, p.d_ue, p.d_us, p.n_unpack,
                                                         h->d_recv); slbm::count_launch(); }
    SLBM_CUDA_TRY(cudaGetLastError());
  }
  SLBM_CUDA_TRY(cudaEventRecord(h->ev_done, h->comm));
  return SLBM_OK;
}
}  // namespace

extern "C" {

int slbm_halo_wait(SlbmHalo* h, void* stream) {
  if (!h) return fail(SLBM_ECONFIG, "null halo");
  if (stream) {
    SLBM_CUDA_TRY(cudaStreamWaitEvent((cudaStream_t)stream, h->ev_done, 0));
  } else {
    SLBM_CUDA_TRY(cudaEventSynchronize(h->ev_done));
  }
  return SLBM_OK;
}

int slbm_halo_peer_sizes(const SlbmHalo* h, int phase, int npeers, int64_t* send_counts,
                         int64_t* recv_counts) {
  SLBM_TRY(check_phase(h, phase));
  const PhaseProg& p = h->ph[phase];
  for (int i = 0; i < npeers; ++i) {
    send_counts[i] = 0;
    recv_counts[i] = 0;
  }
  if (h->committed) {
    for (size_t i = 0; i < p.send_peer.size(); ++i)
      if (p.send_peer[i] < npeers) send_counts[p.send_peer[i]] = p.send_cnt[i];
    for (size_t i = 0; i < p.recv_peer.size(); ++i)
      if (p.recv_peer[i] < npeers) recv_counts[p.recv_peer[i]] = p.recv_cnt[i];
  } else {
    for (auto& kv : p.sends)
      if (kv.first < npeers) send_counts[kv.first] = int64_t(kv.second.eng.size());
    for (auto& kv : p.recvs)
      if (kv.first < npeers) recv_counts[kv.first] = kv.second.n_wire;
  }
  return SLBM_OK;
}

int slbm_halo_pack_host(SlbmHalo* h, int phase, int peer, double* host_out) {
  SLBM_TRY(check_phase(h, phase));
  if (!h->committed) return fail(SLBM_ECONFIG, "halo not committed");
  cudaSetDevice(h->device);
  PhaseProg& p = h->ph[phase];
  auto it = std::find(p.send_peer.begin(), p.send_peer.end(), peer);
  if (it == p.send_peer.end()) return SLBM_OK;
  const size_t i = size_t(it - p.send_peer.begin());
  const int64_t off = p.send_off[i], cnt = p.send_cnt[i];
  if (cnt == 0) return SLBM_OK;
  { k_pack<<<grid_for(cnt), 256, 0, h->comm>>>(h->table(), p.d_pe + off, p.d_ps + off, cnt,
                                              h->d_send + off); slbm::count_launch(); }
  SLBM_CUDA_TRY(cudaGetLastError());
  SLBM_CUDA_TRY(cudaMemcpyAsync(host_out, h->d_send + off, cnt * sizeof(double),
                                cudaMemcpyDeviceToHost, h->comm));
  SLBM_CUDA_TRY(cudaStreamSynchronize(h->comm));
  return SLBM_OK;
}

int slbm_halo_unpack_host(SlbmHalo* h, int phase, int peer, const double* host_in) {
  SLBM_TRY(check_phase(h, phase));
  if (!h->committed) return fail(SLBM_ECONFIG, "halo not committed");
  cudaSetDevice(h->device);
  PhaseProg& p = h->ph[phase];
  auto it = std::find(p.recv_peer.begin(), p.recv_peer.end(), peer);
  if (it == p.recv_peer.end()) return SLBM_OK;
  const size_t i = size_t(it - p.recv_peer.begin());
  const int64_t roff = p.recv_off[i], rcnt = p.recv_cnt[i];
  const int64_t uoff = p.unpack_off[i], ucnt = p.unpack_cnt[i];
  if (rcnt)
    SLBM_CUDA_TRY(cudaMemcpyAsync(h->d_recv + roff, host_in, rcnt * sizeof(double),
                                  cudaMemcpyHostToDevice, h->comm));
  if (ucnt) {
    { k_unpack<<<grid_for(ucnt), 256, 0, h->comm>>>(h->table(), p.d_upos + uoff, p.d_ue + uoff,
                                                   p.d_us + uoff, ucnt, h->d_recv); slbm::count_launch(); }
    SLBM_CUDA_TRY(cudaGetLastError());
  }
  SLBM_CUDA_TRY(cudaStreamSynchronize(h->comm));
  return SLBM_OK;
}

int slbm_halo_use_peer(SlbmHalo* h, int rank) {
  if (!h) return fail(SLBM_ECONFIG, "null halo");
  if (h->committed) return fail(SLBM_ECONFIG, "halo already committed");
  if (rank < 0 || rank >= kMaxPeers) return fail(SLBM_ECONFIG, "peer transport: rank out of range");
  h->peer = true;
  h->rank = rank;
  return SLBM_OK;
}

int slbm_halo_ipc_handles(const SlbmHalo* h, void* recv_handle, void* flags_handle) {
  if (!h || !h->committed || !h->peer) return fail(SLBM_ECONFIG, "peer halo not committed");
  cudaSetDevice(h->device);
  cudaIpcMemHandle_t a, b;
  SLBM_CUDA_TRY(cudaIpcGetMemHandle(&a, h->d_recv));
  SLBM_CUDA_TRY(cudaIpcGetMemHandle(&b, h->d_flags));
  std::memcpy(recv_handle, &a, sizeof(a));
  std::memcpy(flags_handle, &b, sizeof(b));
  return SLBM_OK;
}

int slbm_halo_recv_section(const SlbmHalo* h, int phase, int peer, int64_t* offset,
                           int64_t* count) {
  SLBM_TRY(check_phase(h, phase));
  if (!h->committed) return fail(SLBM_ECONFIG, "halo not committed");
  const PhaseProg& p = h->ph[phase];
  *offset = -1;
  *count = 0;
  for (size_t i = 0; i < p.recv_peer.size(); ++i)
    if (p.recv_peer[i] == peer) {
      *offset = p.recv_off[i];
      *count = p.recv_cnt[i];
    }
  return SLBM_OK;
}

int slbm_halo_connect(SlbmHalo* h, int peer, const void* recv_handle, const void* flags_handle,
                      const int64_t* section_offset, const int64_t* section_count) {
  if (!h || !h->committed || !h->peer) return fail(SLBM_ECONFIG, "peer halo not committed");
  if (peer < 0 || peer >= kMaxPeers) return fail(SLBM_ECONFIG, "peer rank out of range");
  cudaSetDevice(h->device);
  double* recv = nullptr;
  uint64_t* flags = nullptr;
  if (peer == h->rank) {  // loopback: this process's own buffers
    recv = h->d_recv;
    flags = h->d_flags;
  } else {
    cudaIpcMemHandle_t a, b;
    std::memcpy(&a, recv_handle, sizeof(a));
    std::memcpy(&b, flags_handle, sizeof(b));
    void* pa = nullptr;
    void* pb = nullptr;
    SLBM_CUDA_TRY(cudaIpcOpenMemHandle(&pa, a, cudaIpcMemLazyEnablePeerAccess));
    SLBM_CUDA_TRY(cudaIpcOpenMemHandle(&pb, b, cudaIpcMemLazyEnablePeerAccess));
    h->opened.push_back(pa);
    h->opened.push_back(pb);
    recv = static_cast<double*>(pa);
    flags = static_cast<uint64_t*>(pb);
  }
  h->peer_recv[peer] = recv;
  h->peer_flags[peer] = flags;
  for (int ph = 0; ph < 2; ++ph) {
    PhaseProg& p = h->ph[ph];
    for (size_t i = 0; i < p.send_peer.size(); ++i) {
      if (p.send_peer[i] != peer) continue;
      if (section_count[ph] != p.send_cnt[i] || section_offset[ph] < 0)
        return fail(SLBM_EPROTOCOL, "peer transport: message length disagrees with the receiver");
      p.remote_dst[i] = recv + section_offset[ph];
    }
  }
  return SLBM_OK;
}

int slbm_nccl_get_unique_id(void* unique_id_out) {
  if (!unique_id_out) return fail(SLBM_ECONFIG, "null id buffer");
  ncclUniqueId id;
  NCCL_TRY(ncclGetUniqueId(&id));
  std::memcpy(unique_id_out, &id, sizeof(id));
  return SLBM_OK;
}

int slbm_nccl_comm_init(const void* unique_id, int nranks, int rank, int device, void** comm) {
  if (!unique_id || !comm) return fail(SLBM_ECONFIG, "null argument");
  cudaSetDevice(device);
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  ncclComm_t c = nullptr;
  NCCL_TRY(ncclCommInitRank(&c, nranks, id, rank));
  *comm = (void*)c;
  return SLBM_OK;
}

int slbm_nccl_comm_destroy(void* comm) {
  if (!comm) return SLBM_OK;
  NCCL_TRY(ncclCommDestroy((ncclComm_t)comm));
  return SLBM_OK;
}

}  // extern "C"
