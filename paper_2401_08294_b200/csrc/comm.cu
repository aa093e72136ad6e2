// comm.cu — peer-memory communicator for the tensor-parallel merges ("merged
// twice") and the layer-pipeline hand-off.
//
// One process per GPU.  Every rank owns one cudaMalloc'd mailbox, exported with
// a CUDA IPC handle and mapped by its peers (NVLink / NVSwitch P2P on an HGX
// B200 box).  All protocol state lives in device memory (epoch counters, flags)
// so the operations are stream-ordered and CUDA-graph replayable:
//
//  all-reduce (one-shot, deterministic): each rank copies its partial into its
//    own mailbox slot [epoch % 2], publishes flag[me] = epoch on every group
//    peer (st.release.sys), waits until all group peers published the same
//    epoch into its own mailbox, then sums the peers' slots IN RANK ORDER —
//    every rank computes bit-identical sums.  Slot reuse is safe: a peer can
//    only publish epoch e+1 after finishing epoch e.
//  send/recv: the sender waits for the receiver's ack of epoch s-2, writes the
//    payload straight into the receiver's slot [s % 2], fences, and publishes
//    the flag; the receiver waits, copies out, and acks into the sender's box.
//
// Each kernel runs a small grid (<= 32 CTAs, all co-resident) and uses an
// in-mailbox arrival counter as the grid barrier between phases.
//
// NCCL mode (if_comm_init, the library-collective baseline of SURVEY §8(b)): the same
// calls map to ncclAllReduce on the TP group's communicator (ncclCommSplit by stage)
// and ncclSend/ncclRecv on the world communicator.  NCCL is opened with dlopen at
// if_comm_init time (no link dependency: a process that already loaded torch's
// libnccl.so.2 reuses it).
#include <dlfcn.h>
#include <nccl.h>
#include <stdlib.h>
#include <string.h>

#include "comm.cuh"
#include "common.cuh"

namespace ifb {

struct MailboxHdr {
  unsigned long long ar_flag[8];  // written by group peers: epoch of their published partial
  unsigned long long p2p_flag;    // written by the previous stage
  unsigned long long p2p_ack;     // written by the next stage
  unsigned long long ar_epoch;    // local counters
  unsigned long long send_epoch;
  unsigned long long recv_epoch;
  unsigned int arrive[4];  // grid-barrier counters (local)
  unsigned int pad[2];
};
static_assert(sizeof(MailboxHdr) <= 256, "header");
static constexpr size_t kHdr = 256;

}  // namespace ifb

struct if_comm_s {
  int kind = 0;  // 0 = peer memory (CUDA IPC), 1 = NCCL
  ncclComm_t world = nullptr, group_comm = nullptr;
  if_plan plan;
  int rank, stage, group_rank;
  int64_t max_elems;
  unsigned char* box = nullptr;        // own mailbox
  unsigned char* peer[8] = {nullptr};  // mapped mailboxes (peer[rank] = box)
  bool opened[8] = {false};
  int group[8], ngroup = 0;  // ranks of my TP group in group-rank order
  int next = -1, prev = -1;  // pipeline neighbours (same group rank)
  int hidden = 0;            // rows of the decode engine's TP exchange region
  int engine_grid = 0;       // CTAs of this rank's decode engine (0: every SM; ranks sharing a GPU split them)
  bool local = false;        // if_comm_create_local: every rank in this process, concurrent streams
  bool shared_gpu = false;   // a peer process maps a mailbox on this same GPU (no concurrency guarantee)
};

namespace ifb {

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// grid barrier among the CTAs of one (small, co-resident) launch; counter reset by the last arriver
__device__ void grid_sync(unsigned int* counter, unsigned int* gen_counter) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int* gen = gen_counter;
    unsigned int g = *gen;
    __threadfence();
    if (atomicAdd(counter, 1u) == gridDim.x - 1) {
      *counter = 0;
      __threadfence();
      atomicAdd(gen_counter, 1u);
    } else {
      while (*gen == g) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

struct ARArgs {
  unsigned char* box;                // own mailbox
  unsigned char* peers[8];           // mailboxes of the group members in group-rank order
  int ngroup, me;                    // my index in the group
  int64_t slot_elems;
};

// dst[i] (+)= sum_g partial_g[i] over the TP group, fixed order g = 0..ngroup-1
__global__ void __launch_bounds__(256) allreduce_kernel(ARArgs a, const float* __restrict__ src, float* dst,
                                                       int64_t n, int accumulate) {
  MailboxHdr* h = reinterpret_cast<MailboxHdr*>(a.box);
  const unsigned long long e = h->ar_epoch + 1;  // same value for every CTA (updated at the very end)
  const int slot = (int)(e & 1ull);
  float* mine = reinterpret_cast<float*>(a.box + kHdr) + (size_t)slot * a.slot_elems;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = tid; i < n; i += stride) mine[i] = src[i];
  grid_sync(&h->arrive[0], &h->arrive[1]);
  if (blockIdx.x == 0 && threadIdx.x < a.ngroup) {
    __threadfence_system();
    MailboxHdr* ph = reinterpret_cast<MailboxHdr*>(a.peers[threadIdx.x]);
    st_release_sys(&ph->ar_flag[a.me], e);
  }
  if (threadIdx.x < a.ngroup) {
    while (ld_acquire_sys(&h->ar_flag[threadIdx.x]) < e) __nanosleep(64);
  }
  __syncthreads();
  for (int64_t i = tid; i < n; i += stride) {
    float s = 0.f;
    for (int g = 0; g < a.ngroup; g++) {
      const volatile float* p = reinterpret_cast<const volatile float*>(a.peers[g] + kHdr) + (size_t)slot * a.slot_elems;
      s += p[i];
    }
    dst[i] = accumulate ? dst[i] + s : s;
  }
  grid_sync(&h->arrive[0], &h->arrive[1]);
  if (blockIdx.x == 0 && threadIdx.x == 0) h->ar_epoch = e;
}

struct P2PArgs {
  unsigned char* box;   // own mailbox
  unsigned char* peer;  // receiver's (send) or sender's (recv) mailbox
  int64_t slot_elems;
};

// payload slots live after the two all-reduce slots
__device__ __forceinline__ float* p2p_slot(unsigned char* box, int64_t slot_elems, int s) {
  return reinterpret_cast<float*>(box + kHdr) + (size_t)(2 + s) * slot_elems;
}

__global__ void __launch_bounds__(256) send_kernel(P2PArgs a, const float* __restrict__ src, int64_t n) {
  MailboxHdr* h = reinterpret_cast<MailboxHdr*>(a.box);
  MailboxHdr* rh = reinterpret_cast<MailboxHdr*>(a.peer);
  const unsigned long long e = h->send_epoch + 1;
  if (threadIdx.x == 0) {
    // the receiver must have consumed epoch e-2 (same slot)
    while (e > 2 && ld_acquire_sys(&h->p2p_ack) < e - 2) __nanosleep(64);
  }
  __syncthreads();
  float* dst = p2p_slot(a.peer, a.slot_elems, (int)(e & 1ull));
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = tid; i < n; i += stride) dst[i] = src[i];
  __threadfence_system();
  grid_sync(&h->arrive[2], &h->arrive[3]);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    __threadfence_system();
    st_release_sys(&rh->p2p_flag, e);
    h->send_epoch = e;
  }
}

__global__ void __launch_bounds__(256) recv_kernel(P2PArgs a, float* __restrict__ dst, int64_t n) {
  MailboxHdr* h = reinterpret_cast<MailboxHdr*>(a.box);
  MailboxHdr* sh = reinterpret_cast<MailboxHdr*>(a.peer);
  const unsigned long long e = h->recv_epoch + 1;
  if (threadIdx.x == 0) {
    while (ld_acquire_sys(&h->p2p_flag) < e) __nanosleep(64);
  }
  __syncthreads();
  const volatile float* src = p2p_slot(a.box, a.slot_elems, (int)(e & 1ull));
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = tid; i < n; i += stride) dst[i] = src[i];
  grid_sync(&h->arrive[2], &h->arrive[3]);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    __threadfence_system();
    st_release_sys(&sh->p2p_ack, e);
    h->recv_epoch = e;
  }
}

// ---- NCCL (dlopen'ed) ---------------------------------------------------------
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  const char* (*GetErrorString)(ncclResult_t);
  bool ok = false;
};
static NcclApi* nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
#define IFB_SYM(f) *reinterpret_cast<void**>(&api.f) = dlsym(h, "nccl" #f)
      IFB_SYM(GetUniqueId); IFB_SYM(CommInitRank); IFB_SYM(CommSplit); IFB_SYM(CommDestroy);
      IFB_SYM(AllReduce); IFB_SYM(Send); IFB_SYM(Recv); IFB_SYM(GetErrorString);
#undef IFB_SYM
      api.ok = api.GetUniqueId && api.CommInitRank && api.CommSplit && api.CommDestroy && api.AllReduce && api.Send &&
               api.Recv && api.GetErrorString;
    }
  }
  return api.ok ? &api : nullptr;
}
static if_status nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return IF_OK;
  NcclApi* a = nccl();
  return set_error(IF_ERR_COMM, "%s: NCCL: %s", what, a ? a->GetErrorString(r) : "?");
}

// dst[i] += src[i]  (the NCCL path's accumulate: the stack's residual add after a merge)
__global__ void __launch_bounds__(256) add_into_kernel(const float* __restrict__ src, float* __restrict__ dst, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] += src[i];
}

static int comm_grid(int64_t n) {
  int64_t g = (n + 2047) / 2048;
  if (g < 1) g = 1;
  if (g > 32) g = 32;
  return (int)g;
}

if_status comm_allreduce_into(if_comm c, const float* src, float* dst, int64_t n, int accumulate, cudaStream_t st) {
  if (!c) return set_error(IF_ERR_ARG, "allreduce: null comm");
  if (c->kind == 1) {
    // NCCL: sum in place over the TP group (src is the caller's partial buffer), then
    // add into dst when accumulating (reduction order is NCCL's, Q21)
    float* buf = accumulate ? const_cast<float*>(src) : dst;
    if_status r = nccl_check(nccl()->AllReduce(src, buf, (size_t)n, ncclFloat32, ncclSum, c->group_comm, st),
                             "allreduce");
    if (r) return r;
    if (accumulate) {
      add_into_kernel<<<comm_grid(n), 256, 0, st>>>(buf, dst, n);
      count_launch();
    }
    return check_launch("allreduce");
  }
  if (n > c->max_elems) return set_error(IF_ERR_SHAPE, "allreduce: n=%lld > capacity %lld", (long long)n, (long long)c->max_elems);
  ARArgs a;
  a.box = c->box;
  a.ngroup = c->ngroup;
  a.me = c->group_rank;
  a.slot_elems = c->max_elems;
  for (int g = 0; g < 8; g++) a.peers[g] = g < c->ngroup ? c->peer[c->group[g]] : nullptr;
  for (int g = 0; g < c->ngroup; g++)
    if (!a.peers[g]) return set_error(IF_ERR_COMM, "allreduce: peer %d not opened", c->group[g]);
  allreduce_kernel<<<comm_grid(n), 256, 0, st>>>(a, src, dst, n, accumulate);
  count_launch();
  return check_launch("allreduce");
}

if_status comm_send(if_comm c, const float* src, int64_t n, cudaStream_t st) {
  if (!c || c->next < 0) return set_error(IF_ERR_ARG, "send: no next stage");
  if (c->kind == 1) return nccl_check(nccl()->Send(src, (size_t)n, ncclFloat32, c->next, c->world, st), "send");
  if (n > c->max_elems) return set_error(IF_ERR_SHAPE, "send: n too large");
  if (!c->peer[c->next]) return set_error(IF_ERR_COMM, "send: peer not opened");
  P2PArgs a{c->box, c->peer[c->next], c->max_elems};
  send_kernel<<<comm_grid(n), 256, 0, st>>>(a, src, n);
  count_launch();
  return check_launch("send");
}

if_status comm_recv(if_comm c, float* dst, int64_t n, cudaStream_t st) {
  if (!c || c->prev < 0) return set_error(IF_ERR_ARG, "recv: no previous stage");
  if (c->kind == 1) return nccl_check(nccl()->Recv(dst, (size_t)n, ncclFloat32, c->prev, c->world, st), "recv");
  if (n > c->max_elems) return set_error(IF_ERR_SHAPE, "recv: n too large");
  if (!c->peer[c->prev]) return set_error(IF_ERR_COMM, "recv: peer not opened");
  P2PArgs a{c->box, c->peer[c->prev], c->max_elems};
  recv_kernel<<<comm_grid(n), 256, 0, st>>>(a, dst, n);
  count_launch();
  return check_launch("recv");
}

int comm_group_size(if_comm c) { return c ? c->ngroup : 1; }

// the decode engine's TP exchange regions of my group (group-rank order), or false
// when this communicator cannot carry them (NCCL kind, peers not opened)
bool comm_engine(if_comm c, float** boxes, int* ngroup, int* me, int* hidden, int* grid) {
  // ranks in other processes on this same GPU are time-sliced, never co-resident:
  // the in-engine merge would wait forever for a peer that cannot run
  if (!c || c->kind != 0 || c->ngroup < 2 || c->shared_gpu) return false;
  for (int g = 0; g < c->ngroup; g++) {
    unsigned char* b = c->peer[c->group[g]];
    if (!b) return false;
    boxes[g] = reinterpret_cast<float*>(b + kHdr + (size_t)4 * c->max_elems * sizeof(float));
  }
  *ngroup = c->ngroup;
  *me = c->group_rank;
  *hidden = c->hidden;
  *grid = c->engine_grid;
  return true;
}

}  // namespace ifb

using namespace ifb;

static void comm_topology(if_comm c, const if_plan* plan, int rank) {
  c->plan = *plan;
  c->rank = rank;
  c->stage = plan->a[rank].stage;
  c->group_rank = plan->a[rank].group_rank;
  for (int d = 0; d < plan->devices; d++)
    if (plan->a[d].stage == c->stage) c->group[plan->a[d].group_rank] = d;
  c->ngroup = plan->groups;
  // pipeline ring: stage s sends to s+1; the last stage's "next" wraps to stage 0 (the
  // decode loop's feedback of the step output -- if_run_stack itself only sends forward
  // from non-last stages and receives on non-first stages)
  if (plan->stages > 1) {
    c->next = ((c->stage + 1) % plan->stages) * plan->groups + c->group_rank;
    c->prev = ((c->stage + plan->stages - 1) % plan->stages) * plan->groups + c->group_rank;
  }
}

// Load the communicator's kernels now.  With CUDA's lazy module loading the first
// launch of a kernel loads its module, which can wait for the device to drain: a
// first send launched while this rank's decode engine spins on a TP peer that is not
// running yet would then deadlock.
static void comm_preload() {
  static bool done = false;
  if (done) return;
  done = true;
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, allreduce_kernel);
  cudaFuncGetAttributes(&fa, send_kernel);
  cudaFuncGetAttributes(&fa, recv_kernel);
  cudaFuncGetAttributes(&fa, add_into_kernel);
}

extern "C" if_status if_comm_create(const if_plan* plan, int32_t rank, int64_t max_tokens, int32_t hidden, if_comm* out) {
  comm_preload();
  if (!plan || !out) return set_error(IF_ERR_ARG, "if_comm_create: null pointer");
  if (rank < 0 || rank >= plan->devices) return set_error(IF_ERR_ARG, "if_comm_create: rank %d outside plan", rank);
  if (max_tokens < 1 || hidden < 1) return set_error(IF_ERR_SHAPE, "if_comm_create: max_tokens/hidden");
  if_comm c = new if_comm_s();
  comm_topology(c, plan, rank);
  c->max_elems = max_tokens * (int64_t)hidden;
  c->hidden = hidden;
  // [header][2 all-reduce slots][2 p2p slots][decode-engine TP exchange: 2 slots x 8 ranks x hidden]
  const size_t bytes = kHdr + (size_t)4 * c->max_elems * sizeof(float) + (size_t)16 * hidden * sizeof(float);
  if (cudaMalloc(&c->box, bytes) != cudaSuccess || cudaMemset(c->box, 0, bytes) != cudaSuccess ||
      cudaDeviceSynchronize() != cudaSuccess) {
    delete c;
    return check_launch("if_comm_create");
  }
  c->peer[rank] = c->box;
  *out = c;
  return IF_OK;
}

extern "C" if_status if_comm_create_local(const if_plan* plan, int64_t max_tokens, int32_t hidden, if_comm* outs) {
  if (!plan || !outs) return set_error(IF_ERR_ARG, "if_comm_create_local: null pointer");
  int sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  for (int r = 0; r < plan->devices; r++) {
    if_status st = if_comm_create(plan, r, max_tokens, hidden, &outs[r]);
    if (st) {
      for (int q = 0; q < r; q++) if_comm_destroy(outs[q]);
      return st;
    }
  }
  for (int r = 0; r < plan->devices; r++) {
    for (int q = 0; q < plan->devices; q++) outs[r]->peer[q] = outs[q]->box;  // same device: plain pointers
    // every rank's engine grid co-resident on this GPU, leaving two SMs per rank for
    // the small hand-off kernels (a 227 KB engine CTA cannot share an SM with them)
    outs[r]->engine_grid = (sms - 2 * plan->devices) / plan->devices;
    outs[r]->local = true;
  }
  return IF_OK;
}

extern "C" if_status if_comm_nccl_unique_id(uint8_t* id128) {
  if (!id128) return set_error(IF_ERR_ARG, "if_comm_nccl_unique_id: null pointer");
  NcclApi* a = nccl();
  if (!a) return set_error(IF_ERR_COMM, "if_comm_nccl_unique_id: libnccl.so.2 not loadable");
  ncclUniqueId id;
  if_status r = nccl_check(a->GetUniqueId(&id), "ncclGetUniqueId");
  if (r) return r;
  static_assert(sizeof(id) == 128, "nccl unique id size");
  memcpy(id128, &id, 128);
  return IF_OK;
}

extern "C" if_status if_comm_init(const if_plan* plan, int32_t rank, const uint8_t* nccl_unique_id, if_comm* out) {
  if (!plan || !out || !nccl_unique_id) return set_error(IF_ERR_ARG, "if_comm_init: null pointer");
  if (rank < 0 || rank >= plan->devices) return set_error(IF_ERR_ARG, "if_comm_init: rank %d outside plan", rank);
  NcclApi* a = nccl();
  if (!a) return set_error(IF_ERR_COMM, "if_comm_init: libnccl.so.2 not loadable");
  comm_preload();
  if_comm c = new if_comm_s();
  c->kind = 1;
  comm_topology(c, plan, rank);
  ncclUniqueId id;
  memcpy(&id, nccl_unique_id, 128);
  if_status r = nccl_check(a->CommInitRank(&c->world, plan->devices, id, rank), "ncclCommInitRank");
  if (!r) r = nccl_check(a->CommSplit(c->world, c->stage, c->group_rank, &c->group_comm, nullptr), "ncclCommSplit");
  if (r) {
    if (c->world) a->CommDestroy(c->world);
    delete c;
    return r;
  }
  *out = c;
  return IF_OK;
}

extern "C" if_status if_comm_ipc_handle(if_comm c, uint8_t* handle64) {
  if (!c || !handle64) return set_error(IF_ERR_ARG, "if_comm_ipc_handle: null pointer");
  if (c->kind != 0) return set_error(IF_ERR_ARG, "if_comm_ipc_handle: not a peer-memory communicator");
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, c->box) != cudaSuccess) return check_launch("if_comm_ipc_handle");
  static_assert(sizeof(h) == 64, "ipc handle size");
  memcpy(handle64, &h, 64);
  return IF_OK;
}

extern "C" if_status if_comm_open_peers(if_comm c, const uint8_t* handles) {
  if (!c || !handles) return set_error(IF_ERR_ARG, "if_comm_open_peers: null pointer");
  if (c->kind != 0) return set_error(IF_ERR_ARG, "if_comm_open_peers: not a peer-memory communicator");
  // only the ranks we talk to: my TP group and my pipeline neighbours
  for (int d = 0; d < c->plan.devices; d++) {
    bool need = (c->plan.a[d].stage == c->stage) || d == c->next || d == c->prev;
    if (!need || d == c->rank || c->opened[d]) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, handles + 64 * d, 64);
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
      return set_error(IF_ERR_COMM, "if_comm_open_peers: rank %d: %s", d, cudaGetErrorString(cudaGetLastError()));
    c->peer[d] = static_cast<unsigned char*>(p);
    c->opened[d] = true;
    cudaPointerAttributes pa;
    int me = -1;
    cudaGetDevice(&me);
    if (cudaPointerGetAttributes(&pa, p) == cudaSuccess && pa.device == me) c->shared_gpu = true;
  }
  return IF_OK;
}

extern "C" if_status if_comm_destroy(if_comm c) {
  if (!c) return IF_OK;
  cudaDeviceSynchronize();
  if (c->kind == 1) {
    if (c->group_comm) nccl()->CommDestroy(c->group_comm);
    if (c->world) nccl()->CommDestroy(c->world);
    delete c;
    return IF_OK;
  }
  for (int d = 0; d < 8; d++)
    if (c->opened[d]) cudaIpcCloseMemHandle(c->peer[d]);
  if (c->box) cudaFree(c->box);
  delete c;
  return IF_OK;
}

extern "C" if_status if_comm_allreduce(if_comm c, float* buf, int64_t n, if_stream_t stream) {
  if (!buf && n > 0) return set_error(IF_ERR_ARG, "if_comm_allreduce: null buffer");
  if (n == 0) return IF_OK;
  return comm_allreduce_into(c, buf, buf, n, 0, (cudaStream_t)stream);
}

extern "C" if_status if_comm_send_next(if_comm c, const float* buf, int64_t n, if_stream_t stream) {
  if (!buf && n > 0) return set_error(IF_ERR_ARG, "if_comm_send_next: null buffer");
  return comm_send(c, buf, n, (cudaStream_t)stream);
}

extern "C" if_status if_comm_recv_prev(if_comm c, float* buf, int64_t n, if_stream_t stream) {
  if (!buf && n > 0) return set_error(IF_ERR_ARG, "if_comm_recv_prev: null buffer");
  return comm_recv(c, buf, n, (cudaStream_t)stream);
}
