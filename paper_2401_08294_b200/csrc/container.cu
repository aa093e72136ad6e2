// container.cu — packed-tensor container I/O (SPEC S:122-123 section
// layout, Q28) and the partition cost model / auto-planner calibrated on
// measured B200 numbers (S:629-637 estimate, "merged twice", Table 5 P:224-237;
// Q29).
// ifb-build: -std=c++17
//   (host-only file; nvcc 12.9's C++20 front end aborts on the STL here)
//
// File: "IFQC" | u32 version 1 | u32 tensor count | sections.  Section: u16 name
// length, name, u8 scheme id (qtype), u16 block, u8 ndim, u32 dims[ndim], u32 block
// count, then the packed blocks exactly as if_quantize writes them.
//
// Loading into HBM is a pipelined host->device stream: R reader threads each own two
// pinned staging buffers; a thread pread()s its next chunk into a free buffer (the
// buffer's event says its previous H2D copy drained), enqueues the async copy on the
// caller's stream and records the event.  File reads, PCIe transfers and the other
// readers overlap; the destination needs no staging copy in device memory.
#include <fcntl.h>
#include <stdio.h>
#include <string.h>
#include <sys/stat.h>
#include <unistd.h>

#include <string>
#include <thread>
#include <vector>

#include "common.cuh"

namespace ifb {

constexpr uint32_t CT_VERSION = 1;
constexpr int CT_READERS = 4;
constexpr size_t CT_CHUNK = (size_t)16 << 20;

struct CtEntry {
  std::string name;
  if_scheme s;
  int32_t ndim;
  int64_t dims[8];
  int64_t nblocks;
  int64_t offset;  // payload offset in the file
  int64_t bytes;
};

}  // namespace ifb

struct if_container_s {
  int fd = -1;
  std::vector<ifb::CtEntry> e;
  void* stage[ifb::CT_READERS][2] = {};
  cudaEvent_t ev[ifb::CT_READERS][2] = {};
  bool staged = false;
};

using namespace ifb;

static bool rd(int fd, int64_t off, void* dst, size_t n) {
  size_t got = 0;
  while (got < n) {
    const ssize_t r = pread(fd, static_cast<char*>(dst) + got, n - got, off + (int64_t)got);
    if (r <= 0) return false;
    got += (size_t)r;
  }
  return true;
}

static void ct_free(if_container c) {
  if (c->fd >= 0) close(c->fd);
  for (int t = 0; t < CT_READERS; t++)
    for (int b = 0; b < 2; b++) {
      if (c->ev[t][b]) cudaEventDestroy(c->ev[t][b]);
      if (c->stage[t][b]) cudaFreeHost(c->stage[t][b]);
    }
  delete c;
}

extern "C" if_status if_container_open(const char* path, if_container* out) {
  if (!path || !out) return set_error(IF_ERR_ARG, "if_container_open: null pointer");
  *out = nullptr;
  const int fd = open(path, O_RDONLY);
  if (fd < 0) return set_error(IF_ERR_IO, "if_container_open: cannot open %s", path);
  struct stat stt;
  if (fstat(fd, &stt) != 0) {
    close(fd);
    return set_error(IF_ERR_IO, "if_container_open: cannot stat %s", path);
  }
  const int64_t size = stt.st_size;
  if_container c = new if_container_s();
  c->fd = fd;
  int64_t off = 0;
  auto fail = [&](const char* what) {
    ct_free(c);
    return set_error(IF_ERR_IO, "if_container_open: %s: %s at byte %lld", path, what, (long long)off);
  };
  auto take = [&](void* dst, size_t n) {
    if (off + (int64_t)n > size || !rd(fd, off, dst, n)) return false;
    off += (int64_t)n;
    return true;
  };
  char magic[4];
  uint32_t ver = 0, count = 0;
  if (!take(magic, 4) || memcmp(magic, "IFQC", 4)) return fail("bad magic");
  if (!take(&ver, 4) || ver != CT_VERSION) return fail("unsupported version");
  if (!take(&count, 4)) return fail("truncated file header");
  for (uint32_t i = 0; i < count; i++) {
    CtEntry en;
    uint16_t ln = 0, bs = 0;
    uint8_t qt = 0, nd = 0;
    if (!take(&ln, 2)) return fail("truncated name length");
    en.name.resize(ln);
    if (!take(en.name.data(), ln)) return fail("truncated name");
    if (!take(&qt, 1) || !take(&bs, 2)) return fail("truncated scheme");
    en.s = if_scheme{(int32_t)qt, (int32_t)bs};
    if (!scheme_ok(en.s)) {
      off -= 3;
      return fail("invalid scheme");
    }
    if (!take(&nd, 1) || nd < 1 || nd > 8) return fail("dim count");
    en.ndim = nd;
    int64_t n = 1;
    for (int k = 0; k < nd; k++) {
      uint32_t d = 0;
      if (!take(&d, 4)) return fail("truncated dims");
      en.dims[k] = d;
      n *= d;
    }
    uint32_t nb = 0;
    if (!take(&nb, 4)) return fail("truncated block count");
    if (en.dims[nd - 1] % bs || (int64_t)nb != n / bs) {
      off -= 4;
      return fail("block count inconsistent with dims");
    }
    en.nblocks = nb;
    en.bytes = (int64_t)nb * q_block_bytes(qt, bs);
    en.offset = off;
    if (off + en.bytes > size) return fail("truncated payload");
    off += en.bytes;
    c->e.push_back(std::move(en));
  }
  if (off != size) return fail("trailing bytes");
  *out = c;
  return IF_OK;
}

extern "C" if_status if_container_close(if_container c) {
  if (!c) return set_error(IF_ERR_ARG, "if_container_close: null");
  if (c->staged) cudaDeviceSynchronize();  // staging buffers may still feed copies
  ct_free(c);
  return IF_OK;
}

extern "C" int32_t if_container_count(if_container c) { return c ? (int32_t)c->e.size() : -1; }

extern "C" if_status if_container_info(if_container c, int32_t i, char* name, int32_t name_cap, if_scheme* s,
                                       int32_t* ndim, int64_t* dims, int64_t* bytes) {
  if (!c || i < 0 || i >= (int32_t)c->e.size()) return set_error(IF_ERR_ARG, "if_container_info: index %d", i);
  const CtEntry& en = c->e[i];
  if (name && name_cap > 0) snprintf(name, (size_t)name_cap, "%s", en.name.c_str());
  if (s) *s = en.s;
  if (ndim) *ndim = en.ndim;
  if (dims)
    for (int k = 0; k < en.ndim; k++) dims[k] = en.dims[k];
  if (bytes) *bytes = en.bytes;
  return IF_OK;
}

extern "C" if_status if_container_find(if_container c, const char* name, int32_t* index) {
  if (!c || !name || !index) return set_error(IF_ERR_ARG, "if_container_find: null pointer");
  for (size_t i = 0; i < c->e.size(); i++)
    if (c->e[i].name == name) {
      *index = (int32_t)i;
      return IF_OK;
    }
  *index = -1;
  return set_error(IF_ERR_ARG, "if_container_find: no tensor named %s", name);
}

extern "C" if_status if_container_read_host(if_container c, int32_t i, void* dst) {
  if (!c || !dst || i < 0 || i >= (int32_t)c->e.size()) return set_error(IF_ERR_ARG, "if_container_read_host: args");
  const CtEntry& en = c->e[i];
  if (!rd(c->fd, en.offset, dst, (size_t)en.bytes)) return set_error(IF_ERR_IO, "if_container_read_host: read failed");
  return IF_OK;
}

extern "C" if_status if_container_load(if_container c, int32_t i, void* dst_device, if_stream_t stream) {
  if (!c || !dst_device || i < 0 || i >= (int32_t)c->e.size()) return set_error(IF_ERR_ARG, "if_container_load: args");
  cudaStream_t st = (cudaStream_t)stream;
  if (!c->staged) {
    for (int t = 0; t < CT_READERS; t++)
      for (int b = 0; b < 2; b++)
        if (cudaMallocHost(&c->stage[t][b], CT_CHUNK) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev[t][b], cudaEventDisableTiming) != cudaSuccess)
          return set_error(IF_ERR_CUDA, "if_container_load: staging buffers");
    c->staged = true;
  }
  const CtEntry& en = c->e[i];
  const int64_t chunks = (en.bytes + (int64_t)CT_CHUNK - 1) / (int64_t)CT_CHUNK;
  const int readers = (int)std::min<int64_t>(CT_READERS, std::max<int64_t>(chunks, 1));
  std::vector<int> err(readers, 0);
  auto reader = [&](int t) {
    int b = 0;
    for (int64_t j = t; j < chunks; j += readers, b ^= 1) {
      const int64_t o = j * (int64_t)CT_CHUNK;
      const size_t n = (size_t)std::min<int64_t>((int64_t)CT_CHUNK, en.bytes - o);
      if (cudaEventSynchronize(c->ev[t][b]) != cudaSuccess) {  // the buffer's previous copy drained
        err[t] = 2;
        return;
      }
      if (!rd(c->fd, en.offset + o, c->stage[t][b], n)) {
        err[t] = 1;
        return;
      }
      if (cudaMemcpyAsync(static_cast<char*>(dst_device) + o, c->stage[t][b], n, cudaMemcpyHostToDevice, st) !=
              cudaSuccess ||
          cudaEventRecord(c->ev[t][b], st) != cudaSuccess) {
        err[t] = 2;
        return;
      }
    }
  };
  std::vector<std::thread> th;
  for (int t = 1; t < readers; t++) th.emplace_back(reader, t);
  reader(0);
  for (auto& x : th) x.join();
  for (int t = 0; t < readers; t++) {
    if (err[t] == 1) return set_error(IF_ERR_IO, "if_container_load: read of %s failed", en.name.c_str());
    if (err[t] == 2) return check_launch("if_container_load");
  }
  return IF_OK;
}

extern "C" if_status if_container_save(const char* path, int32_t n, const char* const* names, const if_scheme* schemes,
                                       const int32_t* ndims, const int64_t* dims /* n x 8 */,
                                       const void* const* data, int32_t data_on_device, if_stream_t stream) {
  if (!path || n < 0 || (n > 0 && (!names || !schemes || !ndims || !dims || !data)))
    return set_error(IF_ERR_ARG, "if_container_save: null pointer");
  FILE* f = fopen(path, "wb");
  if (!f) return set_error(IF_ERR_IO, "if_container_save: cannot create %s", path);
  auto put = [&](const void* p, size_t k) { return fwrite(p, 1, k, f) == k; };
  const uint32_t ver = CT_VERSION, cnt = (uint32_t)n;
  bool ok = put("IFQC", 4) && put(&ver, 4) && put(&cnt, 4);
  void* host = nullptr;
  if (data_on_device && cudaMallocHost(&host, CT_CHUNK) != cudaSuccess) ok = false;
  if_status st = IF_OK;
  for (int32_t i = 0; ok && i < n; i++) {
    const if_scheme s = schemes[i];
    const int nd = ndims[i];
    const size_t ln = strlen(names[i]);
    int64_t cnt_w = 1;
    for (int k = 0; k < nd; k++) cnt_w *= dims[i * 8 + k];
    if (!scheme_ok(s) || nd < 1 || nd > 8 || ln > 65535 || dims[i * 8 + nd - 1] % s.block || cnt_w / s.block > UINT32_MAX) {
      st = set_error(IF_ERR_SHAPE, "if_container_save: tensor %d (%s) has an invalid scheme or dims", i, names[i]);
      break;
    }
    const uint16_t ln16 = (uint16_t)ln, bs = (uint16_t)s.block;
    const uint8_t qt = (uint8_t)s.type, nd8 = (uint8_t)nd;
    const uint32_t nb = (uint32_t)(cnt_w / s.block);
    ok = put(&ln16, 2) && put(names[i], ln) && put(&qt, 1) && put(&bs, 2) && put(&nd8, 1);
    for (int k = 0; ok && k < nd; k++) {
      const uint32_t d = (uint32_t)dims[i * 8 + k];
      ok = put(&d, 4);
    }
    ok = ok && put(&nb, 4);
    const int64_t bytes = (int64_t)nb * q_block_bytes(s.type, s.block);
    if (!data_on_device) {
      ok = ok && put(data[i], (size_t)bytes);
    } else {
      for (int64_t o = 0; ok && o < bytes; o += (int64_t)CT_CHUNK) {
        const size_t k = (size_t)std::min<int64_t>((int64_t)CT_CHUNK, bytes - o);
        if (cudaMemcpyAsync(host, static_cast<const char*>(data[i]) + o, k, cudaMemcpyDeviceToHost,
                            (cudaStream_t)stream) != cudaSuccess ||
            cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) {
          st = check_launch("if_container_save");
          ok = false;
          break;
        }
        ok = put(host, k);
      }
    }
  }
  if (host) cudaFreeHost(host);
  if (fclose(f) != 0) ok = false;
  if (st) return st;
  if (!ok) return set_error(IF_ERR_IO, "if_container_save: write to %s failed", path);
  return IF_OK;
}

// ---------------------------------------------------------------------------
// partition cost model (Q29) and the auto-planner
// ---------------------------------------------------------------------------
static int64_t layer_packed_bytes(const if_stack_shape& s) {
  const int64_t d = s.hidden, nq = (int64_t)s.heads * s.head_dim, nkv = (int64_t)s.kv_heads * s.head_dim;
  const int64_t bb = q_block_bytes(s.scheme.type, s.scheme.block), bs = s.scheme.block;
  // qkv [nq + 2 nkv, d], o [d, nq], gate/up [2F, d], down [d, F]: rows x (K / block) blocks
  return ((nq + 2 * nkv) * (d / bs) + d * (nq / bs) + 2 * (int64_t)s.ffn * (d / bs) + d * (s.ffn / bs)) * bb;
}

extern "C" if_status if_cost_estimate(const if_stack_shape* shape, int32_t stages, int32_t groups,
                                      const if_cost_model* cm, int32_t micro_batches, double* decode,
                                      double* throughput) {
  if (!shape || !cm || !decode || !throughput) return set_error(IF_ERR_ARG, "if_cost_estimate: null pointer");
  if (stages < 1 || groups < 1 || groups > 8 || micro_batches < 1 || !(cm->bw_bytes_s > 0.0) || !scheme_ok(shape->scheme))
    return set_error(IF_ERR_ARG, "if_cost_estimate: stages=%d groups=%d micro_batches=%d", stages, groups, micro_batches);
  const double L = shape->layers;
  // per token: L layers on a 1/groups shard + 2 merges per layer + hand-offs
  double lat = L * (cm->t_fixed_s + ((double)layer_packed_bytes(*shape) / groups) / cm->bw_bytes_s);
  if (groups > 1) lat += 2.0 * L * cm->t_merge_s[groups];
  lat += (double)(stages - 1) * cm->t_hop_s;
  *decode = 1.0 / lat;
  *throughput = *decode * (double)std::min(stages, micro_batches);
  return IF_OK;
}

extern "C" if_status if_plan_auto(int32_t objective, const if_stack_shape* shape, int32_t devices,
                                  const if_cost_model* cm, int32_t micro_batches, if_plan* out, double* decode,
                                  double* throughput) {
  if (!shape || !cm || !out) return set_error(IF_ERR_ARG, "if_plan_auto: null pointer");
  if (objective != 0 && objective != 1) return set_error(IF_ERR_ARG, "if_plan_auto: objective %d", objective);
  bool found = false;
  double best = 0.0;
  for (int32_t g = 1; g <= devices; g++) {
    if (devices % g) continue;
    const int32_t S = devices / g;
    const int32_t strategy = g == 1 ? IF_BY_LAYER : (S == 1 ? IF_BY_TENSOR : IF_HYBRID);
    if_plan p;
    if (if_plan_partition(strategy, shape, devices, S, g, &p) != IF_OK) continue;  // invalid grid for this shape
    double dec = 0, thr = 0;
    if_status st = if_cost_estimate(shape, S, g, cm, micro_batches, &dec, &thr);
    if (st) return st;
    const double v = objective == 0 ? dec : thr;
    if (!found || v > best) {  // ties keep the grid with fewer TP ranks
      found = true;
      best = v;
      *out = p;
      if (decode) *decode = dec;
      if (throughput) *throughput = thr;
    }
  }
  if (!found) return set_error(IF_ERR_PLAN, "if_plan_auto: no valid partition of this shape over %d devices", devices);
  return IF_OK;
}
