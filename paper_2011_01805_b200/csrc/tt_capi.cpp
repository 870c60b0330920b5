// tt_capi.cpp -- the extern "C" boundary (include/tiletensor_b200.h).
//
// Each entry point: (1) validates shapes / chains on the host exactly as the
// reference operator would (raising the same error kinds and messages),
// (2) adds the reference's primitive counts to the session counters,
// (3) launches the sm_100a kernels on the session stream.  Nothing here
// computes slot values on the CPU: a session cannot be created without a
// CUDA device (TT_ERR_NO_DEVICE), so there is no host fallback path.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "tt_internal.hpp"
#include "tt_launch.hpp"

struct tt_session {
  int64_t slots = 1;
  int64_t depth = 1;
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  std::atomic<uint64_t> adds{0}, muls{0}, masks{0}, rots{0}, boots{0}, pow2{0};
  uint64_t launches = 0;
  std::mutex mu;  // serialises launches + scratch (counters are atomic)
  double* scratch = nullptr;
  std::vector<double*> retired;  // outgrown scratch buffers (see scratch_fn)
  // work-queue counters of dynamically scheduled kernels: a ring of
  // kSchedSlots (next, done) pairs, each left at zero by the launch using it
  unsigned int* sched = nullptr;
  unsigned int sched_next = 0;
  unsigned int chain_next = 0;
  size_t scratch_bytes = 0;
  int sm_count = 148;
  size_t smem_optin = 227 * 1024;
  size_t l2_bytes = size_t{126} << 20;
  // compiled rotate-and-sum schedules, keyed by (ext, t, stride, used,
  // unknown, variant): a schedule depends only on these (slots are fixed per
  // session), and rebuilding it per call costs more host time than a small
  // op's kernels take on the GPU
  std::map<std::array<int64_t, 6>, std::shared_ptr<const ttb::Program>> programs;
  // stream-ordered memory pool of tt_device_alloc / tt_device_free (operator
  // results and staging buffers of the C++ drop-in): allocations and frees are
  // ordered on the session stream, never synchronise the device, and are legal
  // inside stream capture; freed blocks stay cached in the pool (no release
  // threshold) so a steady-state op chain does no driver allocation at all
  cudaMemPool_t pool = nullptr;
  // result-tile cache of tt_tiles_alloc / tt_tiles_release: blocks freed by
  // their owner go to a free list keyed by (stream, bytes) and are handed out
  // again only on that stream (stream order makes the reuse safe, as in
  // torch's caching allocator), so a repeated op allocates with no driver call
  struct CachedBlock {
    size_t bytes;
    cudaStream_t stream;
    bool cacheable;
  };
  std::unordered_map<void*, CachedBlock> live;
  std::unordered_set<void*> direct;  // blocks from cudaMalloc (large), not the pool
  std::map<std::pair<cudaStream_t, size_t>, std::vector<void*>> free_blocks;
  size_t cached_bytes = 0;
  size_t cache_cap = size_t{8} << 30;  // a quarter of the device memory (set at creation)
};

namespace {

using namespace ttb;

thread_local std::string g_error;
thread_local int64_t g_error_pos = -1;

int set_error(int code, const std::string& msg, int64_t pos = -1) {
  g_error = msg;
  g_error_pos = pos;
  return code;
}

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    g_error.clear();
    g_error_pos = -1;
    return TT_OK;
  } catch (const Error& e) {
    return set_error(e.code, e.what(), e.position);
  } catch (const std::bad_alloc&) {
    return set_error(TT_ERR_CUDA, "out of memory");
  } catch (const std::exception& e) {
    return set_error(TT_ERR_LOGIC, e.what());
  }
}

double* scratch_fn(void* owner, size_t bytes) {
  auto* s = static_cast<tt_session*>(owner);
  if (bytes > s->scratch_bytes) {
    // a smaller buffer is retired, not freed: work already enqueued -- or
    // captured into a CUDA graph -- may still reference it (freed at destroy)
    if (s->scratch) s->retired.push_back(s->scratch);
    s->scratch = nullptr;
    bytes = std::max(bytes, s->scratch_bytes + s->scratch_bytes / 2);  // geometric growth
    check_cuda(cudaMalloc(&s->scratch, bytes), "scratch alloc");
    s->scratch_bytes = bytes;
  }
  return s->scratch;
}

LaunchCtx ctx_of(tt_session* s) {
  check_cuda(cudaSetDevice(s->device), "cudaSetDevice");
  LaunchCtx c;
  c.stream = s->stream;
  c.device = s->device;
  c.sm_count = s->sm_count;
  c.smem_optin = s->smem_optin;
  c.l2_bytes = s->l2_bytes;
  c.launches = &s->launches;
  c.scratch = scratch_fn;
  c.scratch_owner = s;
  c.sched_base = s->sched;
  c.sched_next = &s->sched_next;
  c.chain_base = s->sched ? s->sched + 2 * kSchedSlots : nullptr;
  c.chain_next = &s->chain_next;
  return c;
}

void need_session(const tt_session* s) {
  if (s == nullptr) invalid_argument("null session");
}

void add_cost(tt_session* s, const tt_cost& c, uint64_t times) {
  s->adds += c.additions * times;
  s->muls += c.multiplications * times;
  s->masks += c.mask_multiplications * times;
  s->rots += c.rotations * times;
  s->boots += c.bootstraps * times;
  s->pow2 += c.power_of_two_rotations * times;
}

void check_tiles_addressable(const Shape& sh) {
  if (sh.tile_count() >= (int64_t{1} << 31))
    invalid_argument("tile count exceeds 2^31 - 1 per tensor (shard the tensor)");
}

void copy_tiles(const LaunchCtx& c, double* out, const double* in, int64_t count) {
  if (out == in || count == 0) return;
  check_cuda(cudaMemcpyAsync(out, in, static_cast<size_t>(count) * sizeof(double),
                             cudaMemcpyDeviceToDevice, c.stream),
             "device copy");
}

// Operand tile-index strides of a broadcast operand over the out grid.
void operand_strides(const Shape& op, std::vector<int64_t>& st) {
  const auto e = op.external();
  const auto rs = row_major_strides(e);
  st.resize(e.size());
  for (size_t i = 0; i < e.size(); ++i) st[i] = e[i] == 1 ? 0 : rs[i];
}

// Group grid of a reduction over dim `di` of a product grid with external
// extents `ext`.  Dims along which an operand broadcasts are iterated
// innermost so that consecutive groups share that operand's tiles in L2.
GroupSpec make_group_spec(const std::vector<int64_t>& ext, int di,
                          const std::vector<int64_t>& a_st, const std::vector<int64_t>& b_st,
                          bool has_b) {
  GroupSpec g;
  std::vector<int64_t> gext = ext;
  gext[di] = 1;
  const auto out_st = row_major_strides(gext);
  std::vector<int> order;
  for (int i = 0; i < static_cast<int>(ext.size()); ++i)
    if (i != di && ext[i] > 1) order.push_back(i);
  auto broadcast = [&](int i) { return a_st[i] == 0 || (has_b && b_st[i] == 0); };
  std::stable_partition(order.begin(), order.end(), [&](int i) { return !broadcast(i); });
  g.nd = static_cast<int>(order.size());
  g.groups = 1;
  for (int k = 0; k < g.nd; ++k) {
    const int i = order[k];
    g.ext[k] = ext[i];
    g.out_stride[k] = out_st[i];
    g.a_stride[k] = a_st[i];
    g.b_stride[k] = has_b ? b_st[i] : 0;
    g.groups *= ext[i];
  }
  g.astep = a_st[di];
  g.bstep = has_b ? b_st[di] : 0;
  return g;
}

// Shared body of tt_sum / tt_mul_sum for a non-degenerate summed dim.
void run_reduction(tt_session* s, const Shape& prod, int di, int variant, const double* ta,
                   const std::vector<int64_t>& a_st, const double* tb,
                   const std::vector<int64_t>& b_st, double* out,
                   const Epilogue* epi = nullptr) {
  const Dim& ds = prod.dims[di];
  if (ds.interleaved && ds.unknown && ds.used() < prod.ext(di) * ds.t)
    shape_error("sum over an unknown interleaved dimension requires clean_unknowns first");
  const auto ext = prod.external();
  const int64_t stride = tile_strides(prod)[di];
  const std::array<int64_t, 6> key{ext[di], ds.t, stride, ds.used(), ds.unknown ? 1 : 0, variant};
  auto it = s->programs.find(key);
  if (it == s->programs.end()) {
    if (s->programs.size() >= 256) s->programs.clear();
    it = s->programs
             .emplace(key, std::make_shared<const Program>(build_sum_program(
                               ext[di], ds.t, stride, s->slots, ds.used(), ds.unknown, variant)))
             .first;
  }
  const Program& prog = *it->second;
  const GroupSpec g = make_group_spec(ext, di, a_st, b_st, tb != nullptr);
  add_cost(s, prog.per_group, static_cast<uint64_t>(g.groups));
  launch_group_program(ctx_of(s), prog, g, s->slots, ta, tb, out, epi);
}

// The program and group grid run_reduction would launch for tt_sum(tt_mul(a, b), dim)
// (counted like it); false when the sum is degenerate (the product itself).
struct PreparedProduct {
  std::shared_ptr<const Program> prog;
  GroupSpec g;
  Shape prod, so;
};
bool prepare_product(tt_session* s, const Shape& sa, const Shape& sb, int dim, int variant,
                     PreparedProduct& pp) {
  pp.prod = elementwise_result_shape(sa, sb, TT_OP_MUL);
  pp.so = sum_result_shape(pp.prod, dim);
  const int di = dim - 1;
  const Dim& ds = pp.prod.dims[di];
  if (ds.n == 1 && ds.d > 1) return false;
  if (ds.interleaved && ds.unknown && ds.used() < pp.prod.ext(di) * ds.t) return false;
  const auto ext = pp.prod.external();
  const int64_t stride = tile_strides(pp.prod)[di];
  const std::array<int64_t, 6> key{ext[di], ds.t, stride, ds.used(), ds.unknown ? 1 : 0, variant};
  auto it = s->programs.find(key);
  if (it == s->programs.end()) {
    if (s->programs.size() >= 256) s->programs.clear();
    it = s->programs
             .emplace(key, std::make_shared<const Program>(build_sum_program(
                               ext[di], ds.t, stride, s->slots, ds.used(), ds.unknown, variant)))
             .first;
  }
  pp.prog = it->second;
  std::vector<int64_t> ast, bst;
  operand_strides(sa, ast);
  operand_strides(sb, bst);
  pp.g = make_group_spec(ext, di, ast, bst, true);
  return true;
}

void require_slots(const tt_session* s, const Shape& sh, const char* who) {
  if (!sh.relaxed && sh.tile_slots() != s->slots)
    shape_error(std::string(who) + ": shape " + format_shape(sh) + " needs " +
                std::to_string(sh.tile_slots()) + " slots per tile, backend has " +
                std::to_string(s->slots));
  if (sh.relaxed && sh.tile_slots() > s->slots)
    shape_error(std::string(who) + ": relaxed shape exceeds the backend slot count");
}

int64_t mul_chain(int64_t ca, int64_t cb) {
  const int64_t c = std::min(ca, cb);
  if (c < 1) depth_error("multiplication at chain index 0 (bootstrap required)");
  return c - 1;
}

}  // namespace

extern "C" {

const char* tt_last_error(void) { return g_error.c_str(); }
int64_t tt_last_error_position(void) { return g_error_pos; }
const char* tt_version(void) { return "tiletensor_b200 0.1 (sm_100a)"; }

// ---- shape algebra ------------------------------------------------------------

int tt_shape_parse(const char* text, tt_shape* out) {
  return guarded([&] {
    if (!text || !out) invalid_argument("null argument");
    to_c(parse_shape(text), out);
  });
}

int tt_shape_format(const tt_shape* s, char* buf, int64_t cap) {
  return guarded([&] {
    const std::string f = format_shape(from_c(s));
    if (cap < static_cast<int64_t>(f.size()) + 1) invalid_argument("format buffer too small");
    std::memcpy(buf, f.c_str(), f.size() + 1);
  });
}

int tt_shape_check(const tt_shape* s) {
  return guarded([&] { (void)from_c(s); });
}

int tt_shape_external(const tt_shape* s, int64_t* ext_out) {
  return guarded([&] {
    const Shape sh = from_c(s);
    for (int i = 0; i < sh.rank(); ++i) ext_out[i] = sh.ext(i);
  });
}

int64_t tt_shape_tile_count(const tt_shape* s) {
  try {
    return from_c(s).tile_count();
  } catch (...) {
    return -1;
  }
}
int64_t tt_shape_tile_slots(const tt_shape* s) {
  try {
    return from_c(s).tile_slots();
  } catch (...) {
    return -1;
  }
}
int64_t tt_shape_used_slots(const tt_shape* s) {
  try {
    return from_c(s).used_slots();
  } catch (...) {
    return -1;
  }
}

int tt_shape_elementwise_result(const tt_shape* a, const tt_shape* b, int op, tt_shape* out) {
  return guarded([&] { to_c(elementwise_result_shape(from_c(a), from_c(b), op), out); });
}

int tt_shape_sum_result(const tt_shape* s, int dim, tt_shape* out) {
  return guarded([&] { to_c(sum_result_shape(from_c(s), dim), out); });
}

// logical_indices tile_tensor.hpp:96-111
int tt_logical_indices(const tt_shape* s, const int64_t* tile_index, int64_t h, int64_t* j_out) {
  return guarded([&] {
    const Shape sh = from_c(s);
    if (h < 0 || h >= sh.tile_slots()) shape_error("slot index out of range");
    const auto st = tile_strides(sh);
    for (int i = 0; i < sh.rank(); ++i) {
      if (tile_index[i] < 0 || tile_index[i] >= sh.ext(i)) shape_error("tile index out of range");
      const int64_t m = (h / st[i]) % sh.dims[i].t;
      j_out[i] = sh.dims[i].interleaved ? m * sh.ext(i) + tile_index[i]
                                        : tile_index[i] * sh.dims[i].t + m;
    }
  });
}

// slot_of tile_tensor.hpp:114-128
int tt_slot_of(const tt_shape* s, const int64_t* j, int64_t* tile_index_out, int64_t* h_out) {
  return guarded([&] {
    const Shape sh = from_c(s);
    const auto st = tile_strides(sh);
    int64_t h = 0;
    for (int i = 0; i < sh.rank(); ++i) {
      const int64_t t = sh.dims[i].t;
      const int64_t e = sh.ext(i);
      if (j[i] < 0 || j[i] >= e * t) shape_error("logical index out of range");
      if (sh.dims[i].interleaved) {
        tile_index_out[i] = j[i] % e;
        h += (j[i] / e) * st[i];
      } else {
        tile_index_out[i] = j[i] / t;
        h += (j[i] % t) * st[i];
      }
    }
    *h_out = h;
  });
}

int64_t tt_rotations_left_to_right(int64_t n) { return ttb::rotations_left_to_right(n); }
int64_t tt_rotations_right_to_left(int64_t n) { return ttb::rotations_right_to_left(n); }

// ---- session --------------------------------------------------------------------

int tt_device_count(int* out) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) n = 0;
  cudaGetLastError();
  *out = n;
  return TT_OK;
}

int tt_session_create(int64_t slot_count, int64_t max_chain_index, int device, tt_session** out) {
  return guarded([&] {
    *out = nullptr;
    if (slot_count < 1) invalid_argument("slot count must be >= 1");       // backend.hpp:86
    if (max_chain_index < 1) invalid_argument("max chain index must be >= 1");  // :87-88
    if (slot_count >= (int64_t{1} << 31)) invalid_argument("slot count must be < 2^31");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
      cudaGetLastError();
      throw Error(TT_ERR_NO_DEVICE, "no CUDA device: the tile-tensor backend runs only on the GPU");
    }
    if (device < 0 || device >= n) invalid_argument("device ordinal out of range");
    auto* s = new tt_session();
    s->slots = slot_count;
    s->depth = max_chain_index;
    s->device = device;
    try {
      check_cuda(cudaSetDevice(device), "cudaSetDevice");
      check_cuda(cudaStreamCreateWithFlags(&s->own_stream, cudaStreamNonBlocking), "stream");
      s->stream = s->own_stream;
      cudaMemPoolProps props{};
      props.allocType = cudaMemAllocationTypePinned;
      props.handleTypes = cudaMemHandleTypeNone;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = device;
      check_cuda(cudaMemPoolCreate(&s->pool, &props), "memory pool");
      uint64_t keep = ~uint64_t{0};
      check_cuda(cudaMemPoolSetAttribute(s->pool, cudaMemPoolAttrReleaseThreshold, &keep), "pool threshold");
      size_t free_mem = 0, total_mem = 0;
      if (cudaMemGetInfo(&free_mem, &total_mem) == cudaSuccess) s->cache_cap = total_mem / 4;
      cudaDeviceProp prop{};
      check_cuda(cudaGetDeviceProperties(&prop, device), "device properties");
      s->sm_count = prop.multiProcessorCount;
      s->smem_optin = prop.sharedMemPerBlockOptin;
      s->l2_bytes = static_cast<size_t>(prop.l2CacheSize);
      const size_t sched_bytes = (2 * kSchedSlots + kChainSlots * kChainCounters) * sizeof(unsigned int);
      check_cuda(cudaMalloc(&s->sched, sched_bytes), "scheduler counters");
      check_cuda(cudaMemset(s->sched, 0, sched_bytes), "scheduler counters");
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

void tt_session_destroy(tt_session* s) {
  if (!s) return;
  cudaSetDevice(s->device);
  if (s->own_stream) cudaStreamSynchronize(s->own_stream);
  if (s->scratch) cudaFree(s->scratch);
  for (double* p : s->retired) cudaFree(p);
  if (s->sched) cudaFree(s->sched);
  if (s->stream && s->stream != s->own_stream) cudaStreamSynchronize(s->stream);
  for (auto& kv : s->free_blocks)
    for (void* p : kv.second) cudaFree(p);
  for (auto& kv : s->live) cudaFree(kv.first);
  if (s->pool) cudaMemPoolDestroy(s->pool);
  if (s->own_stream) cudaStreamDestroy(s->own_stream);
  delete s;
}

int64_t tt_session_slot_count(const tt_session* s) { return s ? s->slots : -1; }
int64_t tt_session_max_chain_index(const tt_session* s) { return s ? s->depth : -1; }
int tt_session_device(const tt_session* s) { return s ? s->device : -1; }

int tt_session_set_stream(tt_session* s, void* stream) {
  return guarded([&] {
    need_session(s);
    std::lock_guard<std::mutex> lk(s->mu);
    s->stream = static_cast<cudaStream_t>(stream);
  });
}

int tt_session_use_own_stream(tt_session* s) {
  return guarded([&] {
    need_session(s);
    std::lock_guard<std::mutex> lk(s->mu);
    s->stream = s->own_stream;
  });
}

void* tt_session_stream(const tt_session* s) { return s ? s->stream : nullptr; }

int tt_session_synchronize(tt_session* s) {
  return guarded([&] {
    need_session(s);
    check_cuda(cudaSetDevice(s->device), "cudaSetDevice");
    check_cuda(cudaStreamSynchronize(s->stream), "stream synchronize");
  });
}

void tt_session_cost(const tt_session* s, tt_cost* out) {
  std::memset(out, 0, sizeof(*out));
  if (!s) return;
  out->additions = s->adds.load(std::memory_order_relaxed);
  out->multiplications = s->muls.load(std::memory_order_relaxed);
  out->mask_multiplications = s->masks.load(std::memory_order_relaxed);
  out->rotations = s->rots.load(std::memory_order_relaxed);
  out->bootstraps = s->boots.load(std::memory_order_relaxed);
  out->power_of_two_rotations = s->pow2.load(std::memory_order_relaxed);
}

void tt_session_reset_counters(tt_session* s) {
  if (!s) return;
  s->adds = 0;
  s->muls = 0;
  s->masks = 0;
  s->rots = 0;
  s->boots = 0;
  s->pow2 = 0;
}

uint64_t tt_session_launches(const tt_session* s) { return s ? s->launches : 0; }

void tt_session_count_bootstraps(tt_session* s, int64_t count) {
  if (s && count > 0) s->boots += static_cast<uint64_t>(count);
}

// ---- memory -----------------------------------------------------------------------

namespace {
// Blocks handed out by tt_device_alloc / tt_tiles_alloc come from the session's
// stream-ordered pool and, once released, from a free list keyed by (stream,
// bytes): a repeated op of the same shape allocates with no driver call.  (The
// pool alone is not enough: reusing a released 16 GiB block through
// cudaMallocFromPoolAsync measured 27 ms per call on config 5 -- the pool
// re-maps large blocks -- against 5.7 ms for the op itself.)  The cache keeps at
// most a quarter of the device memory; beyond it blocks go back to the pool.
void* cache_take(tt_session* s, size_t nb) {
  auto it = s->free_blocks.find({s->stream, nb});
  if (it == s->free_blocks.end() || it->second.empty()) return nullptr;
  void* p = it->second.back();
  it->second.pop_back();
  s->cached_bytes -= nb;
  return p;
}

// Large blocks outside stream capture come from cudaMalloc: growing the
// stream-ordered pool maps physical memory at ~20 GB/s (a first 16 GiB result
// took 0.8 s), cudaMalloc does it in a few ms.  They are cached like the rest and
// returned with cudaFree only beyond the cache cap or at session end.
constexpr size_t kDirectAllocBytes = size_t{64} << 20;

void* block_alloc(tt_session* s, size_t nb, bool cacheable) {
  void* p = cacheable ? cache_take(s, nb) : nullptr;
  bool direct = false;
  if (!p) {
    check_cuda(cudaSetDevice(s->device), "cudaSetDevice");
    if (cacheable && nb >= kDirectAllocBytes) {
      check_cuda(cudaMalloc(&p, nb), "cudaMalloc");
      direct = true;
    } else {
      check_cuda(cudaMallocFromPoolAsync(&p, nb, s->pool, s->stream), "cudaMallocFromPoolAsync");
    }
  } else {
    direct = s->direct.count(p) != 0;
  }
  if (direct) s->direct.insert(p);
  s->live[p] = {nb, s->stream, cacheable};
  return p;
}

void block_release(tt_session* s, void* p) {
  auto it = s->live.find(p);
  if (it == s->live.end()) invalid_argument("release of a block this session did not allocate");
  const tt_session::CachedBlock b = it->second;
  s->live.erase(it);
  if (b.cacheable && s->cached_bytes + b.bytes <= s->cache_cap) {
    s->free_blocks[{b.stream, b.bytes}].push_back(p);
    s->cached_bytes += b.bytes;
  } else if (s->direct.erase(p)) {
    check_cuda(cudaSetDevice(s->device), "cudaSetDevice");
    check_cuda(cudaStreamSynchronize(b.stream), "stream synchronize");  // its last users
    check_cuda(cudaFree(p), "cudaFree");
  } else {
    check_cuda(cudaSetDevice(s->device), "cudaSetDevice");
    check_cuda(cudaFreeAsync(p, s->stream), "cudaFreeAsync");
  }
}

bool capturing(const tt_session* s) {
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  check_cuda(cudaStreamIsCapturing(s->stream, &cap), "capture status");
  return cap != cudaStreamCaptureStatusNone;
}
}  // namespace

int tt_device_alloc(tt_session* s, int64_t bytes, void** out) {
  return guarded([&] {
    need_session(s);
    *out = nullptr;
    if (bytes <= 0) return;
    std::lock_guard<std::mutex> lk(s->mu);
    // a block allocated under stream capture is graph memory: never cached
    *out = block_alloc(s, static_cast<size_t>(bytes), !capturing(s));
  });
}

int tt_device_free(tt_session* s, void* p) {
  return guarded([&] {
    need_session(s);
    if (!p) return;
    std::lock_guard<std::mutex> lk(s->mu);
    block_release(s, p);
  });
}

int tt_tiles_alloc(tt_session* s, int64_t bytes, void** out) {
  return guarded([&] {
    need_session(s);
    *out = nullptr;
    if (bytes <= 0) bytes = 8;
    std::lock_guard<std::mutex> lk(s->mu);
    // under stream capture the result must live in the capturing framework's
    // graph memory: hand out nothing, the caller allocates it itself
    if (capturing(s)) return;
    *out = block_alloc(s, static_cast<size_t>(bytes), true);
  });
}

int tt_tiles_release(tt_session* s, void* p) {
  return guarded([&] {
    need_session(s);
    if (!p) return;
    std::lock_guard<std::mutex> lk(s->mu);
    block_release(s, p);
  });
}

int tt_copy_h2d(tt_session* s, void* dst, const void* src, int64_t bytes) {
  return guarded([&] {
    need_session(s);
    std::lock_guard<std::mutex> lk(s->mu);
    check_cuda(cudaSetDevice(s->device), "cudaSetDevice");
    if (bytes > 0)
      check_cuda(cudaMemcpyAsync(dst, src, static_cast<size_t>(bytes), cudaMemcpyHostToDevice,
                                 s->stream),
                 "h2d copy");
  });
}

int tt_copy_d2h(tt_session* s, void* dst, const void* src, int64_t bytes) {
  return guarded([&] {
    need_session(s);
    std::lock_guard<std::mutex> lk(s->mu);
    check_cuda(cudaSetDevice(s->device), "cudaSetDevice");
    if (bytes > 0) {
      check_cuda(cudaMemcpyAsync(dst, src, static_cast<size_t>(bytes), cudaMemcpyDeviceToHost,
                                 s->stream),
                 "d2h copy");
      check_cuda(cudaStreamSynchronize(s->stream), "d2h sync");
    }
  });
}

int tt_copy_d2d(tt_session* s, void* dst, const void* src, int64_t bytes) {
  return guarded([&] {
    need_session(s);
    std::lock_guard<std::mutex> lk(s->mu);
    check_cuda(cudaSetDevice(s->device), "cudaSetDevice");
    if (bytes > 0)
      check_cuda(cudaMemcpyAsync(dst, src, static_cast<size_t>(bytes), cudaMemcpyDeviceToDevice,
                                 s->stream),
                 "d2d copy");
  });
}

int tt_fill_uniform(tt_session* s, double* out, int64_t count, uint64_t seed, int64_t offset,
                    double lo, double hi) {
  return guarded([&] {
    need_session(s);
    std::lock_guard<std::mutex> lk(s->mu);
    launch_fill_uniform(ctx_of(s), out, count, seed, offset, lo, hi);
  });
}

// ---- tile-tensor operators ------------------------------------------------------

int tt_pack(tt_session* s, const double* dense, const tt_shape* shape, double* tiles) {
  return guarded([&] {
    need_session(s);
    const Shape sh = from_c(shape);
    if (sh.has_unknown())  // tile_tensor.hpp:169-170
      shape_error("pack target shape may not contain '?': " + format_shape(sh));
    require_slots(s, sh, "pack");
    check_tiles_addressable(sh);
    std::lock_guard<std::mutex> lk(s->mu);
    const LaunchCtx c = ctx_of(s);
    const int path = kernel_path();  // 2 (regs) / 3 (generic) force the gather kernel
    if ((path == 2 || path == 3) || !launch_pack_tma(c, sh, s->slots, dense, tiles))
      launch_pack(c, sh, s->slots, dense, tiles);
  });
}

int tt_unpack(tt_session* s, const tt_shape* shape, const double* tiles, double* dense) {
  return guarded([&] {
    need_session(s);
    const Shape sh = from_c(shape);
    require_slots(s, sh, "unpack");
    check_tiles_addressable(sh);
    std::lock_guard<std::mutex> lk(s->mu);
    const LaunchCtx c = ctx_of(s);
    const int path = kernel_path();
    if ((path == 2 || path == 3) || !launch_unpack_tma(c, sh, s->slots, tiles, dense))
      launch_unpack(c, sh, s->slots, tiles, dense);
  });
}

int tt_elementwise(tt_session* s, int op, const tt_shape* a, const double* ta, int64_t chain_a,
                   const tt_shape* b, const double* tb, int64_t chain_b, tt_shape* out_shape,
                   double* out, int64_t* out_chain) {
  return guarded([&] {
    need_session(s);
    if (op != TT_OP_ADD && op != TT_OP_MUL) invalid_argument("unknown elementwise op");
    const Shape sa = from_c(a), sb = from_c(b);
    const Shape so = elementwise_result_shape(sa, sb, op);
    require_slots(s, sa, "elementwise");
    require_slots(s, sb, "elementwise");
    check_tiles_addressable(so);
    const int64_t chain = op == TT_OP_MUL ? mul_chain(chain_a, chain_b) : std::min(chain_a, chain_b);
    to_c(so, out_shape);
    if (out_chain) *out_chain = chain;
    const uint64_t n = static_cast<uint64_t>(so.tile_count());
    if (op == TT_OP_ADD)
      s->adds += n;
    else
      s->muls += n;
    std::lock_guard<std::mutex> lk(s->mu);
    launch_elementwise(ctx_of(s), op, so, sa, sb, s->slots, ta, tb, out);
  });
}

int tt_sum(tt_session* s, const tt_shape* in_shape, const double* tin, int dim, int variant,
           tt_shape* out_shape, double* out) {
  return guarded([&] {
    need_session(s);
    const Shape sh = from_c(in_shape);
    const Shape so = sum_result_shape(sh, dim);
    require_slots(s, sh, "tt_sum");
    check_tiles_addressable(sh);
    to_c(so, out_shape);
    const int di = dim - 1;
    const Dim& ds = sh.dims[di];
    std::lock_guard<std::mutex> lk(s->mu);
    if (ds.n == 1 && ds.d > 1) {  // degenerate: tiles unchanged (tile_tensor.hpp:295)
      copy_tiles(ctx_of(s), out, tin, sh.tile_count() * s->slots);
      return;
    }
    std::vector<int64_t> st;
    operand_strides(sh, st);
    run_reduction(s, sh, di, variant, tin, st, nullptr, st, out);
  });
}

int tt_mul_sum(tt_session* s, const tt_shape* a, const double* ta, int64_t chain_a,
               const tt_shape* b, const double* tb, int64_t chain_b, int dim, int variant,
               tt_shape* out_shape, double* out, int64_t* out_chain) {
  return guarded([&] {
    need_session(s);
    const Shape sa = from_c(a), sb = from_c(b);
    const Shape prod = elementwise_result_shape(sa, sb, TT_OP_MUL);  // tt_mul
    require_slots(s, sa, "tt_mul");
    require_slots(s, sb, "tt_mul");
    check_tiles_addressable(prod);
    const int64_t chain = mul_chain(chain_a, chain_b);
    const Shape so = sum_result_shape(prod, dim);  // tt_sum
    to_c(so, out_shape);
    if (out_chain) *out_chain = chain;
    s->muls += static_cast<uint64_t>(prod.tile_count());
    std::lock_guard<std::mutex> lk(s->mu);
    const int di = dim - 1;
    const Dim& ds = prod.dims[di];
    if (ds.n == 1 && ds.d > 1) {  // degenerate sum: the product itself
      launch_elementwise(ctx_of(s), TT_OP_MUL, prod, sa, sb, s->slots, ta, tb, out);
      return;
    }
    std::vector<int64_t> ast, bst;
    operand_strides(sa, ast);
    operand_strides(sb, bst);
    run_reduction(s, prod, di, variant, ta, ast, tb, bst, out);
  });
}

int tt_mul_sum_affine(tt_session* s, const tt_shape* a, const double* ta, int64_t chain_a,
                      const tt_shape* b, const double* tb, int64_t chain_b, int dim, int variant,
                      const tt_shape* c, const double* tc, int64_t chain_c, int square,
                      tt_shape* out_shape, double* out, int64_t* out_chain) {
  // Validate the whole composition first; anything the fused pass does not
  // cover (C broadcasting the sum to a larger grid, a depth error at the
  // square, a C from the wrong slot count) runs as the plain composition so
  // that counters and errors match it call for call.
  bool fused = true;
  Shape sa, sb, prod, so, sr;
  int64_t chain1 = 0, chain2 = 0;
  int rc = guarded([&] {
    need_session(s);
    sa = from_c(a);
    sb = from_c(b);
    prod = elementwise_result_shape(sa, sb, TT_OP_MUL);
    require_slots(s, sa, "tt_mul");
    require_slots(s, sb, "tt_mul");
    check_tiles_addressable(prod);
    chain1 = mul_chain(chain_a, chain_b);
    so = sum_result_shape(prod, dim);
  });
  if (rc != TT_OK) return rc;
  sr = so;
  chain2 = chain1;
  if (c != nullptr) {
    try {
      const Shape sc = from_c(c);
      require_slots(s, sc, "elementwise");
      sr = elementwise_result_shape(so, sc, TT_OP_ADD);
      chain2 = std::min(chain1, chain_c);
      if (sr.tile_count() != so.tile_count()) fused = false;
    } catch (const std::exception&) {
      fused = false;
    }
  }
  if (square && chain2 < 1) fused = false;
  if (square && fused) {
    try {
      sr = elementwise_result_shape(sr, sr, TT_OP_MUL);
    } catch (const std::exception&) {
      fused = false;
    }
  }
  if (!fused) {  // the composition, through the public entry points
    void* tmp[2] = {nullptr, nullptr};
    auto alloc_tiles = [&](const tt_shape* sh, int k) {
      return tt_device_alloc(s, std::max<int64_t>(1, tt_shape_tile_count(sh)) * s->slots * 8, &tmp[k]);
    };
    tt_shape cur{}, next{};
    int64_t ch = 0;
    to_c(so, &cur);
    rc = alloc_tiles(&cur, 0);
    if (rc == TT_OK)
      rc = tt_mul_sum(s, a, ta, chain_a, b, tb, chain_b, dim, variant, &cur,
                      static_cast<double*>(tmp[0]), &ch);
    const double* src = static_cast<double*>(tmp[0]);
    if (rc == TT_OK && c != nullptr) {
      rc = tt_shape_elementwise_result(&cur, c, TT_OP_ADD, &next);
      if (rc == TT_OK && square) rc = alloc_tiles(&next, 1);
      double* dst = square ? static_cast<double*>(tmp[1]) : out;
      if (rc == TT_OK)
        rc = tt_elementwise(s, TT_OP_ADD, &cur, src, ch, c, tc, chain_c, &next, dst, &ch);
      src = dst;
      cur = next;
    }
    if (rc == TT_OK) {
      if (square)
        rc = tt_elementwise(s, TT_OP_MUL, &cur, src, ch, &cur, src, ch, out_shape, out, &ch);
      else
        *out_shape = cur;
    }
    if (rc == TT_OK && out_chain) *out_chain = ch;
    const std::string err = g_error;
    const int64_t pos = g_error_pos;
    for (void* t : tmp)
      if (t) tt_device_free(s, t);
    if (rc != TT_OK) set_error(rc, err, pos);
    return rc;
  }
  return guarded([&] {
    to_c(sr, out_shape);
    if (out_chain) *out_chain = square ? chain2 - 1 : chain2;
    s->muls += static_cast<uint64_t>(prod.tile_count());
    std::lock_guard<std::mutex> lk(s->mu);
    Epilogue epi;
    epi.square = square != 0;
    const auto ext = so.external();
    epi.nd = static_cast<int>(ext.size());
    for (int i = 0; i < epi.nd; ++i) epi.ext[i] = ext[i];
    if (c != nullptr) {
      std::vector<int64_t> cst;
      operand_strides(from_c(c), cst);
      epi.c = tc;
      for (int i = 0; i < epi.nd; ++i) epi.c_stride[i] = cst[i];
    }
    const int di = dim - 1;
    const Dim& ds = prod.dims[di];
    if (ds.n == 1 && ds.d > 1) {  // degenerate sum: the product itself, then the tail
      launch_elementwise(ctx_of(s), TT_OP_MUL, prod, sa, sb, s->slots, ta, tb, out);
      launch_epilogue(ctx_of(s), epi, s->slots, out, so.tile_count());
    } else {
      std::vector<int64_t> ast, bst;
      operand_strides(sa, ast);
      operand_strides(sb, bst);
      run_reduction(s, prod, di, variant, ta, ast, tb, bst, out, &epi);
    }
    // the tail's counters: one tt_add and one tt_mul over the result tiles
    if (c != nullptr) s->adds += static_cast<uint64_t>(sr.tile_count());
    if (square) s->muls += static_cast<uint64_t>(sr.tile_count());
  });
}

int tt_mul_sum_clean(tt_session* s, const tt_shape* a, const double* ta, int64_t chain_a,
                     const tt_shape* b, const double* tb, int64_t chain_b, int dim, int variant,
                     tt_shape* out_shape, double* out, int64_t* out_chain) {
  Shape sa, sb, prod, so;
  int64_t chain1 = 0;
  int rc = guarded([&] {
    need_session(s);
    sa = from_c(a);
    sb = from_c(b);
    prod = elementwise_result_shape(sa, sb, TT_OP_MUL);
    require_slots(s, sa, "tt_mul");
    require_slots(s, sb, "tt_mul");
    check_tiles_addressable(prod);
    chain1 = mul_chain(chain_a, chain_b);
    so = sum_result_shape(prod, dim);
  });
  if (rc != TT_OK) return rc;
  if (!so.has_unknown())  // clean_unknowns returns its input as is (tile_tensor.hpp:354)
    return tt_mul_sum(s, a, ta, chain_a, b, tb, chain_b, dim, variant, out_shape, out, out_chain);
  // the mask of clean_unknowns (tile_tensor.hpp:364-378) as a reduction
  // epilogue: cut dims (used < ext * t) need power-of-two extents and strides
  Epilogue epi;
  bool fused = so.has_unknown() && chain1 >= 1 && !so.relaxed;
  const Dim& ds = prod.dims[dim - 1];
  if (ds.n == 1 && ds.d > 1) fused = false;  // degenerate sum: the product itself
  if (fused) {
    const auto ext = so.external();
    const auto tst = tile_strides(so);
    epi.nd = static_cast<int>(ext.size());
    for (int i = 0; i < epi.nd; ++i) epi.ext[i] = ext[i];
    for (int i = 0; i < so.rank() && fused; ++i) {
      const Dim& d = so.dims[i];
      if (d.used() >= ext[i] * d.t) continue;
      const bool pow2 = (d.t & (d.t - 1)) == 0 && (tst[i] & (tst[i] - 1)) == 0;
      if (d.interleaved || !pow2 || epi.nmask == kEpiMaskDims) {
        fused = false;
        break;
      }
      epi.mask_dim[epi.nmask] = i;
      epi.mask_t[epi.nmask] = d.t;
      epi.mask_stride[epi.nmask] = tst[i];
      epi.mask_used[epi.nmask] = d.used();
      ++epi.nmask;
    }
  }
  if (!fused) {  // the composition: product + sum, then clean_unknowns in place
    tt_shape mid{};
    int64_t ch = 0;
    rc = tt_mul_sum(s, a, ta, chain_a, b, tb, chain_b, dim, variant, &mid, out, &ch);
    if (rc != TT_OK) return rc;
    return tt_clean_unknowns(s, &mid, out, ch, out_shape, out, out_chain);
  }
  return guarded([&] {
    s->muls += static_cast<uint64_t>(prod.tile_count());
    {
      std::lock_guard<std::mutex> lk(s->mu);
      std::vector<int64_t> ast, bst;
      operand_strides(sa, ast);
      operand_strides(sb, bst);
      run_reduction(s, prod, dim - 1, variant, ta, ast, tb, bst, out, &epi);
    }
    s->masks += static_cast<uint64_t>(so.tile_count());
    for (auto& d : so.dims) d.unknown = false;
    to_c(so, out_shape);
    if (out_chain) *out_chain = chain1 - 1;
  });
}

int tt_linalg_product(tt_session* s, int which, const tt_shape* a, const double* ta,
                      int64_t chain_a, const tt_shape* b, const double* tb, int64_t chain_b,
                      int variant, tt_shape* out_shape, double* out, int64_t* out_chain) {
  int rc = guarded([&] {
    static const char* names[] = {"matvec_a", "matvec_b", "matmul_a", "matmul_b"};
    if (which < 0 || which > 3) invalid_argument("unknown product form");
    const Shape sa = from_c(a), sb = from_c(b);
    const int rank = which < 2 ? 2 : 3;
    if (sa.rank() != rank || sb.rank() != rank)
      shape_error(std::string(names[which]) + " expects rank-" + std::to_string(rank) +
                  " operands");
    // require_replicated linalg.hpp:32-37
    auto req = [&](const Shape& sh, int d0) {
      const Dim& ds = sh.dims[d0];
      if (!(ds.n == 1 && ds.d == ds.t))
        shape_error(std::string(names[which]) + ": operand dimension " + std::to_string(d0 + 1) +
                    " must be fully replicated, got " + format_shape(sh));
    };
    if (which == 0) req(sb, 0);
    if (which == 1) req(sb, 1);
    if (which == 2) {
      req(sa, 2);
      req(sb, 0);
    }
    if (which == 3) {
      req(sa, 2);
      req(sb, 1);
    }
  });
  if (rc != TT_OK) return rc;
  const int dim = (which == 0 || which == 2) ? 2 : 1;
  return tt_mul_sum(s, a, ta, chain_a, b, tb, chain_b, dim, variant, out_shape, out, out_chain);
}

int tt_linalg_chain2(tt_session* s, int which1, const tt_shape* a1, const double* ta1,
                     int64_t chain_a1, const tt_shape* b1, const double* tb1, int64_t chain_b1,
                     int which2, const tt_shape* x, const double* tx, int64_t chain_x, int r1_pos,
                     int variant, tt_shape* out1_shape, double* out1, int64_t* out1_chain,
                     tt_shape* out2_shape, double* out2, int64_t* out2_chain) {
  // Dry validation of both calls on the host (no launch, no counters): any
  // error -- or a pair the chain kernel does not take -- runs the two calls.
  tt_shape r1{};
  int64_t c1 = 0;
  bool fusable = true;
  {
    const std::string err = g_error;
    const int64_t pos = g_error_pos;
    try {
      need_session(s);
      if (which1 < 0 || which1 > 3 || which2 < 0 || which2 > 3 || (r1_pos != 0 && r1_pos != 1))
        invalid_argument("tt_linalg_chain2: bad product form or operand position");
      const Shape sa = from_c(a1), sb = from_c(b1), sx = from_c(x);
      auto check = [&](int which, const Shape& l, const Shape& r) {
        const int rank = which < 2 ? 2 : 3;
        if (l.rank() != rank || r.rank() != rank) throw std::runtime_error("rank");
        auto req = [](const Shape& sh, int d0) {
          const Dim& ds = sh.dims[d0];
          if (!(ds.n == 1 && ds.d == ds.t)) throw std::runtime_error("replication");
        };
        if (which == 0) req(r, 0);
        if (which == 1) req(r, 1);
        if (which == 2) {
          req(l, 2);
          req(r, 0);
        }
        if (which == 3) {
          req(l, 2);
          req(r, 1);
        }
        require_slots(s, l, "tt_mul");
        require_slots(s, r, "tt_mul");
      };
      check(which1, sa, sb);
      const Shape p1 = elementwise_result_shape(sa, sb, TT_OP_MUL);
      check_tiles_addressable(p1);
      c1 = mul_chain(chain_a1, chain_b1);
      const int dim1 = (which1 == 0 || which1 == 2) ? 2 : 1;
      const Shape s1 = sum_result_shape(p1, dim1);
      to_c(s1, &r1);
      const Shape& l2 = r1_pos ? sx : s1;
      const Shape& rr2 = r1_pos ? s1 : sx;
      check(which2, l2, rr2);
      const Shape p2 = elementwise_result_shape(l2, rr2, TT_OP_MUL);
      check_tiles_addressable(p2);
      (void)mul_chain(r1_pos ? chain_x : c1, r1_pos ? c1 : chain_x);
      (void)sum_result_shape(p2, (which2 == 0 || which2 == 2) ? 2 : 1);
    } catch (const std::exception&) {
      fusable = false;
    }
    g_error = err;
    g_error_pos = pos;
  }
  if (!fusable) {  // the two calls, with their own errors and counters
    tt_shape mid{};
    int64_t ch = 0;
    int rc = tt_linalg_product(s, which1, a1, ta1, chain_a1, b1, tb1, chain_b1, variant, &mid, out1, &ch);
    if (rc != TT_OK) return rc;
    if (out1_shape) *out1_shape = mid;
    if (out1_chain) *out1_chain = ch;
    return r1_pos ? tt_linalg_product(s, which2, x, tx, chain_x, &mid, out1, ch, variant, out2_shape, out2,
                                      out2_chain)
                  : tt_linalg_product(s, which2, &mid, out1, ch, x, tx, chain_x, variant, out2_shape, out2,
                                      out2_chain);
  }
  return guarded([&] {
    const Shape sa = from_c(a1), sb = from_c(b1), sx = from_c(x), s1 = from_c(&r1);
    const int dim1 = (which1 == 0 || which1 == 2) ? 2 : 1;
    const int dim2 = (which2 == 0 || which2 == 2) ? 2 : 1;
    const Shape& l2 = r1_pos ? sx : s1;
    const Shape& rr2 = r1_pos ? s1 : sx;
    std::lock_guard<std::mutex> lk(s->mu);
    PreparedProduct pp[2];
    const bool ok1 = prepare_product(s, sa, sb, dim1, variant, pp[0]);
    const bool ok2 = prepare_product(s, l2, rr2, dim2, variant, pp[1]);
    const LaunchCtx c = ctx_of(s);
    ChainStep steps[2];
    steps[0].prog = pp[0].prog.get();
    steps[0].g = pp[0].g;
    steps[0].ta = ta1;
    steps[0].tb = tb1;
    steps[0].tout = out1;
    steps[1].prog = pp[1].prog.get();
    steps[1].g = pp[1].g;
    steps[1].ta = r1_pos ? tx : out1;
    steps[1].tb = r1_pos ? out1 : tx;
    steps[1].tout = out2;
    if (!(ok1 && ok2 && launch_chain(c, steps, 2, s->slots))) {
      // not fusable after all: the two reductions back to back (same kernels
      // the separate calls launch)
      auto one = [&](const Shape& l, const Shape& r, int dim, const double* tl, const double* tr,
                     double* o) {
        const Shape prod = elementwise_result_shape(l, r, TT_OP_MUL);
        const Dim& ds = prod.dims[dim - 1];
        if (ds.n == 1 && ds.d > 1) {
          launch_elementwise(c, TT_OP_MUL, prod, l, r, s->slots, tl, tr, o);
          return;
        }
        std::vector<int64_t> ast, bst;
        operand_strides(l, ast);
        operand_strides(r, bst);
        run_reduction(s, prod, dim - 1, variant, tl, ast, tr, bst, o);
      };
      one(sa, sb, dim1, ta1, tb1, out1);
      one(l2, rr2, dim2, steps[1].ta, steps[1].tb, out2);
    } else {
      add_cost(s, pp[0].prog->per_group, static_cast<uint64_t>(pp[0].g.groups));
      add_cost(s, pp[1].prog->per_group, static_cast<uint64_t>(pp[1].g.groups));
    }
    s->muls += static_cast<uint64_t>(pp[0].prod.tile_count() + pp[1].prod.tile_count());
    if (out1_shape) *out1_shape = r1;
    if (out1_chain) *out1_chain = c1;
    const int64_t c2 = std::min(r1_pos ? chain_x : c1, r1_pos ? c1 : chain_x) - 1;
    to_c(sum_result_shape(elementwise_result_shape(l2, rr2, TT_OP_MUL), dim2), out2_shape);
    if (out2_chain) *out2_chain = c2;
  });
}

int tt_clean_unknowns(tt_session* s, const tt_shape* in_shape, const double* tin, int64_t chain,
                      tt_shape* out_shape, double* out, int64_t* out_chain) {
  return guarded([&] {
    need_session(s);
    Shape sh = from_c(in_shape);
    require_slots(s, sh, "clean_unknowns");
    check_tiles_addressable(sh);
    std::lock_guard<std::mutex> lk(s->mu);
    if (!sh.has_unknown()) {  // tile_tensor.hpp:354: returned as is, zero cost
      to_c(sh, out_shape);
      if (out_chain) *out_chain = chain;
      copy_tiles(ctx_of(s), out, tin, sh.tile_count() * s->slots);
      return;
    }
    if (chain < 1)  // backend.hpp:142-143
      depth_error("plaintext multiplication at chain index 0 (bootstrap required)");
    const LaunchCtx c = ctx_of(s);
    launch_clean(c, sh, s->slots, tin, out);
    s->masks += static_cast<uint64_t>(sh.tile_count());
    for (auto& d : sh.dims) d.unknown = false;
    to_c(sh, out_shape);
    if (out_chain) *out_chain = chain - 1;
  });
}

int tt_replicate_dim(tt_session* s, const tt_shape* in_shape, const double* tin, int dim,
                     tt_shape* out_shape, double* out) {
  return guarded([&] {
    need_session(s);
    Shape sh = from_c(in_shape);
    if (dim < 1 || dim > sh.rank()) shape_error("replicate dimension out of range");
    const int di = dim - 1;
    const Dim ds = sh.dims[di];
    if (ds.unknown)
      shape_error("replicate_dim requires a clean dimension (run clean_unknowns first)");
    if (ds.n != 1 || ds.d != 1)
      shape_error("replicate_dim requires a degenerate dimension (n=1, d=1)");
    if (sh.relaxed) shape_error("replicate_dim is not defined for relaxed shapes");
    require_slots(s, sh, "replicate_dim");
    check_tiles_addressable(sh);
    std::lock_guard<std::mutex> lk(s->mu);
    if (ds.t == 1) {
      to_c(sh, out_shape);
      copy_tiles(ctx_of(s), out, tin, sh.tile_count() * s->slots);
      return;
    }
    const int64_t stride = tile_strides(sh)[di];
    const Program prog = build_replicate_program(ds.t, stride, s->slots);
    GroupSpec g;
    g.nd = 1;
    g.ext[0] = sh.tile_count();
    g.out_stride[0] = 1;
    g.a_stride[0] = 1;
    g.groups = sh.tile_count();
    add_cost(s, prog.per_group, static_cast<uint64_t>(g.groups));
    launch_group_program(ctx_of(s), prog, g, s->slots, tin, nullptr, out);
    sh.dims[di].d = ds.t;
    sh.dims[di].interleaved = false;
    to_c(sh, out_shape);
  });
}

// ---- tile-level primitives ----------------------------------------------------------

int tt_tiles_binary(tt_session* s, int op, const double* a, const double* b, double* out,
                    int64_t n_tiles, const int64_t* chain_a, const int64_t* chain_b,
                    int64_t* chain_out) {
  return guarded([&] {
    need_session(s);
    if (op != TT_OP_ADD && op != TT_OP_MUL) invalid_argument("unknown elementwise op");
    if (chain_a && chain_b) {
      for (int64_t i = 0; i < n_tiles; ++i) {
        const int64_t c = op == TT_OP_MUL ? mul_chain(chain_a[i], chain_b[i])
                                          : std::min(chain_a[i], chain_b[i]);
        if (chain_out) chain_out[i] = c;
      }
    }
    if (op == TT_OP_ADD)
      s->adds += static_cast<uint64_t>(n_tiles);
    else
      s->muls += static_cast<uint64_t>(n_tiles);
    std::lock_guard<std::mutex> lk(s->mu);
    launch_binary_flat(ctx_of(s), op, a, b, out, n_tiles * s->slots);
  });
}

namespace {
// product (or a alone) and the checks shared by tt_mul_fold / tt_fold_shape
Shape fold_product(const tt_shape* a, const tt_shape* b, int dim, int& di) {
  const Shape sa = from_c(a);
  const Shape prod = b ? elementwise_result_shape(sa, from_c(b), TT_OP_MUL) : sa;
  if (dim < 1 || dim > prod.rank()) shape_error("sum dimension out of range");
  di = dim - 1;
  const Dim& ds = prod.dims[di];
  if (ds.n == 1 && ds.d > 1) invalid_argument("fold chains need a non-degenerate summed dim");
  if (ds.interleaved) invalid_argument("fold chains do not take an interleaved (~) summed dim");
  if (ds.unknown && ds.used() % ds.t != 0)
    invalid_argument("fold chains do not take a '?' boundary split (clean_unknowns first)");
  return prod;
}
}  // namespace

int tt_fold_shape(const tt_shape* a, const tt_shape* b, int dim, tt_shape* out) {
  return guarded([&] {
    int di = 0;
    Shape prod = fold_product(a, b, dim, di);
    prod.dims[di].n = prod.dims[di].t;
    prod.dims[di].d = 1;
    to_c(prod, out);
  });
}

int tt_mul_fold(tt_session* s, const tt_shape* a, const double* ta, int64_t chain_a,
                const tt_shape* b, const double* tb, int64_t chain_b, int dim,
                int64_t out_begin, int64_t out_end, const double* init, double* acc,
                int64_t* out_chain) {
  return guarded([&] {
    need_session(s);
    if ((b == nullptr) != (tb == nullptr)) invalid_argument("operand b and its tiles go together");
    int di = 0;
    const Shape prod = fold_product(a, b, dim, di);
    const Shape sa = from_c(a);
    require_slots(s, sa, "tt_mul_fold");
    if (b) require_slots(s, from_c(b), "tt_mul_fold");
    check_tiles_addressable(prod);
    const auto ext = prod.external();
    std::vector<int64_t> gext = ext;
    gext[di] = 1;
    int64_t n_out = 1;
    for (auto e : gext) n_out *= e;
    if (out_begin < 0 || out_end > n_out || out_begin > out_end)
      invalid_argument("output tile range out of bounds");
    const int64_t chain = b ? mul_chain(chain_a, chain_b) : chain_a;
    if (out_chain) *out_chain = chain;
    const int64_t tiles = out_end - out_begin, count = ext[di];
    if (b) s->muls += static_cast<uint64_t>(tiles * count);
    s->adds += static_cast<uint64_t>(tiles * (count - (init ? 0 : 1)));
    std::vector<int64_t> ast, bst;
    operand_strides(sa, ast);
    if (b) operand_strides(from_c(b), bst);
    FoldRange fr;
    fr.rank = prod.rank();
    for (int i = 0; i < fr.rank; ++i) {
      fr.gext[i] = gext[i];
      fr.a_stride[i] = i == di ? 0 : ast[i];
      fr.b_stride[i] = b && i != di ? bst[i] : 0;
    }
    fr.astep = ast[di];
    fr.bstep = b ? bst[di] : 0;
    fr.first = 0;
    fr.count = count;
    std::lock_guard<std::mutex> lk(s->mu);
    launch_fold_range(ctx_of(s), fr, s->slots, out_begin, out_end, ta, tb, init, acc);
  });
}

int tt_batch_affine(tt_session* s, const double* in, int64_t n_in, int64_t n_out,
                    const int64_t* row_ptr, const int64_t* src, const double* w,
                    const double* bias, double* out, int64_t chain_in, int64_t* chain_out) {
  return guarded([&] {
    need_session(s);
    if (n_in < 0 || n_out < 0) invalid_argument("negative tile count");
    if (n_out > 0 && (!row_ptr || !bias)) invalid_argument("null layer arrays");
    if (n_out > 0 && row_ptr[0] != 0) invalid_argument("row_ptr must start at 0");
    for (int64_t o = 0; o < n_out; ++o)
      if (row_ptr[o + 1] < row_ptr[o]) invalid_argument("row_ptr must be non-decreasing");
    const int64_t nnz = n_out > 0 ? row_ptr[n_out] : 0;
    if (nnz > 0 && (!src || !w)) invalid_argument("null tap arrays");
    for (int64_t k = 0; k < nnz; ++k)
      if (src[k] < 0 || src[k] >= n_in) invalid_argument("tap source tile out of range");
    if (n_in > 0 && n_out > 0 && in && out && out < in + n_in * s->slots && in < out + n_out * s->slots)
      invalid_argument("batch affine output must not overlap its input");
    if (nnz > 0 && chain_in < 1)
      depth_error("multiplication at chain index 0 (bootstrap required)");
    if (chain_out) *chain_out = nnz > 0 ? chain_in - 1 : s->depth;
    s->muls += static_cast<uint64_t>(nnz);
    s->adds += static_cast<uint64_t>(nnz);
    if (n_out == 0) return;
    std::lock_guard<std::mutex> lk(s->mu);
    const LaunchCtx c = ctx_of(s);
    // stage the plaintext layer description in session scratch (stream-ordered)
    const size_t b_rp = static_cast<size_t>(n_out + 1) * sizeof(int64_t);
    const size_t b_src = static_cast<size_t>(nnz) * sizeof(int64_t);
    const size_t b_w = static_cast<size_t>(nnz) * sizeof(double);
    const size_t b_bias = static_cast<size_t>(n_out) * sizeof(double);
    auto* base = reinterpret_cast<unsigned char*>(scratch_fn(s, b_rp + b_src + b_w + b_bias));
    auto* d_rp = reinterpret_cast<int64_t*>(base);
    auto* d_src = reinterpret_cast<int64_t*>(base + b_rp);
    auto* d_w = reinterpret_cast<double*>(base + b_rp + b_src);
    auto* d_bias = reinterpret_cast<double*>(base + b_rp + b_src + b_w);
    check_cuda(cudaMemcpyAsync(d_rp, row_ptr, b_rp, cudaMemcpyHostToDevice, c.stream), "layer upload");
    if (nnz > 0) {
      check_cuda(cudaMemcpyAsync(d_src, src, b_src, cudaMemcpyHostToDevice, c.stream), "layer upload");
      check_cuda(cudaMemcpyAsync(d_w, w, b_w, cudaMemcpyHostToDevice, c.stream), "layer upload");
    }
    check_cuda(cudaMemcpyAsync(d_bias, bias, b_bias, cudaMemcpyHostToDevice, c.stream), "layer upload");
    // largest block (<= 8) of consecutive rows sharing one source list
    int block = 1;
    for (int cand : {8, 5, 4, 2}) {
      bool ok = true;
      for (int64_t o0 = 0; o0 < n_out && ok; o0 += cand) {
        const int64_t len = row_ptr[o0 + 1] - row_ptr[o0];
        for (int64_t r = o0 + 1; r < std::min<int64_t>(o0 + cand, n_out) && ok; ++r)
          ok = row_ptr[r + 1] - row_ptr[r] == len &&
               std::equal(src + row_ptr[r], src + row_ptr[r] + len, src + row_ptr[o0]);
      }
      if (ok) {
        block = cand;
        break;
      }
    }
    launch_batch_affine(c, in, s->slots, n_out, d_rp, d_src, d_w, d_bias, out, block);
  });
}

}  // extern "C"

struct tt_affine_layer {
  int device = 0;
  int64_t n_in = 0, n_out = 0, nnz = 0;
  int block = 1;
  unsigned char* dev = nullptr;  // row_ptr | src | w | bias
  const int64_t* d_rp = nullptr;
  const int64_t* d_src = nullptr;
  const double* d_w = nullptr;
  const double* d_bias = nullptr;
};

namespace {

void check_affine_layer(int64_t n_in, int64_t n_out, const int64_t* row_ptr, const int64_t* src,
                        const double* w, const double* bias) {
  if (n_in < 0 || n_out < 0) invalid_argument("negative tile count");
  if (n_out > 0 && (!row_ptr || !bias)) invalid_argument("null layer arrays");
  if (n_out > 0 && row_ptr[0] != 0) invalid_argument("row_ptr must start at 0");
  for (int64_t o = 0; o < n_out; ++o)
    if (row_ptr[o + 1] < row_ptr[o]) invalid_argument("row_ptr must be non-decreasing");
  const int64_t nnz = n_out > 0 ? row_ptr[n_out] : 0;
  if (nnz > 0 && (!src || !w)) invalid_argument("null tap arrays");
  for (int64_t k = 0; k < nnz; ++k)
    if (src[k] < 0 || src[k] >= n_in) invalid_argument("tap source tile out of range");
}

// largest block (<= 8) of consecutive rows sharing one source list
int affine_block(int64_t n_out, const int64_t* row_ptr, const int64_t* src) {
  for (int cand : {8, 5, 4, 2}) {
    bool ok = true;
    for (int64_t o0 = 0; o0 < n_out && ok; o0 += cand) {
      const int64_t len = row_ptr[o0 + 1] - row_ptr[o0];
      for (int64_t r = o0 + 1; r < std::min<int64_t>(o0 + cand, n_out) && ok; ++r)
        ok = row_ptr[r + 1] - row_ptr[r] == len &&
             std::equal(src + row_ptr[r], src + row_ptr[r] + len, src + row_ptr[o0]);
    }
    if (ok) return cand;
  }
  return 1;
}

}  // namespace

extern "C" {

int tt_affine_layer_create(tt_session* s, int64_t n_in, int64_t n_out, const int64_t* row_ptr,
                           const int64_t* src, const double* w, const double* bias,
                           tt_affine_layer** out) {
  return guarded([&] {
    need_session(s);
    if (!out) invalid_argument("null layer handle");
    check_affine_layer(n_in, n_out, row_ptr, src, w, bias);
    auto* L = new tt_affine_layer;
    L->device = s->device;
    L->n_in = n_in;
    L->n_out = n_out;
    L->nnz = n_out > 0 ? row_ptr[n_out] : 0;
    if (n_out > 0) {
      L->block = affine_block(n_out, row_ptr, src);
      const size_t b_rp = static_cast<size_t>(n_out + 1) * sizeof(int64_t);
      const size_t b_src = static_cast<size_t>(L->nnz) * sizeof(int64_t);
      const size_t b_w = static_cast<size_t>(L->nnz) * sizeof(double);
      const size_t b_bias = static_cast<size_t>(n_out) * sizeof(double);
      try {
        check_cuda(cudaSetDevice(s->device), "cudaSetDevice");
        check_cuda(cudaMalloc(&L->dev, b_rp + b_src + b_w + b_bias), "layer allocation");
        L->d_rp = reinterpret_cast<const int64_t*>(L->dev);
        L->d_src = reinterpret_cast<const int64_t*>(L->dev + b_rp);
        L->d_w = reinterpret_cast<const double*>(L->dev + b_rp + b_src);
        L->d_bias = reinterpret_cast<const double*>(L->dev + b_rp + b_src + b_w);
        check_cuda(cudaMemcpy(L->dev, row_ptr, b_rp, cudaMemcpyHostToDevice), "layer upload");
        if (L->nnz > 0) {
          check_cuda(cudaMemcpy(L->dev + b_rp, src, b_src, cudaMemcpyHostToDevice), "layer upload");
          check_cuda(cudaMemcpy(L->dev + b_rp + b_src, w, b_w, cudaMemcpyHostToDevice), "layer upload");
        }
        check_cuda(cudaMemcpy(L->dev + b_rp + b_src + b_w, bias, b_bias, cudaMemcpyHostToDevice),
                   "layer upload");
      } catch (...) {
        if (L->dev) cudaFree(L->dev);
        delete L;
        throw;
      }
    }
    *out = L;
  });
}

int tt_affine_layer_apply(tt_session* s, const tt_affine_layer* L, const double* in, double* out,
                          int64_t chain_in, int64_t* chain_out) {
  return guarded([&] {
    need_session(s);
    if (!L) invalid_argument("null layer");
    if (L->device != s->device) invalid_argument("layer belongs to another device");
    if (L->n_in > 0 && L->n_out > 0 && in && out && out < in + L->n_in * s->slots &&
        in < out + L->n_out * s->slots)
      invalid_argument("batch affine output must not overlap its input");
    if (L->nnz > 0 && chain_in < 1) depth_error("multiplication at chain index 0 (bootstrap required)");
    if (chain_out) *chain_out = L->nnz > 0 ? chain_in - 1 : s->depth;
    s->muls += static_cast<uint64_t>(L->nnz);
    s->adds += static_cast<uint64_t>(L->nnz);
    if (L->n_out == 0) return;
    std::lock_guard<std::mutex> lk(s->mu);
    launch_batch_affine(ctx_of(s), in, s->slots, L->n_out, L->d_rp, L->d_src, L->d_w, L->d_bias, out,
                        L->block);
  });
}

void tt_affine_layer_destroy(tt_session* s, tt_affine_layer* L) {
  if (!L) return;
  if (s && s->stream) cudaStreamSynchronize(s->stream);
  if (L->dev) cudaFree(L->dev);
  delete L;
}

int tt_tiles_mask_mul(tt_session* s, const double* a, const double* mask, double* out,
                      int64_t n_tiles, const int64_t* chain_a, int64_t* chain_out) {
  return guarded([&] {
    need_session(s);
    if (chain_a) {
      for (int64_t i = 0; i < n_tiles; ++i) {
        if (chain_a[i] < 1)
          depth_error("plaintext multiplication at chain index 0 (bootstrap required)");
        if (chain_out) chain_out[i] = chain_a[i] - 1;
      }
    }
    s->masks += static_cast<uint64_t>(n_tiles);
    std::lock_guard<std::mutex> lk(s->mu);
    launch_binary_flat(ctx_of(s), TT_OP_MUL, a, mask, out, n_tiles * s->slots);
  });
}

int tt_tiles_rotate(tt_session* s, const double* in, int64_t offset, double* out,
                    int64_t n_tiles) {
  return guarded([&] {
    need_session(s);
    const int64_t sl = s->slots;
    const int64_t r = ((offset % sl) + sl) % sl;  // backend.hpp:155
    std::lock_guard<std::mutex> lk(s->mu);
    const LaunchCtx c = ctx_of(s);
    if (r == 0) {  // free and uncounted (backend.hpp:156)
      copy_tiles(c, out, in, n_tiles * sl);
      return;
    }
    if (in == out) invalid_argument("rotate cannot run in place");
    s->rots += static_cast<uint64_t>(n_tiles);
    if ((r & (r - 1)) == 0) s->pow2 += static_cast<uint64_t>(n_tiles);
    launch_rotate(c, in, out, sl, r, n_tiles);
  });
}

namespace {
int run_tile_program(tt_session* s, const Program& prog, const double* in, double* out,
                     int64_t n_tiles) {
  GroupSpec g;
  g.nd = 1;
  g.ext[0] = n_tiles;
  g.out_stride[0] = 1;
  g.a_stride[0] = 1;
  g.groups = n_tiles;
  add_cost(s, prog.per_group, static_cast<uint64_t>(n_tiles));
  launch_group_program(ctx_of(s), prog, g, s->slots, in, nullptr, out);
  return TT_OK;
}
}  // namespace

int tt_sum_tile_strided(tt_session* s, const double* in, int64_t n, int64_t stride, int variant,
                        double* out, int64_t n_tiles) {
  return guarded([&] {
    need_session(s);
    const Program prog = build_strided_program(n, stride, s->slots, variant);
    std::lock_guard<std::mutex> lk(s->mu);
    if (n == 1) {
      copy_tiles(ctx_of(s), out, in, n_tiles * s->slots);
      return;
    }
    run_tile_program(s, prog, in, out, n_tiles);
  });
}

int tt_sum_tile_dim(tt_session* s, const double* in, const int64_t* tile_extents, int rank,
                    int dim, int variant, double* out, int64_t n_tiles) {
  return guarded([&] {
    need_session(s);
    if (dim < 1 || dim > rank) invalid_argument("tile dimension out of range");
    int64_t stride = 1;
    for (int x = dim; x < rank; ++x) stride *= tile_extents[x];
    const int64_t n = tile_extents[dim - 1];
    std::lock_guard<std::mutex> lk(s->mu);
    if (n == 1) {
      copy_tiles(ctx_of(s), out, in, n_tiles * s->slots);
      return;
    }
    run_tile_program(s, build_strided_program(n, stride, s->slots, variant), in, out, n_tiles);
  });
}

int tt_replicate_tile_dim(tt_session* s, const double* in, const int64_t* tile_extents, int rank,
                          int dim, double* out, int64_t n_tiles) {
  return guarded([&] {
    need_session(s);
    if (dim < 1 || dim > rank) invalid_argument("tile dimension out of range");
    int64_t stride = 1;
    for (int x = dim; x < rank; ++x) stride *= tile_extents[x];
    const int64_t t = tile_extents[dim - 1];
    std::lock_guard<std::mutex> lk(s->mu);
    if (t == 1) {
      copy_tiles(ctx_of(s), out, in, n_tiles * s->slots);
      return;
    }
    run_tile_program(s, build_replicate_program(t, stride, s->slots), in, out, n_tiles);
  });
}

// ---- diagnostics --------------------------------------------------------------------

int tt_set_kernel_path(int path) {
  return guarded([&] {
    if (path < 0 || path > 4) invalid_argument("kernel path must be 0..4");
    set_kernel_path(path);
  });
}

int tt_kernel_path(void) { return kernel_path(); }

int tt_set_chain_kernel(int on) {
  set_chain_kernel(on);
  return TT_OK;
}
int tt_chain_kernel(void) { return chain_kernel_enabled(); }

// ---- sharding ---------------------------------------------------------------------

int tt_shard_plan(const tt_shape* shape, int shard_dim, int world, int rank, int64_t* begin,
                  int64_t* end, tt_shape* local_shape) {
  return guarded([&] {
    Shape sh = from_c(shape);
    if (shard_dim < 1 || shard_dim > sh.rank()) shape_error("shard dimension out of range");
    if (world < 1 || rank < 0 || rank >= world) invalid_argument("bad rank/world");
    const int di = shard_dim - 1;
    Dim& d = sh.dims[di];
    if (d.interleaved) shape_error("interleaved dimensions cannot be block-sharded");
    if (d.n == 1 && d.d > 1) shape_error("replicated dimensions are not sharded");
    const int64_t e = sh.ext(di);
    const int64_t b = e * rank / world, en = e * (rank + 1) / world;
    *begin = b;
    *end = en;
    const int64_t lo = b * d.t;
    const int64_t hi = std::min(d.used(), en * d.t);
    d.n = std::max<int64_t>(hi - lo, 0);
    if (d.n == 0) d.n = 1;  // an empty rank still carries a valid shape
    to_c(sh, local_shape);
  });
}

}  // extern "C"
