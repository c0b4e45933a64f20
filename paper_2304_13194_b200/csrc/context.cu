// context.cu — jet_ctx lifetime, error reporting and launch profiling.
#include "common.cuh"
#include "comm.cuh"
#include <algorithm>
#include <cstdlib>
#include <cstdlib>
#include <cstring>
#include <mutex>

namespace jet {

static thread_local std::string g_last_error;

void set_last_error(const std::string& s) { g_last_error = s; }

int resident_blocks(const void* kern, int block, size_t smem) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, size_t>, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(kern, block, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, block, smem));
  if (per_sm < 1) per_sm = 1;
  cache.emplace(key, per_sm);
  return per_sm;
}

void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
  cudaGetLastError();
  std::string m = std::string("CUDA error '") + cudaGetErrorString(e) + "' in " +
                  what + " at " + file + ":" + std::to_string(line);
  throw Error(e == cudaErrorMemoryAllocation ? JET_ENOMEM : JET_ECUDA, m);
}

cudaEvent_t Ctx::take_event() {
  if (!event_pool.empty()) {
    cudaEvent_t e = event_pool.back();
    event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  CK(cudaEventCreate(&e));
  return e;
}

int Ctx::prof_class(const char* name) {
  auto it = cls_index.find(name);
  if (it != cls_index.end()) return it->second;
  int id = (int)agg.size();
  cls_index[name] = id;
  ProfAgg a;
  a.name = name;
  agg.push_back(a);
  return id;
}

// Resolve pending event pairs into per-class totals.
void Ctx::flush_prof() {
  if (recs.empty()) return;
  CK(cudaStreamSynchronize(stream));
  for (auto& r : recs) {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, r.a, r.b));
    ProfAgg& a = agg[r.cls];
    a.launches++;
    a.ms += ms;
    a.bytes += r.bytes;
    event_pool.push_back(r.a);
    event_pool.push_back(r.b);
  }
  recs.clear();
}

void Ctx::ensure_pinned(size_t elems) {
  if (elems <= pinned_elems) return;
  if (pinned) cudaFreeHost(pinned);
  pinned = nullptr;
  size_t want = elems < 4096 ? 4096 : elems;
  CK(cudaMallocHost((void**)&pinned, want * sizeof(int64_t)));
  pinned_elems = want;
}

static std::mutex g_pool_mu;
static cudaMemPool_t g_pool[64];
static int g_pool_users[64];

static cudaMemPool_t pool_for(int dev) {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (!g_pool[dev]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    CK(cudaMemPoolCreate(&g_pool[dev], &props));
    uint64_t thr = ~0ULL;
    CK(cudaMemPoolSetAttribute(g_pool[dev], cudaMemPoolAttrReleaseThreshold, &thr));
  }
  return g_pool[dev];
}

cudaMemPool_t current_pool() {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  return pool_for(dev);
}

void pool_context_opened(int dev) {
  pool_for(dev);
  std::lock_guard<std::mutex> lk(g_pool_mu);
  ++g_pool_users[dev];
}

// The last context on a device gives the pool's memory back to the driver.
void pool_context_closed(int dev) {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (--g_pool_users[dev] == 0 && g_pool[dev]) {
    cudaDeviceSynchronize();
    cudaMemPoolTrimTo(g_pool[dev], 0);
  }
}

// Grow the device pool's reservation to `bytes` (one allocation, freed back to
// the pool, whose release threshold keeps it mapped).
void Ctx::reserve_pool(size_t bytes) {
  if (bytes <= pool_reserved) return;
  void* p = nullptr;
  if (cudaMallocFromPoolAsync(&p, bytes, current_pool(), stream) == cudaSuccess) {
    cudaFreeAsync(p, stream);
    cudaStreamSynchronize(stream);
    pool_reserved = bytes;
  } else {
    cudaGetLastError();
  }
}

void Ctx::ensure_upload_ring() {
  if (up_host[0]) return;
  for (int b = 0; b < UPLOAD_BUFS; ++b) {
    CK(cudaMallocHost(&up_host[b], UPLOAD_CHUNK));
    CK(cudaEventCreateWithFlags(&up_ev[b], cudaEventDisableTiming));
    CK(cudaEventRecord(up_ev[b], stream));
  }
  up_dev.alloc((size_t)UPLOAD_BUFS * UPLOAD_CHUNK, stream);
}

void Ctx::ensure_pinned_up(size_t bytes) {
  if (bytes <= pinned_up_bytes) return;
  if (pinned_up) cudaFreeHost(pinned_up);
  pinned_up = nullptr;
  size_t want = bytes < (1 << 20) ? (1 << 20) : bytes * 2;
  CK(cudaMallocHost((void**)&pinned_up, want));
  pinned_up_bytes = want;
}

}  // namespace jet

using namespace jet;

static void ctx_teardown(Ctx* c) {
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  c->cub_tmp.release();
  c->flush_buf.release();
  c->level_ext.reset();
  delete c->comm;
  c->comm = nullptr;
  for (auto& b : c->scratch_slots) b.release();
  if (c->timer_a) cudaEventDestroy(c->timer_a);
  if (c->timer_b) cudaEventDestroy(c->timer_b);
  for (auto& r : c->recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto e : c->event_pool) cudaEventDestroy(e);
  if (c->pinned) cudaFreeHost(c->pinned);
  if (c->pinned_up) cudaFreeHost(c->pinned_up);
  c->up_dev.release();
  for (int b = 0; b < Ctx::UPLOAD_BUFS; ++b) {
    if (c->up_host[b]) cudaFreeHost(c->up_host[b]);
    if (c->up_ev[b]) cudaEventDestroy(c->up_ev[b]);
  }
  cudaStreamSynchronize(c->stream);
  cudaStreamDestroy(c->stream);
  const int dev = c->device;
  delete c;
  pool_context_closed(dev);
}

namespace jet {
void ctx_retain(Ctx* c) { c->refs.fetch_add(1); }
void ctx_release(Ctx* c) {
  if (c && c->refs.fetch_sub(1) == 1) ctx_teardown(c);
}
}  // namespace jet

extern "C" {

const char* jet_last_error(void) { return g_last_error.c_str(); }
int jet_api_version(void) { return JET_API_VERSION; }

int jet_create(int device, jet_ctx** out) {
  try {
    JET_REQUIRE(out, JET_EINVAL, "out is NULL");
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    JET_REQUIRE(device >= 0 && device < ndev, JET_EINVAL,
                "device index out of range");
    // the pipeline synchronises with the device at a few hundred points per
    // partition (level sizes, matching rounds): spin rather than yield, so a
    // busy host does not stretch each wait (no effect, and ignored, when the
    // device's context already exists)
    CK(cudaSetDevice(device));
    // opt-in (JET_SPIN=1): the flag applies to the whole process's primary
    // context, so the library does not set it unasked
    if (const char* e = getenv("JET_SPIN"); e && e[0] == '1')
      if (cudaSetDeviceFlags(cudaDeviceScheduleSpin) != cudaSuccess) (void)cudaGetLastError();
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    JET_REQUIRE(prop.major >= 10, JET_EUNSUPPORTED,
                std::string("this build targets sm_100a (B200); found ") + prop.name);
    Ctx* c = new Ctx();
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    c->max_smem_optin = (int)prop.sharedMemPerBlockOptin;
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    pool_context_opened(device);
    // Optional up-front reservation in the private pool (JET_POOL_RESERVE_MB):
    // growing the pool inside a partition (mapping new memory) stalled the
    // host for 100s of ms on dense coarse levels of large graphs; the pool
    // is trimmed when the device's last context is destroyed.
    if (const char* e = getenv("JET_POOL_RESERVE_MB")) c->reserve_pool((size_t)atoll(e) << 20);
    c->ensure_pinned(1 << 16);
    const char* hl = getenv("JET_HOST_LEVELS");
    c->host_levels = hl && hl[0] == '1';
    *out = reinterpret_cast<jet_ctx*>(c);
    return JET_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return JET_EINTERNAL;
  }
}

void jet_destroy(jet_ctx* ctx) {
  if (!ctx) return;
  jet::ctx_release(reinterpret_cast<Ctx*>(ctx));
}

int jet_synchronize(jet_ctx* ctx) {
  try {
    Ctx* c = reinterpret_cast<Ctx*>(ctx);
    c->sync();
    return JET_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  }
}

int jet_profile_enable(jet_ctx* ctx, int on) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  c->prof = on != 0;
  return JET_OK;
}

int jet_profile_filter(jet_ctx* ctx, const char* name) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  std::string s = name ? name : "";
  // "@levels" switches on per-level class names instead of filtering
  c->prof_by_level = s == "@levels";
  c->prof_only = c->prof_by_level ? "" : s;
  return JET_OK;
}

int jet_timer_start(jet_ctx* ctx) {
  try {
    Ctx* c = reinterpret_cast<Ctx*>(ctx);
    CK(cudaSetDevice(c->device));
    if (!c->timer_a) {
      CK(cudaEventCreate(&c->timer_a));
      CK(cudaEventCreate(&c->timer_b));
    }
    CK(cudaEventRecord(c->timer_a, c->stream));
    return JET_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  }
}

int jet_timer_stop(jet_ctx* ctx, double* ms) {
  try {
    Ctx* c = reinterpret_cast<Ctx*>(ctx);
    JET_REQUIRE(c->timer_a, JET_EINVAL, "timer not started");
    CK(cudaEventRecord(c->timer_b, c->stream));
    CK(cudaEventSynchronize(c->timer_b));
    float f = 0;
    CK(cudaEventElapsedTime(&f, c->timer_a, c->timer_b));
    *ms = f;
    return JET_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  }
}

int jet_flush_l2(jet_ctx* ctx) {
  try {
    Ctx* c = reinterpret_cast<Ctx*>(ctx);
    CK(cudaSetDevice(c->device));
    const size_t bytes = (size_t)256 << 20;  // 2x the 126 MB L2
    c->flush_buf.ensure(bytes, c->stream);
    CK(cudaMemsetAsync(c->flush_buf.get(), (int)(c->launches & 0xff), bytes, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return JET_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  }
}

int jet_profile_reset(jet_ctx* ctx) {
  try {
    Ctx* c = reinterpret_cast<Ctx*>(ctx);
    c->flush_prof();
    for (auto& a : c->agg) {
      a.launches = 0;
      a.ms = 0;
      a.bytes = 0;
    }
    c->launches = 0;
    return JET_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  }
}

int jet_profile_report(jet_ctx* ctx, char* buf, int64_t cap) {
  try {
    Ctx* c = reinterpret_cast<Ctx*>(ctx);
    c->flush_prof();
    std::string s;
    char line[256];
    snprintf(line, sizeof line, "__total__\t%lld\t0\t0\n", (long long)c->launches);
    s += line;
    for (auto& a : c->agg) {
      if (!a.launches) continue;
      snprintf(line, sizeof line, "%s\t%lld\t%.6f\t%.0f\n", a.name.c_str(),
               (long long)a.launches, a.ms, a.bytes);
      s += line;
    }
    if (buf && cap > 0) {
      size_t n = s.size() < (size_t)(cap - 1) ? s.size() : (size_t)(cap - 1);
      memcpy(buf, s.data(), n);
      buf[n] = 0;
    }
    return (int)s.size();
  } catch (const Error& e) {
    set_last_error(e.what());
    return -e.code;
  }
}

}  // extern "C"
