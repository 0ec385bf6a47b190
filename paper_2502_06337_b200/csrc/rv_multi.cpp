// Multi-GPU in one process (rv_multi_*, include/rotavote_b200.h): one rv_context per device, an
// NCCL communicator clique over the devices (ncclCommInitAll; NVLink / NVSwitch on a B200 box),
// and the sharded estimate_single of SURVEY.md 8(e):
//
//   shard d = [n*d/P, n*(d+1)/P)   H2D + in-order preprocess + band-tiled vote on device d
//   ncclAllReduce(u32 grid, sum)   in place on every device: the single-device grid, bit for bit
//                                  (the reference's own chunked vote relies on the same integer
//                                  order-independence, voting.cpp:102-117)
//   peak + start axis              device 0 (estimate_from_peak, estimator.cpp:94-97)
//   refine_loop (estimator.cpp:51-69), every pass:
//                                  classify + 6 scatter sums + "set changed" on each device's
//                                  shard; the host sums the partials in rank order and solves the
//                                  3x3 (refine_axis, :299-309) -- 8 doubles per device per pass
//   build_estimate (:73-92)        inlier lists concatenated in rank order (= ascending input
//                                  indices); angle histograms summed; peak_angle window sums
//                                  around the summed histogram's peak, summed in rank order
//
// The branches that need the whole input (identity shortcuts, the exactness-guard re-vote and the
// rescue path, estimator.cpp:326-340, :352-368) finish on device 0 from the summed grid. NCCL is
// loaded at run time (libnccl.so.2), so the library itself has no link-time NCCL dependency.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <numbers>
#include <string>
#include <thread>
#include <vector>

#include "../../include/rotavote_b200.h"

namespace {

struct NcclApi {
  void* handle = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
  std::string error;
};

NcclApi* nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      api.handle = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (api.handle) break;
    }
    if (!api.handle) {
      api.error = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return;
    }
    auto sym = [](const char* n) { return dlsym(api.handle, n); };
    api.CommInitAll = reinterpret_cast<decltype(api.CommInitAll)>(sym("ncclCommInitAll"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    api.GetVersion = reinterpret_cast<decltype(api.GetVersion)>(sym("ncclGetVersion"));
    if (!api.CommInitAll || !api.CommDestroy || !api.AllReduce || !api.GroupStart || !api.GroupEnd ||
        !api.GetErrorString || !api.GetVersion) {
      api.error = "libnccl.so.2 lacks an expected symbol";
      api.handle = nullptr;
    }
  });
  return api.handle ? &api : nullptr;
}

struct MultiError {
  rv_status st;
  std::string msg;
};
[[noreturn]] void mfail(rv_status st, const std::string& msg) { throw MultiError{st, msg}; }
void mck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) mfail(RV_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

struct DevMem {
  void* p = nullptr;
  size_t cap = 0;
  template <typename T>
  T* get(size_t count) {
    const size_t bytes = std::max<size_t>(count * sizeof(T), 16);
    if (bytes > cap) {
      if (p) cudaFree(p);
      p = nullptr;
      cap = 0;
      mck(cudaMalloc(&p, bytes), "cudaMalloc (multi)");
      cap = bytes;
    }
    return static_cast<T*>(p);
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

// One worker thread per device (each bound to its device); run(f) calls f(d) on every device in
// parallel and returns when all are done -- the per-device steps of the sharded solve are
// synchronous C-ABI calls, so the devices overlap through the workers.
class DevicePool {
 public:
  explicit DevicePool(const std::vector<int>& devices) : n_((int)devices.size()) {
    if (n_ < 2) return;
    for (int d = 0; d < n_; ++d)
      threads_.emplace_back([this, d, dev = devices[(size_t)d]] {
        cudaSetDevice(dev);
        int seen = 0;
        for (;;) {
          std::function<void(int)> job;
          {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
            if (stop_) return;
            seen = gen_;
            job = job_;
          }
          job(d);
          std::lock_guard<std::mutex> lk(mu_);
          if (--pending_ == 0) done_.notify_all();
        }
      });
  }
  ~DevicePool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : threads_) t.join();
  }
  void run(const std::function<void(int)>& f) {
    if (n_ < 2) {
      for (int d = 0; d < n_; ++d) f(d);
      return;
    }
    std::unique_lock<std::mutex> lk(mu_);
    job_ = f;
    pending_ = n_;
    ++gen_;
    cv_.notify_all();
    done_.wait(lk, [&] { return pending_ == 0; });
  }

 private:
  int n_;
  std::vector<std::thread> threads_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  std::function<void(int)> job_;
  int gen_ = 0, pending_ = 0;
  bool stop_ = false;
};

}  // namespace

struct rv_multi {
  std::vector<int> devices;
  std::vector<rv_context*> ctx;
  std::vector<cudaStream_t> streams;
  std::vector<ncclComm_t> comms;
  std::vector<DevMem> corrs, grid, full, xlines;  // xlines: cross-device refine line buffers
  bool peer_ok = false;                            // peer access between every device pair
  uint64_t xepoch = 0;
  std::vector<int32_t> inliers;
  std::string last_error;
  int nccl_version = 0;
  DevicePool* pool = nullptr;
};

namespace {

int P(const rv_multi* m) { return (int)m->ctx.size(); }

// per-device call of a C-ABI step; the first failing device's status and message win
void run_all(rv_multi* m, const std::function<rv_status(int)>& f) {
  std::vector<rv_status> st((size_t)P(m), RV_OK);
  m->pool->run([&](int d) { st[(size_t)d] = f(d); });
  for (int d = 0; d < P(m); ++d)
    if (st[(size_t)d] != RV_OK) mfail(st[(size_t)d], std::string("device ") + std::to_string(m->devices[(size_t)d]) +
                                                         ": " + rv_context_last_error(m->ctx[(size_t)d]));
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) mfail(RV_ERR_NCCL, std::string(what) + ": " + nccl_api()->GetErrorString(r));
}

// In-place sum of the devices' u32 grids (ncclUint32 wraps like uint32_t: exact).
void allreduce_grids(rv_multi* m, size_t cells) {
  NcclApi* api = nccl_api();
  nccl_check(api->GroupStart(), "ncclGroupStart");
  for (int d = 0; d < P(m); ++d) {
    cudaSetDevice(m->devices[(size_t)d]);
    uint32_t* g = m->grid[(size_t)d].get<uint32_t>(cells);
    nccl_check(api->AllReduce(g, g, cells, ncclUint32, ncclSum, m->comms[(size_t)d], m->streams[(size_t)d]),
               "ncclAllReduce");
  }
  nccl_check(api->GroupEnd(), "ncclGroupEnd");
  for (int d = 0; d < P(m); ++d) {
    cudaSetDevice(m->devices[(size_t)d]);
    mck(cudaStreamSynchronize(m->streams[(size_t)d]), "grid all-reduce");
  }
}

// device 0 finishes from the summed grid with the whole input (rare branches)
void finish_on_device0(rv_multi* m, const double* corrs, int64_t n, const rv_config* cfg, rv_estimate* out) {
  cudaSetDevice(m->devices[0]);
  double* d = m->full[0].get<double>((size_t)n * 6);
  mck(cudaMemcpyAsync(d, corrs, sizeof(double) * 6 * (size_t)n, cudaMemcpyHostToDevice, m->streams[0]), "H2D full");
  mck(cudaStreamSynchronize(m->streams[0]), "H2D full");
  const size_t cells = (size_t)cfg->grid * cfg->grid;
  rv_status st = rv_estimate_single_prevoted(m->ctx[0], d, n, cfg, m->grid[0].get<uint32_t>(cells), out);
  if (st != RV_OK) mfail(st, rv_context_last_error(m->ctx[0]));
  m->inliers.assign((size_t)out->n_inliers, 0);
  st = rv_result_inliers(m->ctx[0], 0, m->inliers.data(), out->n_inliers);
  if (st != RV_OK) mfail(st, rv_context_last_error(m->ctx[0]));
}

template <typename F>
rv_status mguard(rv_multi* m, F&& f) {
  try {
    f();
    return RV_OK;
  } catch (const MultiError& e) {
    m->last_error = e.msg;
    return e.st;
  } catch (const std::bad_alloc&) {
    m->last_error = "host allocation failed";
    return RV_ERR_OUT_OF_MEMORY;
  }
}

}  // namespace

extern "C" {

rv_status rv_multi_create(const int32_t* devices, int32_t n_devices, rv_multi** out) {
  if (!devices || n_devices < 1 || !out) return RV_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  NcclApi* api = nccl_api();
  if (!api) return RV_ERR_NCCL;
  auto* m = new rv_multi();
  for (int d = 0; d < n_devices; ++d) m->devices.push_back(devices[d]);
  rv_status st = RV_OK;
  for (int d = 0; d < n_devices && st == RV_OK; ++d) {
    rv_context* c = nullptr;
    st = rv_context_create(devices[d], &c);
    if (st != RV_OK) break;
    m->ctx.push_back(c);
    cudaSetDevice(devices[d]);
    cudaStream_t s = nullptr;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) {
      st = RV_ERR_CUDA;
      break;
    }
    m->streams.push_back(s);
    rv_context_set_stream(c, s);  // the context's work and the collectives share one stream
  }
  if (st == RV_OK) {
    m->comms.resize((size_t)n_devices);
    if (api->CommInitAll(m->comms.data(), n_devices, m->devices.data()) != ncclSuccess) {
      m->comms.clear();
      st = RV_ERR_NCCL;
    } else {
      api->GetVersion(&m->nccl_version);
    }
  }
  if (st != RV_OK) {
    rv_multi_destroy(m);
    return st;
  }
  m->corrs.resize((size_t)n_devices);
  m->grid.resize((size_t)n_devices);
  m->full.resize((size_t)n_devices);
  m->xlines.resize((size_t)n_devices);
  // the sharded refine exchanges its per-pass partials through peer memory (NVLink): every
  // device needs access to every other's line buffer; without it the host steps the passes
  m->peer_ok = n_devices <= 8;
  for (int d = 0; d < n_devices && m->peer_ok; ++d)
    for (int q = 0; q < n_devices && m->peer_ok; ++q) {
      if (q == d) continue;
      if (devices[q] == devices[d]) {  // one GPU listed twice: its kernels must not wait on each other
        m->peer_ok = false;
        break;
      }
      int can = 0;
      cudaDeviceCanAccessPeer(&can, devices[d], devices[q]);
      if (!can) {
        m->peer_ok = false;
        break;
      }
      cudaSetDevice(devices[d]);
      const cudaError_t e = cudaDeviceEnablePeerAccess(devices[q], 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) m->peer_ok = false;
      cudaGetLastError();
    }
  for (int d = 0; d < n_devices && m->peer_ok; ++d) {
    cudaSetDevice(devices[d]);
    try {
      void* p = m->xlines[(size_t)d].get<char>(8 * 16 * sizeof(double));
      if (cudaMemset(p, 0, 8 * 16 * sizeof(double)) != cudaSuccess) m->peer_ok = false;
    } catch (const MultiError&) {
      m->peer_ok = false;
    }
  }
  m->pool = new DevicePool(m->devices);
  *out = m;
  return RV_OK;
}

void rv_multi_destroy(rv_multi* m) {
  if (!m) return;
  delete m->pool;
  if (NcclApi* api = nccl_api())
    for (ncclComm_t c : m->comms)
      if (c) api->CommDestroy(c);
  for (size_t d = 0; d < m->devices.size(); ++d) {
    cudaSetDevice(m->devices[d]);
    if (d < m->corrs.size()) m->corrs[d].release();
    if (d < m->grid.size()) m->grid[d].release();
    if (d < m->full.size()) m->full[d].release();
    if (d < m->xlines.size()) m->xlines[d].release();
  }
  for (rv_context* c : m->ctx) rv_context_destroy(c);
  for (size_t d = 0; d < m->streams.size(); ++d) {
    cudaSetDevice(m->devices[d]);
    cudaStreamDestroy(m->streams[d]);
  }
  delete m;
}

int32_t rv_multi_size(const rv_multi* m) { return m ? (int32_t)m->ctx.size() : 0; }
const char* rv_multi_last_error(const rv_multi* m) { return m ? m->last_error.c_str() : "null multi context"; }
int32_t rv_multi_nccl_version(const rv_multi* m) { return m ? m->nccl_version : 0; }

rv_status rv_multi_estimate_single(rv_multi* m, const double* corrs, int64_t n, const rv_config* cfg,
                                   rv_estimate* out) {
  if (!m || !cfg || !out || (n > 0 && !corrs)) return RV_ERR_INVALID_ARGUMENT;
  return mguard(m, [&] {
    const auto t0 = std::chrono::steady_clock::now();
    if (n <= 0) mfail(RV_ERR_EMPTY_INPUT, "no correspondences");
    const int np = P(m);
    const size_t cells = (size_t)cfg->grid * cfg->grid;
    std::vector<int64_t> lo((size_t)np + 1), kept((size_t)np, 0);
    for (int d = 0; d <= np; ++d) lo[(size_t)d] = n * d / np;
    // 1. shards: H2D, in-order preprocess, band-tiled vote into each device's grid
    run_all(m, [&](int d) -> rv_status {
      const int64_t nd = lo[(size_t)d + 1] - lo[(size_t)d];
      double* dc = m->corrs[(size_t)d].get<double>((size_t)std::max<int64_t>(nd, 1) * 6);
      uint32_t* g = m->grid[(size_t)d].get<uint32_t>(cells);
      if (nd > 0 && cudaMemcpyAsync(dc, corrs + 6 * lo[(size_t)d], sizeof(double) * 6 * (size_t)nd,
                                    cudaMemcpyHostToDevice, m->streams[(size_t)d]) != cudaSuccess)
        return RV_ERR_CUDA;
      return rv_vote_shard(m->ctx[(size_t)d], dc, nd, cfg, g, &kept[(size_t)d]);
    });
    // 2. one NCCL all-reduce of the u32 grids
    allreduce_grids(m, cells);
    int64_t n_kept = 0;
    for (int64_t k : kept) n_kept += k;
    // identity shortcuts (estimator.cpp:326-340) need the dropped list: device 0 finishes
    if (n_kept == 0 || (n - n_kept) * 10 >= n * 9) return finish_on_device0(m, corrs, n, cfg, out);
    // 3. peak and start axis from the summed grid (identical on every device; device 0 reads it)
    double axis[3];
    uint32_t votes = 0;
    uint64_t total = 0;
    cudaSetDevice(m->devices[0]);
    rv_status st = rv_peak_start_axis(m->ctx[0], m->grid[0].get<uint32_t>(cells), cfg, axis, &votes, &total);
    if (st != RV_OK) mfail(st, rv_context_last_error(m->ctx[0]));
    if (total != (uint64_t)n_kept * (uint64_t)cfg->theta_samples)  // exactness guard: device 0 re-votes
      return finish_on_device0(m, corrs, n, cfg, out);
    // 4. refine_loop (estimator.cpp:51-69) on the shards
    std::vector<int64_t> cnt((size_t)np);
    std::vector<std::array<double, 6>> sc((size_t)np);
    std::vector<int32_t> diff((size_t)np);
    auto classify = [&](const double* ax, int slot, int compare) -> int64_t {
      run_all(m, [&](int d) {
        return rv_shard_classify(m->ctx[(size_t)d], ax, cfg->epsilon, slot, compare, &cnt[(size_t)d],
                                 sc[(size_t)d].data(), &diff[(size_t)d]);
      });
      int64_t c = 0;
      for (int64_t v : cnt) c += v;
      return c;
    };
    int slot = 0;
    int64_t count = 0;
    if (m->peer_ok) {
      // device-resident refine: one cooperative loop per device, partials exchanged through
      // peer memory each pass (rv_shard_refine); every device ends with the same axis
      const uint64_t ep = ++m->xepoch;
      double* lines[8] = {};
      for (int d = 0; d < np; ++d) lines[d] = m->xlines[(size_t)d].get<double>(8 * 16);
      std::vector<std::array<double, 3>> ax((size_t)np);
      std::vector<int64_t> total((size_t)np);
      run_all(m, [&](int d) {
        return rv_shard_refine(m->ctx[(size_t)d], axis, cfg, np, d, lines, ep, ax[(size_t)d].data(),
                               &total[(size_t)d], &cnt[(size_t)d], sc[(size_t)d].data(), nullptr);
      });
      count = total[0];
      std::memcpy(axis, ax[0].data(), sizeof axis);
      // rescue (estimator.cpp:352-368) needs every constraint: device 0 finishes
      if (cfg->refine && (double)count < 3.0 * (cfg->epsilon * (double)n_kept))
        return finish_on_device0(m, corrs, n, cfg, out);
    } else {
    count = classify(axis, slot, 0);
    if (cfg->refine) {
      for (int pass = 0; pass < 10 && count >= 2; ++pass) {
        double s6[6] = {0, 0, 0, 0, 0, 0};
        for (int d = 0; d < np; ++d)  // rank order
          for (int k = 0; k < 6; ++k) s6[k] += sc[(size_t)d][(size_t)k];
        double next[3];
        if (rv_axis_from_scatter(s6, next) != RV_OK) break;  // RankDeficient: keep the axis
        count = classify(next, 1 - slot, 1);
        slot = 1 - slot;
        axis[0] = next[0];
        axis[1] = next[1];
        axis[2] = next[2];
        bool stable = true;
        for (int32_t v : diff) stable = stable && v == 0;
        if (stable) break;
      }
      // rescue (estimator.cpp:352-368) needs every constraint: device 0 finishes
      if ((double)count < 3.0 * (cfg->epsilon * (double)n_kept)) return finish_on_device0(m, corrs, n, cfg, out);
    }
    }
    // 5. build_estimate (estimator.cpp:73-92): inliers in rank order, angle vote over the shards
    m->inliers.assign((size_t)count, 0);
    std::vector<int64_t> off((size_t)np + 1, 0);
    for (int d = 0; d < np; ++d) off[(size_t)d + 1] = off[(size_t)d] + cnt[(size_t)d];
    std::vector<int64_t> got((size_t)np);
    run_all(m, [&](int d) {
      return rv_shard_inliers(m->ctx[(size_t)d], slot, lo[(size_t)d], m->inliers.data() + off[(size_t)d],
                              cnt[(size_t)d], &got[(size_t)d]);
    });
    const int B = cfg->angle_bins;
    std::vector<std::vector<uint32_t>> bins((size_t)np, std::vector<uint32_t>((size_t)std::max(B, 1)));
    std::vector<uint64_t> contrib((size_t)np);
    run_all(m, [&](int d) {
      return rv_shard_angle_hist(m->ctx[(size_t)d], axis, cfg, bins[(size_t)d].data(), &contrib[(size_t)d]);
    });
    std::vector<uint32_t> hist((size_t)B, 0u);
    uint64_t contributing = 0;
    for (int d = 0; d < np; ++d) {
      contributing += contrib[(size_t)d];
      for (int k = 0; k < B; ++k) hist[(size_t)k] += bins[(size_t)d][(size_t)k];
    }
    if (contributing == 0) mfail(RV_ERR_NO_VOTES, "no correspondence produced an angle vote");
    int peak = 0;  // peak_angle (angles.cpp:70-90): the first maximum bin
    for (int k = 1; k < B; ++k)
      if (hist[(size_t)k] > hist[(size_t)peak]) peak = k;
    const double w = 2.0 * std::numbers::pi / B;
    const double center = -std::numbers::pi + (peak + 0.5) * w;
    double angle = center;
    if (cfg->refine) {
      std::vector<std::array<double, 2>> sums((size_t)np);
      run_all(m, [&](int d) {
        return rv_shard_angle_sums(m->ctx[(size_t)d], hist.data(), cfg, sums[(size_t)d].data());
      });
      double s = 0.0, c = 0.0;
      for (int d = 0; d < np; ++d) {
        s += sums[(size_t)d][0];
        c += sums[(size_t)d][1];
      }
      if (!(s == 0.0 && c == 0.0)) {
        angle = std::atan2(s, c);
        if (angle <= -std::numbers::pi) angle += 2.0 * std::numbers::pi;
      }
    }
    out->axis[0] = axis[0];
    out->axis[1] = axis[1];
    out->axis[2] = axis[2];
    out->angle = angle;
    rv_rodrigues(axis, angle, out->rotation);
    out->axis_votes = votes;
    out->n_inliers = count;
    out->elapsed_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

rv_status rv_multi_result_inliers(rv_multi* m, int32_t* dst, int64_t capacity) {
  if (!m || (capacity > 0 && !dst)) return RV_ERR_INVALID_ARGUMENT;
  const size_t k = std::min<size_t>((size_t)std::max<int64_t>(capacity, 0), m->inliers.size());
  std::copy(m->inliers.begin(), m->inliers.begin() + (long)k, dst);
  return RV_OK;
}

rv_status rv_multi_accumulate(rv_multi* m, const double* z, int64_t n, int32_t grid, double extent, int32_t samples,
                              uint32_t* counts_out) {
  if (!m || (n > 0 && !z) || !counts_out) return RV_ERR_INVALID_ARGUMENT;
  return mguard(m, [&] {
    if (n <= 0) mfail(RV_ERR_EMPTY_INPUT, "no constraints to accumulate");
    if (grid < 1 || !(extent > 0.0)) mfail(RV_ERR_INVALID_CONFIG, "accumulator needs grid >= 1, extent > 0");
    const int np = P(m);
    const size_t cells = (size_t)grid * grid;
    // accumulate's own fan-out (voting.cpp:95-117): contiguous chunks, one per device
    run_all(m, [&](int d) -> rv_status {
      const int64_t a = n * d / np, b = n * (d + 1) / np;
      uint32_t* g = m->grid[(size_t)d].get<uint32_t>(cells);
      if (b <= a) return cudaMemsetAsync(g, 0, sizeof(uint32_t) * cells, m->streams[(size_t)d]) == cudaSuccess
                             ? RV_OK : RV_ERR_CUDA;
      double* dz = m->corrs[(size_t)d].get<double>((size_t)(b - a) * 3);
      if (cudaMemcpyAsync(dz, z + 3 * a, sizeof(double) * 3 * (size_t)(b - a), cudaMemcpyHostToDevice,
                          m->streams[(size_t)d]) != cudaSuccess)
        return RV_ERR_CUDA;
      return rv_accumulate_device(m->ctx[(size_t)d], dz, b - a, grid, extent, samples, g);
    });
    allreduce_grids(m, cells);
    cudaSetDevice(m->devices[0]);
    mck(cudaMemcpy(counts_out, m->grid[0].get<uint32_t>(cells), sizeof(uint32_t) * cells, cudaMemcpyDeviceToHost),
        "D2H grid");
  });
}

}  // extern "C"
