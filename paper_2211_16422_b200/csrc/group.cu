// Multi-GPU group: ONE process, ONE handle, n devices (homs_b200_ctx_create_multi).
//
// What it replaces: the reference's only parallel construct is parallel_for
// (include/homs/parallel.hpp:20-48), a thread fan-out over one shared-memory index.  Here the fan-out is
// over GPUs (SURVEY.md 8e / 8b `ctx_create(device_ids[], n)`):
//
//   * the library is cut into contiguous precursor-m/z slices of every charge bucket, slice g resident
//     on member g (library.cu); the metadata (m/z, id ranks) is replicated, so every member computes
//     window bounds in full-bucket coordinates;
//   * queries are replicated to every member;
//   * a search runs the single-GPU pipeline on every member at once.  There is no separate
//     collective: the last kernel of each member's pipeline (tc_reduce / direct / POPC reduce) stores
//     its 16-byte candidate records straight into slot g of a gather block in the LEADING device's
//     memory -- peer-mapped stores over NVLink when the member sits on another device -- and the
//     leader's k-way merge kernel runs once every member's stream has reached its join event.  The
//     exchange is 16 B x k per query and member (256 KB at config 2): launch-latency, not link bound,
//     which is why it is folded into the producing kernel instead of a library collective;
//   * every member is driven by its own host thread (issue latency of ~15 launches per member would
//     otherwise serialise on one thread), the leader's stream orders the whole call: callers see
//     one stream-ordered operation exactly like the single-device context.
//
// A member whose device cannot address the leader's memory (no P2P) writes locally and the records
// travel with cudaMemcpyPeerAsync instead.  Devices may repeat (n aliases of one GPU): that is how the
// tests exercise this very code path on a one-GPU box, results bit-identical to a plain context.
//
// The multi-process form of the same partitioning (one rank per GPU, NCCL all-gather of the records,
// then homs_b200_merge_candidates_dev) lives in paper_2211_16422_b200/sharded.py / bench.py.
#include <condition_variable>
#include <thread>

#include "common.cuh"

namespace hb {

struct GroupWorkers {
  struct Worker {
    std::thread th;
    std::mutex m;
    std::condition_variable cv;
    std::function<void()> job;
    bool has_job = false, stop = false;
  };
  std::vector<std::unique_ptr<Worker>> w;  // w[g - 1] drives member g
  std::mutex done_m;
  std::condition_variable done_cv;
  int pending = 0;

  void start(const std::vector<homs_b200_ctx*>& members) {
    for (size_t g = 1; g < members.size(); ++g) {
      auto wk = std::make_unique<Worker>();
      Worker* raw = wk.get();
      const int device = members[g]->device;
      wk->th = std::thread([this, raw, device] {
        cudaSetDevice(device);
        for (;;) {
          std::function<void()> job;
          {
            std::unique_lock<std::mutex> lk(raw->m);
            raw->cv.wait(lk, [&] { return raw->has_job || raw->stop; });
            if (raw->stop) return;
            job = std::move(raw->job);
            raw->has_job = false;
          }
          job();
          {
            std::lock_guard<std::mutex> lk(done_m);
            --pending;
          }
          done_cv.notify_one();
        }
      });
      w.push_back(std::move(wk));
    }
  }
  void post(size_t g, std::function<void()> job) {
    Worker& wk = *w[g - 1];
    {
      std::lock_guard<std::mutex> lk(wk.m);
      wk.job = std::move(job);
      wk.has_job = true;
    }
    wk.cv.notify_one();
  }
  void stop() {
    for (auto& wk : w) {
      {
        std::lock_guard<std::mutex> lk(wk->m);
        wk->stop = true;
      }
      wk->cv.notify_one();
      wk->th.join();
    }
    w.clear();
  }
};

int group_for_each(homs_b200_ctx* leader, const std::function<int(uint32_t, homs_b200_ctx*)>& fn) {
  const size_t G = leader->members.size();
  std::vector<int> rc(G, HOMS_B200_OK);
  GroupWorkers* gw = leader->workers;
  {
    std::lock_guard<std::mutex> lk(gw->done_m);
    gw->pending = static_cast<int>(G - 1);
  }
  for (size_t g = 1; g < G; ++g)
    gw->post(g, [&, g] { rc[g] = fn(static_cast<uint32_t>(g), leader->members[g]); });
  cudaSetDevice(leader->device);
  rc[0] = fn(0, leader);
  {
    std::unique_lock<std::mutex> lk(gw->done_m);
    gw->done_cv.wait(lk, [&] { return gw->pending == 0; });
  }
  cudaSetDevice(leader->device);
  for (size_t g = 0; g < G; ++g)
    if (rc[g] != HOMS_B200_OK) {
      if (g > 0) leader->error = "device " + std::to_string(leader->members[g]->device) + " (member " +
                                 std::to_string(g) + "): " + leader->members[g]->error;
      return rc[g];
    }
  return HOMS_B200_OK;
}

int group_fork(homs_b200_ctx* leader) {
  cudaSetDevice(leader->device);
  HB_CUDA(leader, cudaEventRecord(leader->ev_fork, leader->stream));
  for (size_t g = 1; g < leader->members.size(); ++g) {
    homs_b200_ctx* m = leader->members[g];
    cudaSetDevice(m->device);
    HB_CUDA(leader, cudaStreamWaitEvent(m->stream, leader->ev_fork, 0));
  }
  cudaSetDevice(leader->device);
  return HOMS_B200_OK;
}

int group_join(homs_b200_ctx* leader) {
  for (size_t g = 1; g < leader->members.size(); ++g) {
    homs_b200_ctx* m = leader->members[g];
    cudaSetDevice(m->device);
    HB_CUDA(leader, cudaEventRecord(leader->ev_join[g], m->stream));
  }
  cudaSetDevice(leader->device);
  for (size_t g = 1; g < leader->members.size(); ++g)
    HB_CUDA(leader, cudaStreamWaitEvent(leader->stream, leader->ev_join[g], 0));
  return HOMS_B200_OK;
}

int sync_all_locked(homs_b200_ctx* ctx) {
  for (size_t g = 1; g < ctx->members.size(); ++g) {
    cudaSetDevice(ctx->members[g]->device);
    HB_CUDA(ctx, cudaStreamSynchronize(ctx->members[g]->stream));
  }
  cudaSetDevice(ctx->device);
  HB_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return HOMS_B200_OK;
}

void group_destroy_members(homs_b200_ctx* leader) {
  if (!is_group(leader)) return;
  if (leader->workers) {
    leader->workers->stop();
    delete leader->workers;
    leader->workers = nullptr;
  }
  for (size_t g = 1; g < leader->members.size(); ++g) {
    homs_b200_ctx* m = leader->members[g];
    ctx_free_resources(m);
    if (g < leader->ev_join.size() && leader->ev_join[g]) cudaEventDestroy(leader->ev_join[g]);
    delete m;
  }
  cudaSetDevice(leader->device);
  if (leader->ev_fork) cudaEventDestroy(leader->ev_fork);
  leader->ev_fork = nullptr;
  leader->members.clear();
}

// ---- the group forms of the single-context building blocks ---------------------------------------

int queries_set_any_locked(homs_b200_ctx* ctx, uint32_t dim, uint64_t nq, const uint64_t* words, const double* mz,
                           const uint8_t* charge, bool on_device) {
  if (!is_group(ctx)) return queries_set_locked(ctx, dim, nq, words, mz, charge, on_device);
  if (!on_device)  // host arrays: every member uploads its own replica over its own PCIe link
    return group_for_each(ctx, [&](uint32_t, homs_b200_ctx* m) -> int {
      return queries_set_locked(m, dim, nq, words, mz, charge, false);
    });
  // device arrays live in the leader's memory, produced on the leader's stream
  HB_TRY(queries_set_locked(ctx, dim, nq, words, mz, charge, true));
  return queries_replicate_locked(ctx);
}

int queries_replicate_locked(homs_b200_ctx* leader) {
  const Queries& src = leader->q;
  HB_TRY(group_fork(leader));
  HB_TRY(group_for_each(leader, [&](uint32_t g, homs_b200_ctx* m) -> int {
    if (g == 0) return int(HOMS_B200_OK);
    Queries& q = m->q;
    q.ready = false;
    q.dim = src.dim;
    q.nq = src.nq;
    const size_t row_bytes = size_t(stride_for(src.dim)) * 8;
    HB_TRY(ensure(m, q.d_words, src.nq * row_bytes));
    HB_TRY(ensure(m, q.d_mz, src.nq * 8));
    HB_TRY(ensure(m, q.d_charge, src.nq));
    if (src.nq) {
      HB_CUDA(m, cudaMemcpyPeerAsync(q.d_words.p, m->device, src.d_words.p, leader->device, src.nq * row_bytes, m->stream));
      HB_CUDA(m, cudaMemcpyPeerAsync(q.d_mz.p, m->device, src.d_mz.p, leader->device, src.nq * 8, m->stream));
      HB_CUDA(m, cudaMemcpyPeerAsync(q.d_charge.p, m->device, src.d_charge.p, leader->device, src.nq, m->stream));
    }
    q.ready = true;
    return int(HOMS_B200_OK);
  }));
  return group_join(leader);  // the leader's buffers may be rewritten by later work on its stream
}

int search_any_locked(homs_b200_ctx* ctx, const uint32_t* d_subset, uint64_t n, const homs_b200_tolerance* tol,
                      uint32_t k, Cand* d_out, uint64_t* d_first, uint64_t* d_last, uint8_t* d_has) {
  if (!is_group(ctx)) return search_dev_locked(ctx, d_subset, n, tol, k, d_out, d_first, d_last, d_has);
  const uint32_t G = static_cast<uint32_t>(ctx->members.size());
  HB_REQUIRE(ctx, k >= 1 && k <= HOMS_B200_MAX_TOPK, HOMS_B200_ERR_ARGUMENT, "search: k must be in [1, 64]");
  const size_t part_bytes = n * k * sizeof(Cand);
  HB_TRY(ensure(ctx, ctx->group_gather, size_t(G) * part_bytes));
  Cand* gather = ctx->group_gather.as<Cand>();
  HB_TRY(group_fork(ctx));
  HB_TRY(group_for_each(ctx, [&](uint32_t g, homs_b200_ctx* m) -> int {
    const uint32_t* sub = d_subset;
    if (g > 0 && d_subset && n) {  // the stage-2 index list of the cascade lives in the leader's memory
      HB_TRY(ensure(m, m->scratch[kScrSubset], n * 4));
      HB_CUDA(m, cudaMemcpyPeerAsync(m->scratch[kScrSubset].p, m->device, d_subset, ctx->device, n * 4, m->stream));
      sub = m->scratch[kScrSubset].as<uint32_t>();
    }
    Cand* slot = gather + size_t(g) * n * k;
    if (ctx->peer_ok[g])  // the member's last kernel stores its records straight into the leader's block
      return search_dev_locked(m, sub, n, tol, k, slot, g == 0 ? d_first : nullptr, g == 0 ? d_last : nullptr,
                               g == 0 ? d_has : nullptr);
    HB_TRY(ensure(m, m->scratch[kScrRecords2], part_bytes));
    HB_TRY(search_dev_locked(m, sub, n, tol, k, m->scratch[kScrRecords2].as<Cand>(), nullptr, nullptr, nullptr));
    if (part_bytes)
      HB_CUDA(m, cudaMemcpyPeerAsync(slot, ctx->device, m->scratch[kScrRecords2].p, m->device, part_bytes, m->stream));
    return int(HOMS_B200_OK);
  }));
  HB_TRY(group_join(ctx));
  ctx->last_engine = ctx->members[0]->last_engine;
  return merge_launch(ctx, n, k, G, gather, d_out);
}

int library_build_any(homs_b200_ctx* ctx, uint32_t dim, uint64_t n, const uint64_t* h_words,
                      const uint64_t* d_words_in, const double* mz, const uint8_t* charge, const uint32_t* id_rank,
                      uint32_t shard_index, uint32_t shard_count, const uint32_t* row_of_entry) {
  if (!is_group(ctx))
    return library_build(ctx, dim, n, h_words, d_words_in, mz, charge, id_rank, shard_index, shard_count, row_of_entry);
  HB_REQUIRE(ctx, shard_index == 0 && shard_count == 1, HOMS_B200_ERR_ARGUMENT,
             "build_index: a multi-device context shards the library itself; pass shard 0 of 1");
  const uint32_t G = static_cast<uint32_t>(ctx->members.size());
  if (d_words_in) HB_TRY(group_fork(ctx));  // the rows were produced on the leader's stream
  HB_TRY(group_for_each(ctx, [&](uint32_t g, homs_b200_ctx* m) -> int {
    const uint64_t* src = d_words_in;
    if (d_words_in && !ctx->peer_ok[g]) {
      // no peer mapping: bring the dense rows over once, gather locally
      uint64_t rows = n;
      if (row_of_entry) {  // rows of the source block that entries refer to
        rows = 0;
        for (uint64_t i = 0; i < n; ++i) rows = std::max<uint64_t>(rows, uint64_t(row_of_entry[i]) + 1);
      }
      const size_t src_bytes = size_t(rows) * words_for(dim) * 8;
      HB_TRY(ensure(m, m->scratch[kScrFusedRows], src_bytes));
      HB_CUDA(m, cudaMemcpyPeerAsync(m->scratch[kScrFusedRows].p, m->device, d_words_in, ctx->device, src_bytes, m->stream));
      src = m->scratch[kScrFusedRows].as<uint64_t>();
    }
    const int rc = library_build(m, dim, n, h_words, src, mz, charge, id_rank, g, G, row_of_entry);
    if (g > 0 && d_words_in && !ctx->peer_ok[g]) release(m->scratch[kScrFusedRows]);
    return rc;
  }));
  return HOMS_B200_OK;  // library_build synchronises every member's stream
}

}  // namespace hb

using namespace hb;

extern "C" int homs_b200_ctx_create_multi(const int* devices, int n_devices, homs_b200_ctx** out) {
  if (!out) return set_error(nullptr, HOMS_B200_ERR_ARGUMENT, "ctx_create_multi: out is null");
  *out = nullptr;
  if (!devices || n_devices < 1 || n_devices > 64)
    return set_error(nullptr, HOMS_B200_ERR_ARGUMENT, "ctx_create_multi: need 1 to 64 devices");
  homs_b200_ctx* leader = nullptr;
  HB_TRY(ctx_create_single(devices[0], &leader));
  if (n_devices == 1) {  // a plain context
    *out = leader;
    return HOMS_B200_OK;
  }
  leader->members.push_back(leader);
  leader->peer_ok.push_back(1);
  leader->ev_join.push_back(nullptr);
  auto fail = [&](int rc, const std::string& msg) {
    leader->members.resize(std::max<size_t>(1, leader->members.size()));
    group_destroy_members(leader);
    ctx_free_resources(leader);
    delete leader;
    return set_error(nullptr, rc, msg);
  };
  for (int g = 1; g < n_devices; ++g) {
    homs_b200_ctx* m = nullptr;
    const int rc = ctx_create_single(devices[g], &m);
    if (rc != HOMS_B200_OK) return fail(rc, std::string("ctx_create_multi: ") + homs_b200_last_error(nullptr));
    leader->members.push_back(m);
    cudaEvent_t ev = nullptr;
    cudaSetDevice(m->device);
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess)
      return fail(HOMS_B200_ERR_CUDA, "ctx_create_multi: cudaEventCreate failed");
    leader->ev_join.push_back(ev);
    // can kernels on this member's device address the leader's memory?
    uint8_t ok = m->device == leader->device;
    if (!ok) {
      int can = 0;
      if (cudaDeviceCanAccessPeer(&can, m->device, leader->device) == cudaSuccess && can) {
        const cudaError_t e = cudaDeviceEnablePeerAccess(leader->device, 0);
        ok = e == cudaSuccess || e == cudaErrorPeerAccessAlreadyEnabled;
        cudaGetLastError();  // clear "already enabled"
      }
    }
    leader->peer_ok.push_back(ok);
  }
  cudaSetDevice(leader->device);
  if (cudaEventCreateWithFlags(&leader->ev_fork, cudaEventDisableTiming) != cudaSuccess)
    return fail(HOMS_B200_ERR_CUDA, "ctx_create_multi: cudaEventCreate failed");
  leader->workers = new GroupWorkers;
  leader->workers->start(leader->members);
  *out = leader;
  return HOMS_B200_OK;
}

extern "C" int homs_b200_ctx_device_count(const homs_b200_ctx* ctx) {
  if (!ctx) return 0;
  return static_cast<int>(std::max<size_t>(1, ctx->members.size()));
}
