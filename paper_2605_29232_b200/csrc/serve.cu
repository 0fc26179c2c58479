// serve.cu -- the native serving loop: dynamic batching (S0) in front of the two-stream executor (S9), driven by
// an open-loop request trace ("Server-Side Batching" / "Hybrid
// CPU-GPU Execution"; Table 6; SPEC.md:633-641 for the batcher's contract).
//
// Host code only.  One host thread busy-polls: it admits the requests whose scheduled arrival has passed into a
// FIFO, retires finished batches (their CUDA event), and -- when a pinned host slot is free -- asks the batcher for
// the next batch, assembles it from the item pool (cvr_gather_items), and enqueues it through cvr_score_host (copy
// stream -> embed stream -> dense stream; the scores land in the slot's page-locked buffer).  Latency of a request =
// the host time its batch's scores were seen complete - its scheduled arrival (A21).
//
// The batcher (Batcher below) is the SAME rule as serving.DynamicBatcher (tests/test_serving.py pins both on the
// SPEC.md goldens; cvr_batcher_simulate replays it on a simulated clock for those tests):
//   * a request is never split; one with more than max_items items, or one arriving at a full queue, is rejected
//   * dispatch when the queued items reach max_items, or when the OLDEST queued request has waited window_s
//   * the batch is the longest FIFO prefix of whole requests with sum(items) <= max_items (and <= max_requests)
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <deque>
#include <limits>
#include <vector>

#include "../../include/cvr.h"

namespace {

struct Batcher {
  double window;
  int max_items, max_requests, capacity;
  std::deque<int> q;  // request ids, FIFO
  int64_t items = 0;
  int64_t rejected = 0;
  const double* t_arr;
  const int32_t* n_items;

  bool submit(int r) {
    if ((int)q.size() >= capacity || n_items[r] > max_items) {
      ++rejected;
      return false;
    }
    q.push_back(r);
    items += n_items[r];
    return true;
  }
  double next_deadline() const { return q.empty() ? std::numeric_limits<double>::infinity() : t_arr[q.front()] + window; }
  // the batch to dispatch at `now` (request ids appended to out), false if none
  bool poll(double now, std::vector<int>& out) {
    out.clear();
    if (q.empty()) return false;
    if (items < max_items && now < t_arr[q.front()] + window) return false;
    int64_t n = 0;
    while (!q.empty() && n + n_items[q.front()] <= max_items && (max_requests <= 0 || (int)out.size() < max_requests)) {
      n += n_items[q.front()];
      out.push_back(q.front());
      q.pop_front();
    }
    items -= n;
    return !out.empty();
  }
};

}  // namespace

extern "C" {

int cvr_batcher_simulate(int n_req, const double* t_arrival, const int32_t* n_items, double window_s, int max_items,
                         int max_requests, int queue_capacity, double service_fixed_s, double service_per_item_s,
                         double* latency, int32_t* batch_of, double* dispatch_time, int* n_batches) {
  if (n_req < 0 || !t_arrival || !n_items || !latency || !batch_of || !dispatch_time || !n_batches || max_items < 1 ||
      window_s < 0 || queue_capacity < 1)
    return CVR_E_ARG;
  for (int i = 1; i < n_req; ++i)
    if (t_arrival[i] < t_arrival[i - 1]) return CVR_E_ARG;
  Batcher b{window_s, max_items, max_requests, queue_capacity, {}, 0, 0, t_arrival, n_items};
  std::vector<int> out;
  double now = 0.0, free_at = 0.0;
  int i = 0, done = 0, nb = 0;
  for (int r = 0; r < n_req; ++r) {
    latency[r] = std::numeric_limits<double>::infinity();
    batch_of[r] = -1;
  }
  while (done < n_req) {
    // next event: an arrival, the oldest request's window expiring (or a full queue), the server freeing up
    double nxt = std::numeric_limits<double>::infinity();
    if (i < n_req) nxt = t_arrival[i];
    if (!b.q.empty()) nxt = std::min(nxt, std::max(b.items < max_items ? b.next_deadline() : free_at, free_at));
    if (std::isinf(nxt)) break;
    now = std::max(now, nxt);
    while (i < n_req && t_arrival[i] <= now) {
      if (!b.submit(i)) ++done;
      ++i;
    }
    if (now >= free_at && b.poll(now, out)) {
      int64_t n = 0;
      for (int r : out) n += n_items[r];
      free_at = now + (service_fixed_s + service_per_item_s * (double)n);
      for (int r : out) {
        latency[r] = free_at - t_arrival[r];
        batch_of[r] = nb;
      }
      dispatch_time[nb++] = now;
      done += (int)out.size();
      continue;
    }
    if (i >= n_req && !b.q.empty() && now < free_at) now = free_at;
  }
  *n_batches = nb;
  return CVR_OK;
}

int cvr_serve_trace(cvr_ctx* ctx, const cvr_serve_config* cfg, int n_tables, int n_dense, int64_t pool_size,
                    const int32_t* pool_offsets, const int32_t* pool_indices, const float* pool_dense, int n_req,
                    const double* t_arrival, const int32_t* n_items, const int64_t* item_start,
                    const int32_t* item_ids, double* latency, float* scores_out, int32_t* batch_sizes,
                    int* n_batches, cvr_serve_stats* stats, cvr_stream_t s_copy, cvr_stream_t s_embed,
                    cvr_stream_t s_dense) {
  if (!ctx || !cfg || !pool_offsets || !pool_indices || (n_dense && !pool_dense) || n_req < 0 || !t_arrival ||
      !n_items || !item_start || !item_ids || !latency || !batch_sizes || !n_batches || !stats)
    return CVR_E_ARG;
  if (cfg->max_items < 1 || cfg->window_s < 0 || cfg->host_slots < 1 || cfg->host_slots > 16 || cfg->max_nnz < 1 ||
      cfg->queue_capacity < 1)
    return CVR_E_ARG;
  for (int i = 1; i < n_req; ++i)
    if (t_arrival[i] < t_arrival[i - 1]) return CVR_E_ARG;
  const int S = cfg->host_slots, MI = cfg->max_items;
  struct Slot {
    int32_t *off = nullptr, *idx = nullptr;
    float *dense = nullptr, *scores = nullptr;
    cudaEvent_t ev = nullptr;
    std::vector<int> reqs;
  };
  std::vector<Slot> slots(S);
  cudaError_t e = cudaSuccess;
  for (auto& sl : slots) {  // page-locked staging per slot (the scores buffer is mapped: zero-copy head stores)
    if (e == cudaSuccess) e = cudaHostAlloc(&sl.off, ((size_t)n_tables * MI + 1) * 4, cudaHostAllocDefault);
    if (e == cudaSuccess) e = cudaHostAlloc(&sl.idx, (size_t)cfg->max_nnz * 4, cudaHostAllocDefault);
    if (e == cudaSuccess) e = cudaHostAlloc(&sl.dense, (size_t)MI * std::max(n_dense, 1) * 4, cudaHostAllocDefault);
    if (e == cudaSuccess) e = cudaHostAlloc(&sl.scores, (size_t)MI * 4, cudaHostAllocMapped);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&sl.ev, cudaEventDisableTiming);
  }
  auto release = [&]() {
    for (auto& sl : slots) {
      if (sl.off) cudaFreeHost(sl.off);
      if (sl.idx) cudaFreeHost(sl.idx);
      if (sl.dense) cudaFreeHost(sl.dense);
      if (sl.scores) cudaFreeHost(sl.scores);
      if (sl.ev) cudaEventDestroy(sl.ev);
    }
  };
  if (e != cudaSuccess) {
    release();
    return CVR_E_CUDA;
  }
  Batcher b{cfg->window_s, MI, cfg->max_requests, cfg->queue_capacity, {}, 0, 0, t_arrival, n_items};
  for (int r = 0; r < n_req; ++r) latency[r] = std::numeric_limits<double>::quiet_NaN();
  std::deque<int> free_slots, inflight;
  for (int s = 0; s < S; ++s) free_slots.push_back(s);
  std::vector<int> batch;
  std::vector<int32_t> ids;
  // warm-up before the trace clock starts: one small batch through every slot pays the one-time costs (OpenMP team
  // creation, first touch of the staging pages, the executor's first calls) outside the measured trace
  if (n_req > 0) {
    for (int s = 0; s < S; ++s) {
      Slot& sl = slots[s];
      int64_t nnz = 0;
      const int n0 = std::min<int>(n_items[0], MI);
      int st0 = cvr_gather_items(n_tables, n_dense, pool_size, pool_offsets, pool_indices, pool_dense, n0,
                                 item_ids + item_start[0], MI, sl.off, sl.idx, cfg->max_nnz, sl.dense, &nnz);
      if (st0 == CVR_OK)
        st0 = cvr_score_host(ctx, sl.idx, sl.off, nnz, n0, sl.dense, sl.scores, s_copy, s_embed, s_dense);
      if (st0 != CVR_OK) {
        release();
        return st0;
      }
    }
    cudaStreamSynchronize((cudaStream_t)s_dense);
  }
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now() + std::chrono::milliseconds(10);
  auto now_s = [&]() { return std::chrono::duration<double>(clk::now() - t0).count(); };
  int i = 0, done = 0, nb = 0, st = CVR_OK;
  double busy_host = 0.0, max_dispatch = 0.0, max_gather = 0.0, last_iter = -1.0;
  int64_t items_served = 0, gaps = 0;
  bool aborted = false;
  while (done < n_req) {
    double now = now_s();
    if (last_iter >= 0.0 && now - last_iter > 1e-3) ++gaps;
    last_iter = now;
    if (cfg->abort_after_s > 0 && !b.q.empty() && now - t_arrival[b.q.front()] > cfg->abort_after_s) {
      aborted = true;  // overloaded: the oldest request has waited too long -- stop this point
      break;
    }
    while (i < n_req && t_arrival[i] <= now) {
      if (!b.submit(i)) {
        latency[i] = std::numeric_limits<double>::infinity();
        ++done;
      }
      ++i;
    }
    while (!inflight.empty()) {  // retire finished batches in order
      Slot& sl = slots[inflight.front()];
      const cudaError_t q = cudaEventQuery(sl.ev);
      if (q == cudaErrorNotReady) break;
      if (q != cudaSuccess) {
        st = CVR_E_CUDA;
        break;
      }
      const double t_done = now_s();
      int64_t row = 0;
      for (int r : sl.reqs) {
        latency[r] = t_done - t_arrival[r];
        if (scores_out) memcpy(scores_out + item_start[r], sl.scores + row, (size_t)n_items[r] * 4);
        row += n_items[r];
      }
      done += (int)sl.reqs.size();
      free_slots.push_back(inflight.front());
      inflight.pop_front();
    }
    if (st != CVR_OK) break;
    if (!free_slots.empty() && b.poll(now_s(), batch)) {
      const auto h0 = clk::now();
      const int s = free_slots.front();
      free_slots.pop_front();
      Slot& sl = slots[s];
      sl.reqs = batch;
      ids.clear();
      for (int r : batch) ids.insert(ids.end(), item_ids + item_start[r], item_ids + item_start[r] + n_items[r]);
      int64_t nnz = 0;
      st = cvr_gather_items(n_tables, n_dense, pool_size, pool_offsets, pool_indices, pool_dense, (int)ids.size(),
                            ids.data(), MI, sl.off, sl.idx, cfg->max_nnz, sl.dense, &nnz);
      const auto h1 = clk::now();
      max_gather = std::max(max_gather, std::chrono::duration<double>(h1 - h0).count());
      if (st == CVR_OK)
        st = cvr_score_host(ctx, sl.idx, sl.off, nnz, (int)ids.size(), sl.dense, sl.scores, s_copy, s_embed, s_dense);
      if (st == CVR_OK && cudaEventRecord(sl.ev, (cudaStream_t)s_dense) != cudaSuccess) st = CVR_E_CUDA;
      if (st != CVR_OK) break;
      batch_sizes[nb++] = (int32_t)ids.size();
      items_served += (int64_t)ids.size();
      inflight.push_back(s);
      const double dt = std::chrono::duration<double>(clk::now() - h0).count();
      busy_host += dt;
      max_dispatch = std::max(max_dispatch, dt);
      last_iter = now_s();
      continue;
    }
    if (i >= n_req && b.q.empty() && inflight.empty()) break;
  }
  cudaStreamSynchronize((cudaStream_t)s_dense);
  for (int r = 0; r < n_req; ++r)
    if (std::isnan(latency[r])) latency[r] = std::numeric_limits<double>::infinity();
  *n_batches = nb;
  stats->rejected = b.rejected;
  stats->aborted = aborted ? 1 : 0;
  stats->items_served = items_served;
  stats->host_dispatch_s = busy_host;
  stats->wall_s = now_s();
  stats->max_dispatch_s = max_dispatch;
  stats->max_gather_s = max_gather;
  stats->loop_gaps_1ms = gaps;
  release();
  return st;
}

}  // extern "C"
