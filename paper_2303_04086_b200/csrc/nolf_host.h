// nolf_host.h -- host side of the sparse frame delivery (nolf_host_scatter):
// packed live chunks (768 B each: 128 encoded pixels in slot order, rgba8
// then depth16) are written back into a row-major encode_frame RAW frame in
// host memory, and chunks written last time but not live now are reset to
// the miss encoding.  A small persistent thread pool splits the chunks.
#pragma once
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/nolf.h"

namespace nolf_host {

// Fixed pool; run(f, n) calls f(0..n-1) on the workers and the caller.
class Pool {
 public:
  explicit Pool(int n) {
    for (int i = 0; i < n; ++i) workers_.emplace_back([this] { loop(); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto &t : workers_) t.join();
  }
  int size() const { return (int)workers_.size() + 1; }
  void run(const std::function<void(int)> &f, int parts) {
    {
      std::lock_guard<std::mutex> g(m_);
      job_ = &f;
      parts_ = parts;
      next_.store(0);
      done_ = 0;
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> l(m_);
    done_cv_.wait(l, [&] { return done_ == parts_; });
    job_ = nullptr;
  }

 private:
  void work() {
    for (;;) {
      const int i = next_.fetch_add(1);
      if (i >= parts_) return;
      (*job_)(i);
      std::lock_guard<std::mutex> g(m_);
      if (++done_ == parts_) done_cv_.notify_all();
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> l(m_);
        cv_.wait(l, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      work();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex m_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)> *job_ = nullptr;
  std::atomic<int> next_{0};
  int parts_ = 0, done_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

inline Pool &pool(int want) {
  static Pool *p = nullptr;
  static std::mutex m;
  std::lock_guard<std::mutex> g(m);
  if (!p) {
    // default: half the host cores, shared by the ranks of this node (the
    // other half drives the GPUs; measured: 8 of 16 cores scatter a 4K frame
    // in ~200 us, 16 oversubscribe)
    int per = 1;
    if (const char *e = getenv("LOCAL_WORLD_SIZE")) per = atoi(e) > 0 ? atoi(e) : 1;
    int n = want > 0 ? want : (int)std::thread::hardware_concurrency() / (2 * per);
    if (const char *e = getenv("NOLF_HOST_THREADS")) n = atoi(e);
    n = n < 1 ? 1 : (n > 64 ? 64 : n);
    p = new Pool(n - 1);
  }
  return *p;
}

struct ScatterJob {
  const uint8_t *runs;         // 48 B per packed run
  const uint32_t *heads;       // per live chunk: {chunk id, run mask, first run}
  uint32_t n;
  const NolfTile *tiles;
  int32_t n_tiles;
  int64_t tile_stride;
  int32_t width, height;
  uint8_t *rgba8;
  uint16_t *depth16;
  uint16_t *dirty;             // per chunk of this frame buffer: runs holding non-miss bytes
};

// (x, y) of packed slot `local` in a w x h tile of 8x4 blocks (render.slot_xy).
inline void block_xy(int64_t local, int w, int &x, int &y) {
  const int64_t blk = local >> 5, l = local & 31, bx = w >> 3;
  x = (int)((blk % bx) * 8 + (l & 7));
  y = (int)((blk / bx) * 4 + (l >> 3));
}

// Write the runs of chunk `id`: bit r of `put` from payload run e + 48 * k
// (k-th set bit), bit r of `clear` to the miss encoding.
inline bool chunk_runs(const ScatterJob &J, uint32_t id, unsigned put, unsigned clear, const uint8_t *e) {
  const int64_t p0 = (int64_t)id * 128;
  const int64_t t = p0 / J.tile_stride, local0 = p0 % J.tile_stride;
  const NolfTile &tp = J.tiles[t];
  const int w = tp.x1 - tp.x0, h = tp.y1 - tp.y0;
  if ((w & 7) || (h & 3)) return false;
  static const uint8_t kMiss8[32] = {}, kMiss16[16] = {0xFF, 0xFF, 0xFF, 0xFF, 0xFF, 0xFF, 0xFF, 0xFF,
                                                        0xFF, 0xFF, 0xFF, 0xFF, 0xFF, 0xFF, 0xFF, 0xFF};
  const int64_t base = (int64_t)tp.cam * J.width * J.height;
  const unsigned any = put | clear;
  for (int r = 0; r < 16; ++r) {
    if (!((any >> r) & 1u)) continue;
    const int64_t local = local0 + 8 * r;
    if (local >= (int64_t)w * h) break;
    int x, y;
    block_xy(local, w, x, y);
    const int64_t q = base + (int64_t)(tp.y0 + y) * J.width + (tp.x0 + x);
    if ((put >> r) & 1u) {
      memcpy(J.rgba8 + 4 * q, e, 32);
      memcpy(J.depth16 + q, e + 32, 16);
      e += 48;
    } else {
      memcpy(J.rgba8 + 4 * q, kMiss8, 32);
      memcpy(J.depth16 + q, kMiss16, 16);
    }
  }
  return true;
}

inline int scatter(const ScatterJob &J, int n_threads) {
  Pool &P = pool(n_threads);
  const uint64_t n_chunks = (uint64_t)J.n_tiles * (uint64_t)(J.tile_stride / 128);
  // chunks live now (bitmap): dirty runs of the others are reset
  thread_local std::vector<uint64_t> live;
  live.assign((n_chunks + 63) / 64, 0ull);
  for (uint32_t i = 0; i < J.n; ++i) live[J.heads[3 * i] >> 6] |= 1ull << (J.heads[3 * i] & 63);
  const std::vector<uint64_t> &lv = live;    // the caller's copy (workers have their own thread_locals)
  const int parts = P.size() * 4;
  std::atomic<int> bad{0};
  const std::function<void(int)> f = [&](int part) {
    // live chunks: packed runs written, dirty runs that are misses now reset
    const uint64_t a = (uint64_t)J.n * part / parts, b = (uint64_t)J.n * (part + 1) / parts;
    for (uint64_t i = a; i < b; ++i) {
      const uint32_t id = J.heads[3 * i], mask = J.heads[3 * i + 1];
      const unsigned clear = J.dirty[id] & ~mask;
      if ((mask | clear) && !chunk_runs(J, id, mask, clear, J.runs + 48ull * J.heads[3 * i + 2])) bad = 1;
      J.dirty[id] = (uint16_t)mask;
    }
    // chunks not live now: reset their dirty runs
    const uint64_t c0 = n_chunks * part / parts, c1 = n_chunks * (part + 1) / parts;
    for (uint64_t c = c0; c < c1; ++c) {
      if (!J.dirty[c] || ((lv[c >> 6] >> (c & 63)) & 1ull)) continue;
      if (!chunk_runs(J, (uint32_t)c, 0u, J.dirty[c], nullptr)) bad = 1;
      J.dirty[c] = 0;
    }
  };
  P.run(f, parts);
  return bad.load();
}

}  // namespace nolf_host
