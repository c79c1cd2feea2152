// CUDA-graph replay of PCG iteration chunks.
//
// One lsg_pcg_iterate(niter) call is niter (2D) or 3*niter (3D) kernel launches whose arguments
// depend only on (operator, workspace, parity, niter).  The first call with a
// given argument set is captured on a private stream (capture records, it does
// not execute) and instantiated; every call launches the instantiated graph on
// the caller's stream, which removes the per-kernel CPU launch cost -- the
// limiter for small grids (cfg1, cfg3, the k = 1 velocity solves).  Converged
// right-hand sides still freeze inside the kernels, so replaying a chunk past
// convergence is harmless.  A small LRU cache bounds the number of live graphs.
//
// Every outer iteration builds a new operator (new material words, new inverse
// diagonal), so the exact argument set changes while the graph's shape (kind,
// grid, k, parity, niter) does not: a miss on the exact key first re-captures
// (host recording only) and updates an executable graph of the same shape in
// place (cudaGraphExecUpdate), which is much cheaper than instantiating again.
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <chrono>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "ops.h"

namespace lsg {

namespace {

struct Key {
  lsg_op op;
  lsg_pcg_ws ws;  // includes the parity at entry
  int niter;
};

struct Shape {  // what fixes the graph topology and the kernels in it
  int kind, k, parity, niter;
  lsg_grid grid;
};

struct Entry {
  Key key;
  Shape shape;
  cudaGraphExec_t exec;
  unsigned long long last_use;
};

std::mutex g_mu;
std::vector<Entry> g_cache;
unsigned long long g_clock = 0;
constexpr int kMaxDev = 64;
cudaStream_t g_capture[kMaxDev] = {};  // one private capture stream per device
constexpr size_t kMaxGraphs = 32;
double g_stats[4] = {0, 0, 0, 0};  // hits, in-place updates, instantiations, host seconds

bool same(const Key &a, const Key &b) { return memcmp(&a, &b, sizeof(Key)) == 0; }
bool same(const Shape &a, const Shape &b) { return memcmp(&a, &b, sizeof(Shape)) == 0; }

bool graphs_off() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("LSG_NO_GRAPHS");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

}  // namespace

int num_sms() {
  constexpr int kMaxDev = 64;
  static int cache[kMaxDev] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return 148;
  if (cache[dev] <= 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    cache[dev] = v;
  }
  return cache[dev];
}

int64_t l2_bytes() {
  constexpr int kMaxDev = 64;
  static int64_t cache[kMaxDev] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return 126ll << 20;
  if (cache[dev] <= 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, dev) != cudaSuccess || v <= 0) v = 126 << 20;
    cache[dev] = v;
  }
  return cache[dev];
}

// 3D rotates three direction buffers (phase = iteration index mod 3), 2D two
void advance_parity(const lsg_op &op, lsg_pcg_ws &ws, int niter) {
  if (op.grid.dim == 3) ws.parity = (ws.parity + niter) % 3;
  else ws.parity ^= (niter & 1);
}

void graph_stats(double *out) {
  std::lock_guard<std::mutex> lock(g_mu);
  for (int i = 0; i < 4; ++i) out[i] = g_stats[i];
}

int pcg_iterate_graph(const lsg_op &op, lsg_pcg_ws &ws, int niter, cudaStream_t st) {
  if (niter <= 0) return LSG_OK;
  if (graphs_off() || (op.grid.dim == 2 && d2::pcg_persistent_ok(op, ws)))  // one launch already
    return (op.grid.dim == 2) ? d2::pcg_iterate(op, ws, niter, st) : d3::pcg_iterate(op, ws, niter, st);
  Key key;
  memset(&key, 0, sizeof(key));
  key.op = op;
  key.ws = ws;
  key.niter = niter;
  Shape shape;
  memset(&shape, 0, sizeof(shape));
  shape.kind = op.kind;
  shape.k = ws.k;
  shape.parity = ws.parity;
  shape.niter = niter;
  shape.grid = op.grid;
  std::lock_guard<std::mutex> lock(g_mu);
  for (auto &e : g_cache) {
    if (same(e.key, key)) {
      e.last_use = ++g_clock;
      g_stats[0] += 1;
      if (cudaGraphLaunch(e.exec, st) != cudaSuccess) return check_launch("graph launch");
      advance_parity(op, ws, niter);
      return check_launch("graph launch");
    }
  }
  const auto t0 = std::chrono::steady_clock::now();
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return check_launch("device");
  cudaStream_t &cap = g_capture[dev];
  if (!cap && cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking) != cudaSuccess)
    return check_launch("capture stream");
  lsg_pcg_ws tmp = ws;
  if (cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
    return check_launch("begin capture");
  int rc = (op.grid.dim == 2) ? d2::pcg_iterate(op, tmp, niter, cap)
                              : d3::pcg_iterate(op, tmp, niter, cap);
  cudaGraph_t graph = nullptr;
  cudaError_t ec = cudaStreamEndCapture(cap, &graph);
  if (rc != LSG_OK) {
    if (graph) cudaGraphDestroy(graph);
    return rc;
  }
  if (ec != cudaSuccess) return check_launch("end capture");
  // same shape, other arguments: update an executable graph in place
  Entry *best = nullptr;
  for (auto &e : g_cache)
    if (same(e.shape, shape) && (!best || e.last_use < best->last_use)) best = &e;
  if (best) {
    cudaGraphExecUpdateResultInfo info;
    if (cudaGraphExecUpdate(best->exec, graph, &info) == cudaSuccess) {
      cudaGraphDestroy(graph);
      best->key = key;
      best->last_use = ++g_clock;
      g_stats[1] += 1;
      g_stats[3] += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (cudaGraphLaunch(best->exec, st) != cudaSuccess) return check_launch("graph launch");
      advance_parity(op, ws, niter);
      return check_launch("graph launch");
    }
    cudaGetLastError();  // clear the failed update; instantiate instead
    static const bool dbg = getenv("LSG_GRAPH_DEBUG") != nullptr;
    if (dbg)
      fprintf(stderr, "lsg graph: in-place update refused (result %d, dim %d, k %d, parity %d, niter %d)\n",
              (int)info.result, op.grid.dim, ws.k, ws.parity, niter);
  }
  cudaGraphExec_t exec = nullptr;
  ec = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ec != cudaSuccess) return check_launch("graph instantiate");
  g_stats[2] += 1;
  g_stats[3] += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (g_cache.size() >= kMaxGraphs) {
    size_t victim = 0;
    for (size_t i = 1; i < g_cache.size(); ++i)
      if (g_cache[i].last_use < g_cache[victim].last_use) victim = i;
    cudaGraphExecDestroy(g_cache[victim].exec);
    g_cache.erase(g_cache.begin() + victim);
  }
  g_cache.push_back(Entry{key, shape, exec, ++g_clock});
  if (cudaGraphLaunch(exec, st) != cudaSuccess) return check_launch("graph launch");
  advance_parity(op, ws, niter);
  return check_launch("graph launch");
}

}  // namespace lsg
