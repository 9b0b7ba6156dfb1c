// Device-initiated survivor rebalancing: the exchange after an exit runs as
// kernels that store straight into the other ranks' windows -- no host synchronisation, no
// host-side plan, no NCCL host calls on the run's critical path.
//
// Every rank owns one symmetric device window (NCCL: ncclMemAlloc + ncclCommWindowRegister,
// peers addressed through the LSA pointers of NVLink / NVSwitch; the in-process transport:
// plain device buffers of the graphs of one process).  Window layout (DrbWin):
//   ctrl   per level and parity: every source's (epoch, survivor count) word, data-ready epoch
//          and results-ready epoch (a rank runs at most one exchange ahead of another, so two
//          parity slots keep a fast rank from overwriting a value a slow one has not read)
//   rows   [max_batch] received rows: the next sub-network's input planes + 16 B of metadata
//   ret    [levels][max_batch] returned results: K logits, path, margin
// Per rebalanced exit (level k):
//   k_drb_counts  (1 thread)  publish (epoch, count) to every rank, wait for all, compute every
//                             rank's plan (the plan of dycl_rebalance_plan), keep this rank's
//   k_drb_push    (grid)      the surplus rows (the LAST n_send survivors, destination rank
//                             ascending) into the destinations' row regions; the last CTA to
//                             finish (ticket) publishes data-ready to each destination
//   k_drb_wait    (1 thread)  wait for the data-ready words of this rank's sources
//   k_drb_pull    (grid)      received rows into the activation buffers after the own survivors,
//                             metadata to the result space; the live count becomes new_count
// End of the run (levels last first): k_drb_ret_push results of the rows received at level k to
// their sources' ret regions + results-ready; k_drb_wait; k_drb_ret_pull scatters the returned
// results of this rank's sent rows to their result-space ids.
// Ordering: data stores, __threadfence_system(), then the flag store (st.release.sys); readers
// spin with ld.acquire.sys.  Every wait is bounded (~20 s of clock64) and records an error code
// instead of hanging.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>

#include "drb.h"

namespace dycl {
namespace {

__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

constexpr long long SPIN_LIMIT = 40000000000ll;      // clock64 cycles (~20 s)

// wait until *p >> 32 >= e (epochs only grow); false (and *err set) on timeout
__device__ bool wait_epoch(const unsigned long long* p, unsigned e, int* err, int code) {
  const long long t0 = clock64();
  while ((unsigned)(ld_acq(p) >> 32) < e) {
    if (clock64() - t0 > SPIN_LIMIT) {
      atomicExch(err, code);
      return false;
    }
  }
  return true;
}

__device__ __forceinline__ DrbCtrl* ctrl_of(void* win) { return reinterpret_cast<DrbCtrl*>(win); }

__global__ void k_drb_begin(unsigned* epoch) { epoch[0] += 1; }

__global__ void k_drb_counts(const DrbArgs a) {
  if (threadIdx.x != 0) return;
  const unsigned e = *a.epoch;
  const int W = a.world, me = a.rank, lv = a.level, par = e & 1;
  const int count = *a.cnt;
  const unsigned long long word = ((unsigned long long)e << 32) | (unsigned)count;
  for (int j = 0; j < W; ++j) st_rel(&ctrl_of(a.peers[j])->cnt[lv][par][me], word);
  DrbCtrl* mine = ctrl_of(a.peers[me]);
  int counts[DRB_MAX_WORLD];
  for (int j = 0; j < W; ++j) {
    if (!wait_epoch(&mine->cnt[lv][par][j], e, a.err, 1)) return;
    counts[j] = (int)(unsigned)(ld_acq(&mine->cnt[lv][par][j]) & 0xffffffffull);
  }
  // every rank's plan: target T = ceil(S / W); surplus ranks give their LAST (c - T) rows, in
  // order, to deficit ranks matched in rank order (surplus ascending x deficit ascending)
  long long S = 0;
  for (int j = 0; j < W; ++j) S += counts[j];
  const int T = (int)((S + W - 1) / W);
  int give[DRB_MAX_WORLD], need[DRB_MAX_WORLD];
  for (int j = 0; j < W; ++j) {
    give[j] = counts[j] > T ? counts[j] - T : 0;
    need[j] = counts[j] < T ? T - counts[j] : 0;
  }
  int flow[DRB_MAX_WORLD][DRB_MAX_WORLD];               // flow[s][d] rows from s to d
  for (int s = 0; s < W; ++s)
    for (int d = 0; d < W; ++d) flow[s][d] = 0;
  int s = 0, d = 0;
  while (s < W && d < W) {
    if (give[s] == 0) { ++s; continue; }
    if (need[d] == 0) { ++d; continue; }
    const int m = give[s] < need[d] ? give[s] : need[d];
    flow[s][d] += m;
    give[s] -= m;
    need[d] -= m;
  }
  DrbPlan P{};
  P.s_own = counts[me];
  int ns = 0, nr = 0;
  for (int j = 0; j < W; ++j) {
    P.send[j] = flow[me][j];
    P.recv[j] = flow[j][me];
    P.send_begin[j] = ns;                              // my send list: destination ascending
    P.recv_off[j] = nr;                                // my row region: source ascending
    // where my rows land in j's row region (after the rows of j's lower-ranked sources)
    int off = 0;
    for (int q = 0; q < me; ++q) off += flow[q][j];
    P.dst_off[j] = off;
    // where the rows j sent me sit in j's send list (for the return path)
    int pos = 0;
    for (int q = 0; q < me; ++q) pos += flow[j][q];
    P.src_pos[j] = pos;
    ns += flow[me][j];
    nr += flow[j][me];
  }
  P.n_send = ns;
  P.n_recv = nr;
  P.keep = P.s_own - ns;
  P.new_count = P.keep + nr;
  if (P.new_count > a.max_rows) {
    atomicExch(a.err, 2);
    P.n_send = P.n_recv = 0;
    P.new_count = P.s_own;
    P.keep = P.s_own;
  }
  a.plan[lv] = P;
}

// thread per 16-byte chunk of the outgoing payload; row layout in a window: [planes | meta]
__global__ void k_drb_push(const DrbArgs a) {
  const DrbPlan& P = a.plan[a.level];
  const unsigned e = *a.epoch;
  const int row_chunks = (int)(a.row_bytes / 16);
  const long long total = (long long)P.n_send * (row_chunks + 1);
  for (long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x; u < total; u += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(u / (row_chunks + 1)), c = (int)(u - (long long)i * (row_chunks + 1));
    int j = 0;                                         // destination of send index i
    while (j + 1 < a.world && (P.send[j] == 0 || i >= P.send_begin[j] + P.send[j])) ++j;
    const int src_row = P.keep + i;
    const long long drow = P.dst_off[j] + (i - P.send_begin[j]);
    uint8_t* dst = reinterpret_cast<uint8_t*>(a.peers[j]) + a.rows_off + drow * (long long)(a.row_bytes + 16);
    if (c < row_chunks) {
      const long long byte = (long long)c * 16;
      const uint8_t* src = byte < a.plane_b_bytes
                               ? a.plane_b + (size_t)src_row * a.plane_b_bytes + byte
                               : a.plane_f + (size_t)src_row * a.plane_f_bytes + (byte - a.plane_b_bytes);
      *reinterpret_cast<uint4*>(dst + byte) = *reinterpret_cast<const uint4*>(src);
    } else {
      const int o = a.orig[src_row];
      a.sent_orig[i] = o;
      const long long gid = o < a.own ? a.gid_base + o : a.ext_gid[o - a.own];
      int4 m;
      m.x = a.res_path[o];
      m.y = a.res_margin ? __float_as_int(a.res_margin[o]) : 0x7f800000;
      m.z = (int)(gid & 0xffffffffll);
      m.w = (int)(gid >> 32);
      *reinterpret_cast<int4*>(dst + a.row_bytes) = m;
    }
  }
  // last CTA out publishes data-ready (epoch) to every destination of this level
  __threadfence_system();
  __syncthreads();
  __shared__ int last;
  if (threadIdx.x == 0) last = atomicAdd(a.ticket, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (last && threadIdx.x == 0) {
    *a.ticket = 0;
    __threadfence_system();
    for (int j = 0; j < a.world; ++j)
      if (P.send[j] > 0)
        st_rel(&ctrl_of(a.peers[j])->ready[a.level][e & 1][a.rank], (unsigned long long)e << 32);
  }
}

// wait for the data-ready (ret == 0) or results-ready (ret == 1) words of this rank's sources
__global__ void k_drb_wait(const DrbArgs a, int ret) {
  if (threadIdx.x != 0) return;
  const DrbPlan& P = a.plan[a.level];
  const unsigned e = *a.epoch;
  DrbCtrl* mine = ctrl_of(a.peers[a.rank]);
  for (int j = 0; j < a.world; ++j) {
    const int n = ret ? P.send[j] : P.recv[j];
    if (n == 0) continue;
    if (!wait_epoch(ret ? &mine->ret[a.level][e & 1][j] : &mine->ready[a.level][e & 1][j], e, a.err, 3 + ret)) return;
  }
}

// received rows -> activation rows [s_own, new_count), metadata -> result space; live count
__global__ void k_drb_pull(const DrbArgs a) {
  const DrbPlan& P = a.plan[a.level];
  const int row_chunks = (int)(a.row_bytes / 16);
  const long long total = (long long)P.n_recv * (row_chunks + 1);
  const uint8_t* win = reinterpret_cast<const uint8_t*>(a.peers[a.rank]) + a.rows_off;
  for (long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x; u < total; u += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(u / (row_chunks + 1)), c = (int)(u - (long long)r * (row_chunks + 1));
    const uint8_t* src = win + (long long)r * (a.row_bytes + 16);
    const int drow = P.s_own + r;
    if (c < row_chunks) {
      const long long byte = (long long)c * 16;
      uint8_t* dst = byte < a.plane_b_bytes ? a.plane_b + (size_t)drow * a.plane_b_bytes + byte
                                            : a.plane_f + (size_t)drow * a.plane_f_bytes + (byte - a.plane_b_bytes);
      *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(src + byte);
    } else {
      const int4 m = *reinterpret_cast<const int4*>(src + a.row_bytes);
      const int o = a.ext0 + r;
      a.orig[drow] = o;
      a.res_path[o] = m.x;
      if (a.res_margin) a.res_margin[o] = __int_as_float(m.y);
      a.ext_gid[o - a.own] = (long long)(uint32_t)m.z | ((long long)m.w << 32);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.cnt = P.new_count;
}

// results of the rows received at this level (ids ext0 + r) back to their sources' ret regions
__global__ void k_drb_ret_push(const DrbArgs a) {
  const DrbPlan& P = a.plan[a.level];
  const unsigned e = *a.epoch;
  const int K = a.K;
  const int rec = K + 4;                               // floats per returned row (K, path, margin, pad)
  for (long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x; u < (long long)P.n_recv * rec;
       u += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(u / rec), c = (int)(u - (long long)r * rec);
    int j = 0;                                         // source of received row r
    while (j + 1 < a.world && (P.recv[j] == 0 || r >= P.recv_off[j] + P.recv[j])) ++j;
    const long long pos = P.src_pos[j] + (r - P.recv_off[j]);   // index in j's send list
    float* dst = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(a.peers[j]) + a.ret_off) +
                 ((size_t)a.level * a.max_rows + pos) * rec;
    const int o = a.ext0 + r;
    if (c < K) dst[c] = a.res_logits[(size_t)o * K + c];
    else if (c == K) dst[c] = __int_as_float(a.res_path[o]);
    else if (c == K + 1) dst[c] = a.res_margin ? a.res_margin[o] : __int_as_float(0x7f800000);
  }
  __threadfence_system();
  __syncthreads();
  __shared__ int last;
  if (threadIdx.x == 0) last = atomicAdd(a.ticket, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (last && threadIdx.x == 0) {
    *a.ticket = 0;
    __threadfence_system();
    for (int j = 0; j < a.world; ++j)
      if (P.recv[j] > 0)
        st_rel(&ctrl_of(a.peers[j])->ret[a.level][e & 1][a.rank], (unsigned long long)e << 32);
  }
}

// this rank's sent rows: returned results -> their result-space ids
__global__ void k_drb_ret_pull(const DrbArgs a) {
  const DrbPlan& P = a.plan[a.level];
  const int K = a.K, rec = K + 4;
  const float* src = reinterpret_cast<const float*>(reinterpret_cast<const uint8_t*>(a.peers[a.rank]) + a.ret_off) +
                     (size_t)a.level * a.max_rows * rec;
  for (long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x; u < (long long)P.n_send * rec;
       u += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(u / rec), c = (int)(u - (long long)i * rec);
    const int o = a.sent_orig[i];
    const float v = src[(size_t)i * rec + c];
    if (c < K) a.res_logits[(size_t)o * K + c] = v;
    else if (c == K) a.res_path[o] = __float_as_int(v);
    else if (c == K + 1 && a.res_margin) a.res_margin[o] = v;
  }
}

__global__ void k_nccl_peers(ncclWindow_t w, int world, void** table) {
  const int p = threadIdx.x;
  if (p < world) table[p] = ncclGetPeerPointer(w, 0, p);
}

int grid_for(long long work, int num_sms) {
  long long b = (work + 255) / 256;
  const long long cap = (long long)num_sms * 8;
  if (b > cap) b = cap;
  return b < 1 ? 1 : (int)b;
}

}  // namespace

cudaError_t drb_begin(unsigned* epoch, cudaStream_t s) {
  k_drb_begin<<<1, 1, 0, s>>>(epoch);
  return cudaGetLastError();
}
cudaError_t drb_counts(const DrbArgs& a, cudaStream_t s) {
  k_drb_counts<<<1, 32, 0, s>>>(a);
  return cudaGetLastError();
}
// grids are sized for the largest possible transfer (the host does not know the plan)
cudaError_t drb_push(const DrbArgs& a, int num_sms, cudaStream_t s) {
  k_drb_push<<<grid_for((long long)a.max_rows * (a.row_bytes / 16 + 1), num_sms), 256, 0, s>>>(a);
  return cudaGetLastError();
}
cudaError_t drb_wait(const DrbArgs& a, int ret, cudaStream_t s) {
  k_drb_wait<<<1, 32, 0, s>>>(a, ret);
  return cudaGetLastError();
}
cudaError_t drb_pull(const DrbArgs& a, int num_sms, cudaStream_t s) {
  k_drb_pull<<<grid_for((long long)a.max_rows * (a.row_bytes / 16 + 1), num_sms), 256, 0, s>>>(a);
  return cudaGetLastError();
}
cudaError_t drb_ret_push(const DrbArgs& a, int num_sms, cudaStream_t s) {
  k_drb_ret_push<<<grid_for((long long)a.max_rows * (a.K + 4), num_sms), 256, 0, s>>>(a);
  return cudaGetLastError();
}
cudaError_t drb_ret_pull(const DrbArgs& a, int num_sms, cudaStream_t s) {
  k_drb_ret_pull<<<grid_for((long long)a.max_rows * (a.K + 4), num_sms), 256, 0, s>>>(a);
  return cudaGetLastError();
}
cudaError_t drb_nccl_peers(void* nccl_window, int world, void** table_dev, cudaStream_t s) {
  k_nccl_peers<<<1, 32, 0, s>>>(reinterpret_cast<ncclWindow_t>(nccl_window), world, table_dev);
  return cudaGetLastError();
}

// Lazy-loading anchor: a kernel of this translation unit's module (preload_kernels, hostmod.cu).
__global__ void k_tu_anchor_drb() {}
const void* tu_anchor_drb() { return reinterpret_cast<const void*>(&k_tu_anchor_drb); }

}  // namespace dycl
