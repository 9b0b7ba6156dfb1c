// Device-initiated survivor rebalancing (drb.cu); internal to libdycl.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace dycl {

constexpr int DRB_MAX_WORLD = 8;            // one NVLink / NVSwitch domain
constexpr int DRB_MAX_LEVELS = 8;           // rebalanced exits per run

// Head of every rank's window (symmetric; zero-initialised; 64-bit words: epoch << 32 | value).
struct DrbCtrl {
  unsigned long long cnt[DRB_MAX_LEVELS][2][DRB_MAX_WORLD];     // (epoch, survivor count) per source
  unsigned long long ready[DRB_MAX_LEVELS][2][DRB_MAX_WORLD];   // rows of this level stored by source
  unsigned long long ret[DRB_MAX_LEVELS][2][DRB_MAX_WORLD];     // results of this level stored by source
};

// One level's plan for this rank (computed on the device from every rank's count).
struct DrbPlan {
  int s_own, keep, n_send, n_recv, new_count;
  int send[DRB_MAX_WORLD], recv[DRB_MAX_WORLD];
  int send_begin[DRB_MAX_WORLD];            // first index of my rows for destination j in my send list
  int recv_off[DRB_MAX_WORLD];              // first row of source j's rows in my row region
  int dst_off[DRB_MAX_WORLD];               // first row of my rows in destination j's row region
  int src_pos[DRB_MAX_WORLD];               // first index of the rows source j sent me in j's send list
};

struct DrbArgs {
  int rank, world, level, max_rows, K;
  void* const* peers;                       // device [world]: every rank's window base (as seen here)
  size_t rows_off, ret_off;                 // byte offsets of the row / return regions in a window
  unsigned* epoch;                          // device: this run's epoch (k_drb_begin)
  int* err;                                 // device: 0 or the first timeout / overflow code
  int* ticket;                              // device: last-CTA ticket of the push kernels
  DrbPlan* plan;                            // device [DRB_MAX_LEVELS]
  int* cnt;                                 // device live-row count of the level (in: survivors, out: held)
  // payload: row i of the level's tensor = plane_b row (bf16) + plane_f row (fp32 / lo), 16 B multiples
  uint8_t* plane_b;
  uint8_t* plane_f;
  long long plane_b_bytes, plane_f_bytes, row_bytes;
  int* orig;                                // row -> result-space id (in / out)
  int* sent_orig;                           // this level's sent rows' result-space ids
  long long gid_base;                       // global index of own row 0
  int own;                                  // own rows (result space [0, own))
  int ext0;                                 // result-space id of the first row received at this level
  long long* ext_gid;                       // global ids of foreign rows (indexed id - own)
  int32_t* res_path;
  float* res_margin;
  float* res_logits;
};

cudaError_t drb_begin(unsigned* epoch, cudaStream_t s);
cudaError_t drb_counts(const DrbArgs& a, cudaStream_t s);
cudaError_t drb_push(const DrbArgs& a, int num_sms, cudaStream_t s);
cudaError_t drb_wait(const DrbArgs& a, int ret, cudaStream_t s);
cudaError_t drb_pull(const DrbArgs& a, int num_sms, cudaStream_t s);
cudaError_t drb_ret_push(const DrbArgs& a, int num_sms, cudaStream_t s);
cudaError_t drb_ret_pull(const DrbArgs& a, int num_sms, cudaStream_t s);
// NCCL: table_dev[p] = ncclGetPeerPointer(window, 0, p) for p < world
cudaError_t drb_nccl_peers(void* nccl_window, int world, void** table_dev, cudaStream_t s);

}  // namespace dycl
