// Transports for survivor rebalancing across ranks; internal to libdycl.
//
// A transport moves bytes between the ranks of one job: an all-gather of one int32 per rank
// (the survivor counts; returns them on the host -- the one host synchronisation of a
// rebalancing step) and a grouped point-to-point exchange (every rank posts all its sends and
// receives of the step at once, so no ordering between peers can deadlock).
//   NcclTransport : ncclAllGather + grouped ncclSend / ncclRecv on the run's stream over a
//                   caller-provided communicator (NVLink / NVSwitch between B200s).  NCCL is
//                   resolved at run time from the libnccl.so.2 already mapped in the process
//                   (torch's), so libdycl has no link-time NCCL dependency.
//   LocalTransport: ranks that are graphs of ONE process, each driven by its own host thread
//                   (same or different devices): host barrier + device-to-device copies.  Used
//                   to test the rebalancing protocol with world > 1 on a single GPU.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

namespace dycl {

struct Transport {
  int rank = 0, world = 1;
  struct Msg {
    int peer;
    void* ptr;        // device buffer (sends: read, receives: written)
    size_t bytes;
  };
  virtual ~Transport() {}
  // host_out[r] = the int32 at dev_val on rank r, for every rank; synchronises `st`.
  virtual bool allgather_int(const int* dev_val, int* host_out, cudaStream_t st, std::string* err) = 0;
  // Post all sends and receives of one step; completion is stream-ordered on `st`.
  virtual bool exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t st,
                        std::string* err) = 0;
  // Device windows for device-initiated rebalancing (drb.cu).  Collective: every
  // rank calls it with the same size at the same point of its run sequence (the first device-
  // rebalanced exit).  *local = this rank's window (zeroed), *peers_dev = device array [world] of
  // every rank's window base as addressable from this rank's kernels (NCCL: the LSA pointers of a
  // registered symmetric window over NVLink; in-process: the graphs' own buffers).
  virtual bool window(size_t bytes, void** local, void*** peers_dev, std::string* err) = 0;
};

// nccl_comm: an ncclComm_t (borrowed, not destroyed).  nullptr + *err on failure.
Transport* make_nccl_transport(void* nccl_comm, int rank, int world, std::string* err);

struct LocalGroup;
LocalGroup* local_group_create(int world);
void local_group_destroy(LocalGroup* g);
int local_group_world(const LocalGroup* g);
Transport* make_local_transport(LocalGroup* g, int rank);

// NCCL helpers for callers without their own communicator (dycl_nccl_*).
bool nccl_get_unique_id(uint8_t out[128], std::string* err);
bool nccl_comm_init_rank(const uint8_t id[128], int rank, int world, void** comm, std::string* err);
bool nccl_comm_destroy(void* comm, std::string* err);

}  // namespace dycl
