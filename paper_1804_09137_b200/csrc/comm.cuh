// comm.cuh — the collectives the 2D block-cyclic factorisation needs
// (SURVEY.md 8(e)), behind one small interface with two backends:
//
//   NCCL      one communicator per process row / column / world, over
//             NVLink / NVSwitch (ncclBroadcast / ncclAllReduce / ncclReduce)
//   loopback  W logical ranks inside one process, one host thread per rank
//             (their devices may coincide): a collective is a host rendezvous
//             of the members followed by stream-ordered device copies and a
//             fixed-order device sum.  No kernel ever waits on another rank —
//             cross-rank order is carried by cudaStreamWaitEvent only — so W
//             ranks may share one GPU.  Used to execute and test the
//             distributed schedule on one B200, and by single-process
//             multi-GPU handles when NCCL cannot take the device list.
//
// Every call is in place and stream ordered on `s`, like NCCL's.
#pragma once
#include "common.cuh"
#include <nccl.h>
#include <memory>

namespace tlrb {

enum class CType { I32, F64 };
inline size_t ctype_size(CType t) { return t == CType::I32 ? 4 : 8; }

class Comm {
 public:
  virtual ~Comm() = default;
  virtual int rank() const = 0;
  virtual int size() const = 0;
  virtual const char* kind() const = 0;
  // the root's buf is copied into every other member's buf
  virtual void bcast(void* buf, size_t count, CType t, int root, cudaStream_t s) = 0;
  // every member's buf <- sum over members (members sum in the same order)
  virtual void allreduce_sum(void* buf, size_t count, CType t, cudaStream_t s) = 0;
  // the root's buf <- sum over members; the others' buf is left unchanged
  virtual void reduce_sum(void* buf, size_t count, CType t, int root, cudaStream_t s) = 0;
  // abandon pending / future collectives (another member failed)
  virtual void abort() = 0;
};

// NCCL backend (takes ownership of the communicator)
std::unique_ptr<Comm> make_nccl_comm(ncclComm_t c);
// split an NCCL communicator (collective over the parent's members)
std::unique_ptr<Comm> split_nccl_comm(Comm& parent, int color, int key);

// loopback backend: one LocalGroup per communicator, shared by its members
struct LocalGroup;
std::shared_ptr<LocalGroup> make_local_group(int size);
std::unique_ptr<Comm> make_local_comm(std::shared_ptr<LocalGroup> g, int rank, int device);

}  // namespace tlrb
