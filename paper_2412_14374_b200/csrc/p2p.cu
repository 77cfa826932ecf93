// NCCL point-to-point channels over NVLink 5 / NVSwitch.
//
// Replaces the reference's in-process FIFO Channel (executor.py:201-254):
//   Channel.send          -> pc_p2p_send  (posted at SendStart on the channel's send stream)
//   Channel.recv          -> pc_p2p_recv  (posted at RecvStart: real prefetch;
//                                          the reference's RecvStart is a no-op, :369-370)
//   watchdog abort         -> pc_p2p_abort (a dropped recv otherwise hangs the GPU)
// Every directed channel (src, dst) gets its own 2-rank communicator and its
// own streams, so channels progress independently: the FIFO-per-directed-pair
// model under which comms.check_deadlock_free proves the plan safe
// (comms.py:331-339).
#include "common.cuh"

#if PP200_HAVE_NCCL
#include <nccl.h>
#endif

using namespace pp200;

#if PP200_HAVE_NCCL
#define PP_NCCL_TRY(expr)                                                     \
  do {                                                                        \
    ncclResult_t _r = (expr);                                                 \
    if (_r != ncclSuccess) {                                                  \
      set_error("%s: %s", #expr, ncclGetErrorString(_r));                     \
      return PC_ERR_NCCL;                                                     \
    }                                                                         \
  } while (0)
#endif

extern "C" int pc_p2p_available(void) {
#if PP200_HAVE_NCCL
  return 1;
#else
  return 0;
#endif
}

extern "C" int pc_p2p_unique_id(void* out128) {
#if PP200_HAVE_NCCL
  ncclUniqueId id;
  PP_NCCL_TRY(ncclGetUniqueId(&id));
  memcpy(out128, &id, sizeof(id));
  return PC_OK;
#else
  set_error("built without NCCL");
  return PC_ERR_UNSUPPORTED;
#endif
}

extern "C" int pc_p2p_comm_init(void** comm, int nranks, const void* id128, int rank) {
#if PP200_HAVE_NCCL
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  ncclComm_t c;
  PP_NCCL_TRY(ncclCommInitRank(&c, nranks, id, rank));
  *comm = c;
  return PC_OK;
#else
  set_error("built without NCCL");
  return PC_ERR_UNSUPPORTED;
#endif
}

extern "C" int pc_p2p_send(void* comm, const void* buf, int64_t bytes, int peer, void* stream) {
#if PP200_HAVE_NCCL
  PP_NCCL_TRY(ncclSend(buf, static_cast<size_t>(bytes), ncclInt8, peer,
                       static_cast<ncclComm_t>(comm), static_cast<cudaStream_t>(stream)));
  return PC_OK;
#else
  set_error("built without NCCL");
  return PC_ERR_UNSUPPORTED;
#endif
}

extern "C" int pc_p2p_recv(void* comm, void* buf, int64_t bytes, int peer, void* stream) {
#if PP200_HAVE_NCCL
  PP_NCCL_TRY(ncclRecv(buf, static_cast<size_t>(bytes), ncclInt8, peer,
                       static_cast<ncclComm_t>(comm), static_cast<cudaStream_t>(stream)));
  return PC_OK;
#else
  set_error("built without NCCL");
  return PC_ERR_UNSUPPORTED;
#endif
}

extern "C" int pc_p2p_abort(void* comm) {
#if PP200_HAVE_NCCL
  PP_NCCL_TRY(ncclCommAbort(static_cast<ncclComm_t>(comm)));
  return PC_OK;
#else
  return PC_OK;
#endif
}

extern "C" int pc_p2p_destroy(void* comm) {
#if PP200_HAVE_NCCL
  PP_NCCL_TRY(ncclCommDestroy(static_cast<ncclComm_t>(comm)));
  return PC_OK;
#else
  return PC_OK;
#endif
}
