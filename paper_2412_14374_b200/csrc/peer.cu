// NVLink peer-memory channels: the receiver owns one slot per plan message
// (CUDA IPC), the sender's producing kernel writes the message straight into
// that slot over NVLink (or a copy engine moves it when the value was not
// produced in place), and a flag word per message, written by a stream
// memory operation ordered after the producer, releases the receiver's
// stream (cuStreamWaitValue32).  Replaces the reference's Channel
// (executor.py:201-254) without a separate transfer on the critical path.
#include "common.cuh"

#include <cuda.h>

#include <vector>

using namespace pp200;

namespace {

using WriteFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using WaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

template <typename F>
F driver_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(p);
}

}  // namespace

extern "C" int pc_peer_alloc(int64_t bytes, void** ptr, void* handle64) {
  PP_CHECK_ARG(bytes > 0 && ptr && handle64, "peer_alloc: bad args");
  void* p = nullptr;
  PP_CUDA_TRY(cudaMalloc(&p, static_cast<size_t>(bytes)));
  PP_CUDA_TRY(cudaMemset(p, 0, static_cast<size_t>(bytes)));
  cudaIpcMemHandle_t h;
  PP_CUDA_TRY(cudaIpcGetMemHandle(&h, p));
  memcpy(handle64, &h, sizeof(h));
  *ptr = p;
  return PC_OK;
}

extern "C" int pc_peer_free(void* ptr) {
  PP_CUDA_TRY(cudaFree(ptr));
  return PC_OK;
}

extern "C" int pc_peer_open(const void* handle64, void** ptr) {
  PP_CHECK_ARG(handle64 && ptr, "peer_open: bad args");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  PP_CUDA_TRY(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return PC_OK;
}

extern "C" int pc_peer_close(void* ptr) {
  PP_CUDA_TRY(cudaIpcCloseMemHandle(ptr));
  return PC_OK;
}

// *addr = value once all prior work on the stream has completed (its memory
// writes, incl. stores into peer memory, visible first: default memory barrier).
extern "C" int pc_stream_write_u32(void* addr, uint32_t value, void* stream) {
  static WriteFn fn = driver_fn<WriteFn>("cuStreamWriteValue32");
  PP_CHECK_ARG(fn != nullptr, "cuStreamWriteValue32 unavailable");
  CUresult r = fn(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(addr), value, 0);
  if (r != CUDA_SUCCESS) {
    set_error("cuStreamWriteValue32 failed (%d)", static_cast<int>(r));
    return PC_ERR_CUDA;
  }
  return PC_OK;
}

// Later work on the stream waits until *addr == value.
extern "C" int pc_stream_wait_u32(void* addr, uint32_t value, void* stream) {
  static WaitFn fn = driver_fn<WaitFn>("cuStreamWaitValue32");
  PP_CHECK_ARG(fn != nullptr, "cuStreamWaitValue32 unavailable");
  CUresult r = fn(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(addr), value,
                  CU_STREAM_WAIT_VALUE_EQ);
  if (r != CUDA_SUCCESS) {
    set_error("cuStreamWaitValue32 failed (%d)", static_cast<int>(r));
    return PC_ERR_CUDA;
  }
  return PC_OK;
}

extern "C" int pc_peer_copy(void* dst, const void* src, int64_t bytes, void* stream) {
  if (bytes <= 0) return PC_OK;
  PP_CUDA_TRY(cudaMemcpyAsync(dst, src, static_cast<size_t>(bytes), cudaMemcpyDeviceToDevice,
                              static_cast<cudaStream_t>(stream)));
  return PC_OK;
}

// Kernel nodes of a captured CUDA graph (child graphs included): the number of
// kernels one replay of a captured step launches (bench.py gpu_launches).
// Driver API: the runtime's node-type query rejects stream-memop nodes.
using NodesFn = CUresult (*)(CUgraph, CUgraphNode*, size_t*);
using TypeFn = CUresult (*)(CUgraphNode, CUgraphNodeType*);
using ChildFn = CUresult (*)(CUgraphNode, CUgraph*);

static int count_kernel_nodes(CUgraph g, int64_t* n) {
  static NodesFn nodes_fn = driver_fn<NodesFn>("cuGraphGetNodes");
  static TypeFn type_fn = driver_fn<TypeFn>("cuGraphNodeGetType");
  static ChildFn child_fn = driver_fn<ChildFn>("cuGraphChildGraphNodeGetGraph");
  PP_CHECK_ARG(nodes_fn && type_fn && child_fn, "graph node queries unavailable");
  size_t num = 0;
  if (nodes_fn(g, nullptr, &num) != CUDA_SUCCESS) {
    set_error("cuGraphGetNodes failed");
    return PC_ERR_CUDA;
  }
  std::vector<CUgraphNode> nodes(num);
  if (num && nodes_fn(g, nodes.data(), &num) != CUDA_SUCCESS) {
    set_error("cuGraphGetNodes failed");
    return PC_ERR_CUDA;
  }
  for (CUgraphNode nd : nodes) {
    CUgraphNodeType t;
    if (type_fn(nd, &t) != CUDA_SUCCESS) continue;
    if (t == CU_GRAPH_NODE_TYPE_KERNEL) {
      ++*n;
    } else if (t == CU_GRAPH_NODE_TYPE_GRAPH) {
      CUgraph child;
      if (child_fn(nd, &child) == CUDA_SUCCESS)
        if (int rc = count_kernel_nodes(child, n)) return rc;
    }
  }
  return PC_OK;
}

extern "C" int pc_graph_kernel_nodes(void* graph, int64_t* n) {
  PP_CHECK_ARG(graph && n, "graph_kernel_nodes: bad args");
  *n = 0;
  return count_kernel_nodes(static_cast<CUgraph>(graph), n);
}

// RecvWait of the peer transport: one thread spins until the message flag
// (written over NVLink by the sender's stream after its producer) reads 1,
// re-arms it to 0, and exits; later work on the stream then reads the slot.
// Every 1024 polls it also reads an abort word in mapped host memory: the
// engine's watchdog sets it from the CPU (no stream, no CUDA call), so a wait
// on a message that will never arrive (dropped SendStart, dead peer) ends and
// the device drains -- a stream-memory-op wait cannot be released that way,
// since work queued to release it may share the blocked stream's hardware
// queue.  Graph-capturable (a kernel node).
__global__ void peer_wait_kernel(unsigned* flag, const volatile unsigned* abort_word) {
  if (threadIdx.x != 0) return;
  unsigned n = 0;
  while (ld_acquire_sys(flag) != 1u) {
    if ((++n & 1023u) == 0 && *abort_word != 0u) return;
    __nanosleep(64);
  }
  *flag = 0u;
}

extern "C" int pc_peer_wait(void* flag, const void* abort_word_dev, void* stream) {
  PP_CHECK_ARG(flag && abort_word_dev, "peer_wait: bad args");
  peer_wait_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<unsigned*>(flag), static_cast<const volatile unsigned*>(abort_word_dev));
  return check_launch("peer_wait_kernel");
}

// A zeroed 64-byte word in page-locked, device-mapped host memory: the host
// writes it with a plain store, kernels read it through *dev.
extern "C" int pc_host_word_alloc(void** host, void** dev) {
  PP_CHECK_ARG(host && dev, "host_word_alloc: bad args");
  void* h = nullptr;
  PP_CUDA_TRY(cudaHostAlloc(&h, 64, cudaHostAllocMapped | cudaHostAllocPortable));
  memset(h, 0, 64);
  PP_CUDA_TRY(cudaHostGetDevicePointer(dev, h, 0));
  *host = h;
  return PC_OK;
}

extern "C" int pc_host_word_free(void* host) {
  PP_CUDA_TRY(cudaFreeHost(host));
  return PC_OK;
}
