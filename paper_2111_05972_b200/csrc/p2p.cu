// p2p.cu — pipeline stage send/recv over NVLink peer memory (the D2D communicator of
// PAPER.md:337-350, modelled by mpsim comm.py:157-225 and pipeline.py:653-712).
//
// Persistent, pre-registered receive rings ("persistent buffers" that
// amortise cross-process handle creation): the receiver cudaMalloc's a ring of slots
// plus a 'ready' sequence word, exports CUDA IPC handles once; the sender maps them
// and, per message, on its side stream:
//     wait  local free-counter >= seq - slots + 1       (cuStreamWaitValue32, flow control)
//     copy  payload -> peer slot[seq % slots]            (cudaMemcpyAsync, copy engine over NVLink)
//     write peer ready-word = seq + 1                   (cuStreamWriteValue32, fenced)
// the receiver, on its stream:
//     wait  local ready-word >= seq + 1
//     copy  slot -> destination tensor (or consume in place)
//     write sender free-counter = seq + 1
// No host synchronisation anywhere; ordering is carried by stream-ordered flag writes.
#include <mutex>

#include "smpk_common.cuh"

namespace smpk {

typedef CUresult (*PFN_waitValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_writeValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

static PFN_waitValue32 g_wait = nullptr;
static PFN_writeValue32 g_write = nullptr;

static bool load_stream_mem_ops() {
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_wait = reinterpret_cast<PFN_waitValue32>(p);
    p = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_write = reinterpret_cast<PFN_writeValue32>(p);
  });
  return g_wait && g_write;
}

}  // namespace smpk

using namespace smpk;

extern "C" int smpk_p2p_alloc(int64_t bytes, void** ptr) {
  SMPK_REQUIRE(bytes > 0 && ptr, SMPK_ERR_BAD_ARG, "smpk_p2p_alloc: bad arguments");
  cudaError_t e = cudaMalloc(ptr, (size_t)bytes);
  SMPK_REQUIRE(e == cudaSuccess, SMPK_ERR_CUDA, "smpk_p2p_alloc: %s", cudaGetErrorString(e));
  e = cudaMemset(*ptr, 0, (size_t)bytes);
  SMPK_REQUIRE(e == cudaSuccess, SMPK_ERR_CUDA, "smpk_p2p_alloc(memset): %s", cudaGetErrorString(e));
  return SMPK_OK;
}

extern "C" int smpk_p2p_free(void* ptr) {
  cudaError_t e = cudaFree(ptr);
  SMPK_REQUIRE(e == cudaSuccess, SMPK_ERR_CUDA, "smpk_p2p_free: %s", cudaGetErrorString(e));
  return SMPK_OK;
}

// handle_out: 64 bytes (cudaIpcMemHandle_t)
extern "C" int smpk_p2p_export(void* ptr, void* handle_out) {
  SMPK_REQUIRE(ptr && handle_out, SMPK_ERR_BAD_ARG, "smpk_p2p_export: bad arguments");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, ptr);
  SMPK_REQUIRE(e == cudaSuccess, SMPK_ERR_CUDA, "smpk_p2p_export: %s", cudaGetErrorString(e));
  memcpy(handle_out, &h, sizeof(h));
  return SMPK_OK;
}

extern "C" int smpk_p2p_import(const void* handle, void** ptr) {
  SMPK_REQUIRE(handle && ptr, SMPK_ERR_BAD_ARG, "smpk_p2p_import: bad arguments");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
  SMPK_REQUIRE(e == cudaSuccess, SMPK_ERR_CUDA, "smpk_p2p_import: %s", cudaGetErrorString(e));
  return SMPK_OK;
}

extern "C" int smpk_p2p_close(void* ptr) {
  cudaError_t e = cudaIpcCloseMemHandle(ptr);
  SMPK_REQUIRE(e == cudaSuccess, SMPK_ERR_CUDA, "smpk_p2p_close: %s", cudaGetErrorString(e));
  return SMPK_OK;
}

// Sender side of one message.  peer_slot: mapped address of the receiver's slot;
// peer_ready: mapped address of the receiver's ready word; local_free: this rank's
// free-counter written by the receiver.  wait_free: value local_free must reach
// (seq - slots + 1, or 0 to skip).  Signals peer_ready = seq + 1.
extern "C" int smpk_p2p_send(void* peer_slot, const void* src, int64_t bytes, void* peer_ready,
                             const void* local_free, uint32_t wait_free, uint32_t seq, void* stream) {
  SMPK_REQUIRE(load_stream_mem_ops(), SMPK_ERR_CUDA, "smpk_p2p_send: stream memory ops unavailable");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (wait_free > 0) {
    CUresult r = g_wait((CUstream)st, (CUdeviceptr)local_free, wait_free, CU_STREAM_WAIT_VALUE_GEQ);
    SMPK_REQUIRE(r == CUDA_SUCCESS, SMPK_ERR_CUDA, "smpk_p2p_send: wait free failed (%d)", (int)r);
  }
  cudaError_t e = cudaMemcpyAsync(peer_slot, src, (size_t)bytes, cudaMemcpyDeviceToDevice, st);
  SMPK_REQUIRE(e == cudaSuccess, SMPK_ERR_CUDA, "smpk_p2p_send: copy: %s", cudaGetErrorString(e));
  CUresult r = g_write((CUstream)st, (CUdeviceptr)peer_ready, seq + 1, CU_STREAM_WRITE_VALUE_DEFAULT);
  SMPK_REQUIRE(r == CUDA_SUCCESS, SMPK_ERR_CUDA, "smpk_p2p_send: signal failed (%d)", (int)r);
  return SMPK_OK;
}

// Plain stream-ordered device copy (copy engine), also to a peer-mapped address: the TP
// exchanges issued on side streams so the SMs keep computing while the bytes move.
extern "C" int smpk_copy_async(void* dst, const void* src, int64_t bytes, void* stream) {
  SMPK_REQUIRE(dst && src && bytes >= 0, SMPK_ERR_BAD_ARG, "smpk_copy_async: bad arguments");
  cudaError_t e = cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToDevice,
                                  reinterpret_cast<cudaStream_t>(stream));
  SMPK_REQUIRE(e == cudaSuccess, SMPK_ERR_CUDA, "smpk_copy_async: %s", cudaGetErrorString(e));
  return SMPK_OK;
}

// Receiver side: wait local_ready >= seq + 1, copy slot -> dst (if dst), then free the
// slot by writing peer_free = seq + 1 (mapped address of the sender's free-counter).
extern "C" int smpk_p2p_recv(void* dst, const void* local_slot, int64_t bytes, const void* local_ready,
                             void* peer_free, uint32_t seq, void* stream) {
  SMPK_REQUIRE(load_stream_mem_ops(), SMPK_ERR_CUDA, "smpk_p2p_recv: stream memory ops unavailable");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  CUresult r = g_wait((CUstream)st, (CUdeviceptr)local_ready, seq + 1, CU_STREAM_WAIT_VALUE_GEQ);
  SMPK_REQUIRE(r == CUDA_SUCCESS, SMPK_ERR_CUDA, "smpk_p2p_recv: wait ready failed (%d)", (int)r);
  if (dst) {
    cudaError_t e = cudaMemcpyAsync(dst, local_slot, (size_t)bytes, cudaMemcpyDeviceToDevice, st);
    SMPK_REQUIRE(e == cudaSuccess, SMPK_ERR_CUDA, "smpk_p2p_recv: copy: %s", cudaGetErrorString(e));
  }
  r = g_write((CUstream)st, (CUdeviceptr)peer_free, seq + 1, CU_STREAM_WRITE_VALUE_DEFAULT);
  SMPK_REQUIRE(r == CUDA_SUCCESS, SMPK_ERR_CUDA, "smpk_p2p_recv: free signal failed (%d)", (int)r);
  return SMPK_OK;
}

// Stream-ordered flag words for the chunked TP exchanges (tp_exchange="chunks", exchange.py):
// a 32-bit word in (possibly peer-mapped) device memory is awaited / written by the stream's
// front end (cuStreamWaitValue32 / cuStreamWriteValue32) -- no SM, capturable in CUDA graphs.
// op 0: wait *word == value (then the caller resets it); op 1: write *word = value, fenced after
// the stream's prior work (a copy into a peer slot is visible before its ready word).
extern "C" int smpk_stream_flag(void* word, uint32_t value, int op, void* stream) {
  SMPK_REQUIRE(word && (op == 0 || op == 1), SMPK_ERR_BAD_ARG, "smpk_stream_flag: bad arguments");
  SMPK_REQUIRE(load_stream_mem_ops(), SMPK_ERR_CUDA, "smpk_stream_flag: stream memory ops unavailable");
  CUstream st = (CUstream) reinterpret_cast<cudaStream_t>(stream);
  CUresult r = op == 0 ? g_wait(st, (CUdeviceptr)word, value, CU_STREAM_WAIT_VALUE_EQ)
                       : g_write(st, (CUdeviceptr)word, value, CU_STREAM_WRITE_VALUE_DEFAULT);
  SMPK_REQUIRE(r == CUDA_SUCCESS, SMPK_ERR_CUDA, "smpk_stream_flag(op %d): driver error %d", op, (int)r);
  return SMPK_OK;
}
