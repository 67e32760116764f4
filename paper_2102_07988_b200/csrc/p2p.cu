// p2p.cu — device-initiated stage-to-stage messages over NVLink (the paper's
// "send activations forward, gradients backward").
//
// The receiving buffers of every stage (its input activations hs[0] and its output gradient
// grad_out) are NCCL symmetric-memory windows (ncclMemAlloc + ncclCommWindowRegister), so every
// rank can address its neighbours' buffers directly (ncclGetPeerPointer: a load/store mapping over
// NVLink). The producing kernels write their outputs straight into the neighbour's buffer — the
// last layer's FC2 residual epilogue (forward) and the first layer's LayerNorm backward (gradient)
// — and a one-thread kernel then publishes "job j of step e is complete" by a system-scope release
// store of e into the neighbour's flag slot j; the consumer's stream waits on its own flag slot with
// an acquire spin before the job's first kernel. No NCCL kernels, copies or host round trips are on
// the data path. Epochs (one per step, a device counter advanced inside the captured step) make the
// flags monotonic, so they are never reset and CUDA-graph replays stay valid.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>

#include "kernels.h"

namespace tp {

namespace {

__global__ void peer_ptr_kernel(ncclWindow_t w, int peer, void** out) { *out = ncclGetPeerPointer(w, 0, peer); }

__global__ void epoch_inc_kernel(unsigned long long* epoch) { *epoch += 1; }

__global__ void p2p_signal_kernel(unsigned long long* remote_slot, const unsigned long long* epoch) {
  const unsigned long long e = *epoch;
  __threadfence_system();  // the producer kernel's peer stores (earlier in this stream) before the flag
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(remote_slot), "l"(e) : "memory");
}

__global__ void p2p_wait_kernel(const unsigned long long* local_slot, const unsigned long long* epoch) {
  const unsigned long long e = *epoch;
  unsigned long long v;
  for (;;) {
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(local_slot) : "memory");
    if (v >= e) break;
    __nanosleep(64);
  }
}

}  // namespace

cudaError_t p2p_peer_pointer(void* window, int peer, void** host_out, cudaStream_t st) {
  void** d = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&d), sizeof(void*), st);
  if (e != cudaSuccess) return e;
  peer_ptr_kernel<<<1, 1, 0, st>>>(reinterpret_cast<ncclWindow_t>(window), peer, d);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(host_out, d, sizeof(void*), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFreeAsync(d, st);
  return e;
}
cudaError_t p2p_epoch_inc(unsigned long long* epoch, cudaStream_t st) {
  epoch_inc_kernel<<<1, 1, 0, st>>>(epoch);
  return cudaGetLastError();
}
cudaError_t p2p_signal(unsigned long long* remote_slot, const unsigned long long* epoch, cudaStream_t st) {
  p2p_signal_kernel<<<1, 1, 0, st>>>(remote_slot, epoch);
  return cudaGetLastError();
}
cudaError_t p2p_wait(const unsigned long long* local_slot, const unsigned long long* epoch, cudaStream_t st) {
  p2p_wait_kernel<<<1, 1, 0, st>>>(local_slot, epoch);
  return cudaGetLastError();
}

}  // namespace tp
