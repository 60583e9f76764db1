// Host-buffer pipelined apply (C-ABI cim_sym_spmm_host_batch).
//
// A user of the reference hands numpy arrays in and gets numpy arrays back
// (contract_observables, pipeline.py:534-570, writes `inputs.accum` on the
// host).  For a host-resident block of vectors the apply is bound by PCIe
// (X in + Y out = 2·n·k·s bytes per block) rather than by the ~1.6 ms kernel,
// so a batch of independent blocks is pipelined over three streams:
//
//   h2d  : X_b  host → X[b%2]                (waits until apply b-2 read X[b%2])
//   comp : Y[b%2] = A·X[b%2]                 (waits for X_b and for Y_{b-2} to leave)
//   d2h  : Y[b%2] → Y_b host
//
// so steady state costs max(H2D, kernel, D2H) per block instead of their sum
// (PCIe is full duplex).  Device workspace (caller-owned) = 2 X + 2 Y buffers
// of n_pad × k.
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "cim_b200.h"
#include "host_util.h"

namespace {

struct PipeState {
  bool init = false;
  cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
  cudaEvent_t x_ready[2], comp_done[2], y_free[2];
  cudaEvent_t entry = nullptr;  // the caller's prior work (legacy default stream)
};
std::mutex g_pipe_mu;
std::vector<PipeState> g_pipe;

int pipe_state(PipeState **out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return cim::set_error(CIM_ECUDA, "cudaGetDevice failed");
  std::lock_guard<std::mutex> lk(g_pipe_mu);
  if ((int)g_pipe.size() <= dev) g_pipe.resize(dev + 1);
  PipeState &p = g_pipe[dev];
  if (!p.init) {
    cudaError_t e = cudaSuccess;
    for (cudaStream_t *s : {&p.h2d, &p.comp, &p.d2h})
      if (e == cudaSuccess) e = cudaStreamCreateWithFlags(s, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p.entry, cudaEventDisableTiming);
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
      e = cudaEventCreateWithFlags(&p.x_ready[i], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p.comp_done[i], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p.y_free[i], cudaEventDisableTiming);
    }
    if (e != cudaSuccess) return cim::set_error(CIM_ECUDA, std::string("pipeline streams: ") + cudaGetErrorString(e));
    p.init = true;
  }
  *out = &p;
  return CIM_OK;
}

size_t elem_size(int32_t dtype) { return dtype == CIM_F64 ? 8 : 4; }

}  // namespace

extern "C" uint64_t cim_host_batch_workspace_bytes(const cim_half_tiles *H, int32_t k) {
  if (!H || k < 1 || H->n < 1) return 0;
  const int64_t n_pad = (H->n + CIM_BLOCK - 1) / CIM_BLOCK * CIM_BLOCK;
  return 4ull * (uint64_t)n_pad * (uint64_t)k * elem_size(H->dtype);
}

extern "C" int cim_sym_spmm_host_batch(const cim_half_tiles *H, const void *const *X_host, void *const *Y_host,
                                       int32_t n_batch, int32_t k, void *workspace, uint64_t ws_bytes) {
  cim::clear_error();
  if (!H) return cim::set_error(CIM_EINVAL, "H is NULL");
  if (n_batch < 0) return cim::set_error(CIM_EINVAL, "n_batch must be >= 0");
  if (n_batch > 0 && (!X_host || !Y_host)) return cim::set_error(CIM_EINVAL, "X_host / Y_host arrays are NULL");
  for (int32_t b = 0; b < n_batch; ++b)
    if (!X_host[b] || !Y_host[b]) return cim::set_error(CIM_EINVAL, "NULL host buffer at batch index " + std::to_string(b));
  if (k < 1) return cim::set_error(CIM_EINVAL, "k must be >= 1");
  if (!cim_layout_supports(H->layout, H->dtype, k)) return cim::set_error(CIM_EUNSUPPORTED, "unsupported (layout, dtype, k)");
  const uint64_t need = cim_host_batch_workspace_bytes(H, k);
  if (!workspace || ws_bytes < need)
    return cim::set_error(CIM_EINVAL, "workspace must hold " + std::to_string(need) + " bytes");
  if (reinterpret_cast<uintptr_t>(workspace) & 15) return cim::set_error(CIM_EINVAL, "workspace must be 16-byte aligned");
  if (n_batch == 0) return CIM_OK;

  PipeState *ps = nullptr;
  int rc = pipe_state(&ps);
  if (rc) return rc;
  const size_t es = elem_size(H->dtype);
  const int64_t n_pad = (H->n + CIM_BLOCK - 1) / CIM_BLOCK * CIM_BLOCK;
  const size_t buf = (size_t)n_pad * k * es, live = (size_t)H->n * k * es;
  unsigned char *ws = static_cast<unsigned char *>(workspace);
  unsigned char *Xd[2] = {ws, ws + buf}, *Yd[2] = {ws + 2 * buf, ws + 3 * buf};

  auto cuda_fail = [](cudaError_t e, const char *what) {
    return cim::set_error(CIM_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  };
  cudaError_t e = cudaSuccess;
  // The library's streams are non-blocking: order them after everything the
  // caller queued on the legacy default stream (e.g. the tile-value fill of a
  // freshly built matrix) — the pipeline must not read H before it is written.
  if ((e = cudaEventRecord(ps->entry, cudaStreamLegacy)) != cudaSuccess) return cuda_fail(e, "record entry");
  for (cudaStream_t st : {ps->h2d, ps->comp})
    if ((e = cudaStreamWaitEvent(st, ps->entry, 0)) != cudaSuccess) return cuda_fail(e, "wait entry");
  // pad rows of the X buffers meet zero matrix entries but must be finite
  if (buf > live) {
    for (int s = 0; s < 2 && e == cudaSuccess; ++s) e = cudaMemsetAsync(Xd[s] + live, 0, buf - live, ps->h2d);
    if (e != cudaSuccess) return cuda_fail(e, "memset X pad rows");
  }
  for (int32_t b = 0; b < n_batch; ++b) {
    const int s = b & 1;
    if ((e = cudaStreamWaitEvent(ps->h2d, ps->comp_done[s], 0)) != cudaSuccess) return cuda_fail(e, "wait");
    if ((e = cudaMemcpyAsync(Xd[s], X_host[b], live, cudaMemcpyHostToDevice, ps->h2d)) != cudaSuccess)
      return cuda_fail(e, "H2D X");
    if ((e = cudaEventRecord(ps->x_ready[s], ps->h2d)) != cudaSuccess) return cuda_fail(e, "record");
    if ((e = cudaStreamWaitEvent(ps->comp, ps->x_ready[s], 0)) != cudaSuccess) return cuda_fail(e, "wait");
    if ((e = cudaStreamWaitEvent(ps->comp, ps->y_free[s], 0)) != cudaSuccess) return cuda_fail(e, "wait");
    rc = cim_sym_spmm(H, Xd[s], Yd[s], k, k, k, 0u, ps->comp);
    if (rc) return rc;
    if ((e = cudaEventRecord(ps->comp_done[s], ps->comp)) != cudaSuccess) return cuda_fail(e, "record");
    if ((e = cudaStreamWaitEvent(ps->d2h, ps->comp_done[s], 0)) != cudaSuccess) return cuda_fail(e, "wait");
    if ((e = cudaMemcpyAsync(Y_host[b], Yd[s], live, cudaMemcpyDeviceToHost, ps->d2h)) != cudaSuccess)
      return cuda_fail(e, "D2H Y");
    if ((e = cudaEventRecord(ps->y_free[s], ps->d2h)) != cudaSuccess) return cuda_fail(e, "record");
  }
  if ((e = cudaStreamSynchronize(ps->d2h)) != cudaSuccess) return cuda_fail(e, "synchronize");
  return CIM_OK;
}
