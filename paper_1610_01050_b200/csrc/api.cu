// C ABI entry points that touch the device: bind, execute, detect, compact, run_host.
// See include/rsft.h for the contract of every call.
#include <cuda_runtime.h>

#include <string>

#include "rsft_internal.h"
#include <nvtx3/nvToolsExt.h>

namespace {
// NVTX range per ABI call (SURVEY §5 tracing): visible in nsys / ncu timelines, no cost without a tool
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

namespace rsft {
rsft_status launch_execute(rsft_plan_s* p, const void* d_x, int64_t batch, int l0, int nl, uint32_t* bm,
                           void* spectra, cudaStream_t st);
rsft_status launch_segments(rsft_plan_s* p, const void* d_x, int64_t batch, uint32_t* bm, void* spectra,
                            cudaStream_t st);
rsft_status launch_partial(rsft_plan_s* p, const void* d_x, int64_t off, int64_t len, void* d_partial,
                           cudaStream_t st);
rsft_status launch_finalize(rsft_plan_s* p, const void* d_folded, int l0, int nl, uint32_t* bm, void* spectra,
                            cudaStream_t st);
rsft_status launch_run(rsft_plan_s* p, const void* d_x, int64_t batch, uint32_t* bm, uint32_t* det, int64_t* idx,
                       int64_t capacity, int64_t* d_count, cudaStream_t st);
rsft_status launch_detect(rsft_plan_s* p, const uint32_t* bm, int64_t batch, int64_t d0b, int64_t d0e,
                          uint32_t* det, uint8_t* counts, cudaStream_t st);
rsft_status launch_compact(rsft_plan_s* p, const uint32_t* det, int64_t batch, int64_t* idx,
                           int64_t capacity, int64_t* d_count, cudaStream_t st);
rsft_status upload_twiddles(cudaStream_t st);
rsft_status upload_bartlett_twiddles(cudaStream_t st);   // bartlett.cu
rsft_status launch_detect_compact(rsft_plan_s* p, const uint32_t* bm, int64_t batch, uint32_t* det,
                                  int64_t* idx, int64_t capacity, int64_t* d_count, cudaStream_t st);

static rsft_status cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return RSFT_OK;
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return RSFT_E_CUDA;
}
static int ilog2i(int64_t v) { int r = 0; while ((int64_t(1) << r) < v) ++r; return r; }
static size_t align256(size_t v) { return (v + 255) & ~size_t(255); }
}  // namespace rsft

using namespace rsft;

extern "C" {

rsft_status rsft_bind(rsft_plan_t p, void* d_ws, size_t bytes, void* stream) {
  NvtxRange nvtx_("rsft_bind");
  if (!p) return RSFT_E_ARG;
  if (!d_ws || bytes < p->ws.total || (reinterpret_cast<uintptr_t>(d_ws) & 255)) return RSFT_E_WORKSPACE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  rsft_status s;
  int dev = 0;
  if ((s = cuda_check(cudaGetDevice(&dev), "cudaGetDevice"))) return s;
  if (p->want_device >= 0 && dev != p->want_device) {
    set_error("rsft_bind: the plan was created for another device (rsft_plan)");
    return RSFT_E_STATE;
  }
  int sms = 0;
  if ((s = cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "sm count"))) return s;
  p->device = dev;
  p->num_sms = sms;
  char* base = reinterpret_cast<char*>(d_ws);
  static thread_local std::vector<LoopDev> loops;
  loops.assign(p->L, LoopDev{});
  for (int l = 0; l < p->L; ++l) {
    for (int d = 0; d < 3; ++d) {
      loops[l].sig[d] = d < p->D ? (int32_t)p->sigma[l * p->D + d] : 1;
      loops[l].sinv[d] = d < p->D ? (int32_t)p->sinv[l * p->D + d] : 1;
      loops[l].tau[d] = d < p->D ? (int32_t)p->tau[l * p->D + d] : 0;
    }
    loops[l].gamma = (float)p->gamma[l];
  }
  if ((s = cuda_check(cudaMemcpyAsync(base + p->ws.loops_off, loops.data(), sizeof(LoopDev) * p->L,
                                      cudaMemcpyHostToDevice, st), "upload loops"))) return s;
  for (int d = 0; d < p->D; ++d)
    if ((s = cuda_check(cudaMemcpyAsync(base + p->ws.h_off[d], p->hf[d].data(), sizeof(float) * p->hf[d].size(),
                                        cudaMemcpyHostToDevice, st), "upload weights"))) return s;
  static thread_local std::vector<float> ht;
  for (int d = 0; d + 1 < p->D; ++d) {            // ht[r][a][l] = h[l][r + B a] (class-major)
    const int64_t n = p->n[d], b = p->b[d], a = n / b, L = p->L;
    ht.assign((size_t)L * n, 0.f);
    for (int64_t l = 0; l < L; ++l)
      for (int64_t sidx = 0; sidx < n; ++sidx) ht[((sidx % b) * a + sidx / b) * L + l] = p->hf[d][l * n + sidx];
    if ((s = cuda_check(cudaMemcpyAsync(base + p->ws.ht_off[d], ht.data(), sizeof(float) * ht.size(),
                                        cudaMemcpyHostToDevice, st), "upload class-major weights"))) return s;
  }
  {                                                // Bartlett baseline: fp32 windows, twiddles
    static thread_local std::vector<float> bw;
    for (int d = 0; d < p->D; ++d) {
      bw.assign(p->prewin[d].begin(), p->prewin[d].end());
      if ((s = cuda_check(cudaMemcpyAsync(base + p->ws.bwin_off[d], bw.data(), 4 * bw.size(), cudaMemcpyHostToDevice, st),
                          "upload bartlett windows"))) return s;
    }
    static thread_local std::vector<float> tw;
    tw.assign(4096 + 1, 0.f);
    tw[4096] = 1.0f;
    for (int k = 0; k < 2048; ++k) {
      tw[2 * k] = (float)std::cos(-2.0 * M_PI * k / 4096.0);
      tw[2 * k + 1] = (float)std::sin(-2.0 * M_PI * k / 4096.0);
    }
    if ((s = cuda_check(cudaMemcpyAsync(base + p->ws.btw_off, tw.data(), 8 * 2048, cudaMemcpyHostToDevice, st),
                        "upload bartlett twiddles"))) return s;
    if ((s = cuda_check(cudaMemcpyAsync(base + p->ws.bone_off, &tw[4096], 4, cudaMemcpyHostToDevice, st),
                        "upload one"))) return s;
  }
  if (!p->ntab.empty() && p->ws.ntab_bytes == p->ntab.size() * 4)
    if ((s = cuda_check(cudaMemcpyAsync(base + p->ws.ntab_off, p->ntab.data(), p->ws.ntab_bytes,
                                        cudaMemcpyHostToDevice, st), "ntab upload")))
      return s;
  if (!p->xmask.empty() && p->ws.xmask_bytes == p->xmask.size() * 4)
    if ((s = cuda_check(cudaMemcpyAsync(base + p->ws.xmask_off, p->xmask.data(), p->ws.xmask_bytes,
                                        cudaMemcpyHostToDevice, st), "upload vote masks"))) return s;
  if ((s = upload_twiddles(st))) return s;
  if ((s = upload_bartlett_twiddles(st))) return s;
  if ((s = cuda_check(cudaStreamSynchronize(st), "bind sync"))) return s;   // tables are host temporaries

  PlanDev& pd = p->dev;
  pd = PlanDev{};
  pd.D = p->D;
  pd.L = p->L;
  pd.mu = p->mu;
  pd.nplanes = 6;
  for (int d = 0; d < 3; ++d) {
    int64_t n = d < p->D ? p->n[d] : 1, b = d < p->D ? p->b[d] : 1;
    pd.n[d] = (int32_t)n; pd.b[d] = (int32_t)b; pd.a[d] = (int32_t)(n / b);
    pd.lgn[d] = ilog2i(n); pd.lgb[d] = ilog2i(b); pd.lga[d] = ilog2i(n / b);
    pd.shift[d] = (d < p->D && b < n) ? 1 : 0;
    pd.h[d] = d < p->D ? reinterpret_cast<const float*>(base + p->ws.h_off[d]) : nullptr;
    pd.ht[d] = d + 1 < p->D ? reinterpret_cast<const float*>(base + p->ws.ht_off[d]) : nullptr;
  }
  pd.ntot = p->ntot;
  pd.btot = p->btot;
  pd.wpl = (int32_t)((p->btot + 31) / 32);
  pd.nlast = (int32_t)p->n[p->D - 1];
  pd.blast = (int32_t)p->b[p->D - 1];
  pd.rows = p->ntot / p->n[p->D - 1];
  pd.bouter = (int32_t)(p->btot / p->b[p->D - 1]);
  int64_t aouter = 1;
  for (int d = 0; d + 1 < p->D; ++d) aouter *= p->a[d];
  pd.aouter = (int32_t)aouter;
  pd.loops = reinterpret_cast<const LoopDev*>(base + p->ws.loops_off);
  pd.fbuf = reinterpret_cast<float2*>(base + p->ws.fbuf_off);
  pd.fbuf_capacity = (int64_t)(p->ws.fbuf_bytes / 8);
  pd.chunk_counts = reinterpret_cast<long long*>(base + p->ws.chunk_off);
  pd.chunk_capacity = p->ws.chunk_capacity;
  pd.xmask = p->ws.xmask_bytes ? reinterpret_cast<const uint32_t*>(base + p->ws.xmask_off) : nullptr;
  pd.ntab = (p->ws.ntab_bytes && p->ntab.size() * 4 == p->ws.ntab_bytes)
                ? reinterpret_cast<const uint32_t*>(base + p->ws.ntab_off) : nullptr;
  pd.region_state = reinterpret_cast<unsigned long long*>(base + p->ws.region_off);
  pd.region_capacity = p->ws.region_capacity;
  pd.region_slots = p->ws.slots_bytes ? reinterpret_cast<uint32_t*>(base + p->ws.slots_off) : nullptr;
  pd.list_cap = (int32_t)p->ws.list_cap;
  pd.etab = p->ws.etab_bytes ? reinterpret_cast<uint32_t*>(base + p->ws.etab_off) : nullptr;
  pd.etab_frames = p->ws.etab_bytes
                       ? (int64_t)(p->ws.etab_bytes / ((size_t)p->L * p->b[0] * p->b[1] * (p->n[2] / 32) * 4)) : 0;
  for (int d = 0; d < 3; ++d) pd.bwin[d] = d < p->D ? reinterpret_cast<const float*>(base + p->ws.bwin_off[d]) : nullptr;
  pd.bone = reinterpret_cast<const float*>(base + p->ws.bone_off);
  pd.btw = reinterpret_cast<const float2*>(base + p->ws.btw_off);
  p->d_ws = d_ws;
  p->bound = true;
  return RSFT_OK;
}

rsft_status rsft_execute(rsft_plan_t p, const void* d_x, int64_t batch, int32_t loop_begin, int32_t loop_end,
                         uint32_t* d_bitmaps, void* d_spectra, void* stream) {
  NvtxRange nvtx_("rsft_execute");
  if (!p || !d_x || !d_bitmaps) return RSFT_E_ARG;
  if (!p->bound) return RSFT_E_STATE;
  if (batch < 0 || batch > p->P.max_batch) return RSFT_E_ARG;
  if (loop_begin < 0 || loop_end > p->L || loop_begin >= loop_end) return RSFT_E_ARG;
  if (reinterpret_cast<uintptr_t>(d_x) & 15) return RSFT_E_ARG;
  p->last_launches = 0;
  if (batch == 0) return RSFT_OK;
  return launch_execute(p, d_x, batch, loop_begin, loop_end - loop_begin, d_bitmaps, d_spectra,
                        reinterpret_cast<cudaStream_t>(stream));
}

rsft_status rsft_execute_segments(rsft_plan_t p, const void* d_x, int64_t batch, uint32_t* d_bitmaps,
                                  void* d_spectra, void* stream) {
  NvtxRange nvtx_("rsft_execute_segments");
  if (!p || !d_x || !d_bitmaps) return RSFT_E_ARG;
  if (!p->bound) return RSFT_E_STATE;
  if (batch < 0 || batch > p->P.max_batch) return RSFT_E_ARG;
  if (reinterpret_cast<uintptr_t>(d_x) & 15) return RSFT_E_ARG;
  p->last_launches = 0;
  if (batch == 0) return RSFT_OK;
  return launch_segments(p, d_x, batch, d_bitmaps, d_spectra, reinterpret_cast<cudaStream_t>(stream));
}

rsft_status rsft_bucketize_partial(rsft_plan_t p, const void* d_x_slab, int64_t off, int64_t len, void* d_partial,
                                   void* stream) {
  NvtxRange nvtx_("rsft_bucketize_partial");
  if (!p || !d_x_slab || !d_partial) return RSFT_E_ARG;
  if (!p->bound) return RSFT_E_STATE;
  if (p->D < 2 || resolve_mode(p, 1) != RSFT_MODE_SPLIT) return RSFT_E_UNSUPPORTED;
  if (off < 0 || len <= 0 || off + len > p->n[0] || off % p->b[0] || len % p->b[0]) return RSFT_E_ARG;
  if ((reinterpret_cast<uintptr_t>(d_x_slab) & 15) || (reinterpret_cast<uintptr_t>(d_partial) & 7)) return RSFT_E_ARG;
  p->last_launches = 0;
  return launch_partial(p, d_x_slab, off, len, d_partial, reinterpret_cast<cudaStream_t>(stream));
}

rsft_status rsft_finalize(rsft_plan_t p, const void* d_folded, int32_t loop_begin, int32_t loop_end,
                          uint32_t* d_bitmaps, void* d_spectra, void* stream) {
  NvtxRange nvtx_("rsft_finalize");
  if (!p || !d_folded || !d_bitmaps) return RSFT_E_ARG;
  if (!p->bound) return RSFT_E_STATE;
  if (p->D < 2 || resolve_mode(p, 1) != RSFT_MODE_SPLIT) return RSFT_E_UNSUPPORTED;
  if (loop_begin < 0 || loop_end > p->L || loop_begin >= loop_end) return RSFT_E_ARG;
  p->last_launches = 0;
  return launch_finalize(p, d_folded, loop_begin, loop_end - loop_begin, d_bitmaps, d_spectra,
                         reinterpret_cast<cudaStream_t>(stream));
}

rsft_status rsft_detect(rsft_plan_t p, const uint32_t* d_bitmaps, int64_t batch, int64_t d0b, int64_t d0e,
                        uint32_t* d_detect, uint8_t* d_counts, void* stream) {
  NvtxRange nvtx_("rsft_detect");
  if (!p || !d_bitmaps || !d_detect) return RSFT_E_ARG;
  if (!p->bound) return RSFT_E_STATE;
  if (batch < 0 || batch > p->P.max_batch) return RSFT_E_ARG;
  if (d0b < 0 || d0e > p->n[0] || d0b >= d0e) return RSFT_E_ARG;
  if (p->D == 1 && (d0b != 0 || d0e != p->n[0])) return RSFT_E_ARG;
  if (((d0e - d0b) * (p->ntot / p->n[0])) % 32) return RSFT_E_ARG;
  p->last_launches = 0;
  if (batch == 0) return RSFT_OK;
  return launch_detect(p, d_bitmaps, batch, d0b, d0e, d_detect, d_counts, reinterpret_cast<cudaStream_t>(stream));
}

rsft_status rsft_compact(rsft_plan_t p, const uint32_t* d_detect, int64_t batch, int64_t* d_idx,
                         int64_t capacity, int64_t* d_count, void* stream) {
  NvtxRange nvtx_("rsft_compact");
  if (!p || !d_detect || !d_count || (capacity > 0 && !d_idx) || capacity < 0) return RSFT_E_ARG;
  if (!p->bound) return RSFT_E_STATE;
  if (batch < 1 || batch > p->P.max_batch) return RSFT_E_ARG;
  p->last_launches = 0;
  return launch_compact(p, d_detect, batch, d_idx, capacity, d_count, reinterpret_cast<cudaStream_t>(stream));
}

rsft_status rsft_detect_compact(rsft_plan_t p, const uint32_t* d_bitmaps, int64_t batch, uint32_t* d_detect,
                                int64_t* d_idx, int64_t capacity, int64_t* d_count, void* stream) {
  NvtxRange nvtx_("rsft_detect_compact");
  if (!p || !d_bitmaps || !d_detect || !d_count || (capacity > 0 && !d_idx) || capacity < 0) return RSFT_E_ARG;
  if (!p->bound) return RSFT_E_STATE;
  if (batch < 1 || batch > p->P.max_batch) return RSFT_E_ARG;
  p->last_launches = 0;
  return launch_detect_compact(p, d_bitmaps, batch, d_detect, d_idx, capacity, d_count,
                               reinterpret_cast<cudaStream_t>(stream));
}

rsft_status rsft_run(rsft_plan_t p, const void* d_x, int64_t batch, uint32_t* d_bitmaps, uint32_t* d_detect,
                     int64_t* d_idx, int64_t capacity, int64_t* d_count, void* stream) {
  NvtxRange nvtx_("rsft_run");
  if (!p || !d_x || !d_bitmaps || !d_detect || !d_count || (capacity > 0 && !d_idx) || capacity < 0) return RSFT_E_ARG;
  if (!p->bound) return RSFT_E_STATE;
  if (batch < 1 || batch > p->P.max_batch) return RSFT_E_ARG;
  if (reinterpret_cast<uintptr_t>(d_x) & 15) return RSFT_E_ARG;
  p->last_launches = 0;
  return launch_run(p, d_x, batch, d_bitmaps, d_detect, d_idx, capacity, d_count, reinterpret_cast<cudaStream_t>(stream));
}

size_t rsft_host_scratch_bytes(rsft_plan_t p, int64_t batch, int64_t capacity) {
  if (!p || batch < 1) return 0;
  size_t x = align256((size_t)batch * p->ntot * 8);
  size_t bm = align256((size_t)batch * p->L * ((p->btot + 31) / 32) * 4);
  size_t det = align256((size_t)batch * ((p->ntot + 31) / 32) * 4);
  size_t idx = align256((size_t)(capacity > 0 ? capacity : 1) * 8);
  return x + bm + det + idx + 256;
}

rsft_status rsft_run_host(rsft_plan_t p, const void* h_x, int64_t batch, int64_t* h_idx, int64_t capacity,
                          int64_t* h_count, void* d_scratch, size_t scratch_bytes, void* stream) {
  NvtxRange nvtx_("rsft_run_host");
  if (!p || !h_x || !h_count || (capacity > 0 && !h_idx) || capacity < 0) return RSFT_E_ARG;
  if (!p->bound) return RSFT_E_STATE;
  if (batch < 1 || batch > p->P.max_batch) return RSFT_E_ARG;
  if (!d_scratch || scratch_bytes < rsft_host_scratch_bytes(p, batch, capacity) ||
      (reinterpret_cast<uintptr_t>(d_scratch) & 255)) return RSFT_E_WORKSPACE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  char* base = reinterpret_cast<char*>(d_scratch);
  size_t off = 0;
  void* dx = base + off; off += align256((size_t)batch * p->ntot * 8);
  uint32_t* dbm = reinterpret_cast<uint32_t*>(base + off); off += align256((size_t)batch * p->L * ((p->btot + 31) / 32) * 4);
  uint32_t* ddet = reinterpret_cast<uint32_t*>(base + off); off += align256((size_t)batch * ((p->ntot + 31) / 32) * 4);
  int64_t* didx = reinterpret_cast<int64_t*>(base + off); off += align256((size_t)(capacity > 0 ? capacity : 1) * 8);
  int64_t* dcount = reinterpret_cast<int64_t*>(base + off);
  rsft_status s;
  int32_t launches = 0;
  if ((s = cuda_check(cudaMemcpyAsync(dx, h_x, (size_t)batch * p->ntot * 8, cudaMemcpyHostToDevice, st), "H2D x"))) return s;
  if ((s = rsft_run(p, dx, batch, dbm, ddet, didx, capacity, dcount, stream))) return s;
  launches += p->last_launches;
  if ((s = cuda_check(cudaMemcpyAsync(h_count, dcount, 8, cudaMemcpyDeviceToHost, st), "D2H count"))) return s;
  if ((s = cuda_check(cudaStreamSynchronize(st), "sync"))) return s;
  int64_t n = *h_count < capacity ? *h_count : capacity;
  if (n > 0) {
    if ((s = cuda_check(cudaMemcpyAsync(h_idx, didx, (size_t)n * 8, cudaMemcpyDeviceToHost, st), "D2H idx"))) return s;
    if ((s = cuda_check(cudaStreamSynchronize(st), "sync"))) return s;
  }
  p->last_launches = launches;
  return RSFT_OK;
}

}  // extern "C"
