// lg_api.cu -- error state, device info, workspaces, host<->device helpers.
#include <cstring>
#include <mutex>

#include "lg_common.cuh"

namespace lg {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

const DevInfo& dev_info() {
  static DevInfo info;
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    cudaDeviceGetAttribute(&info.sm_count, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&info.l2_bytes, cudaDevAttrL2CacheSize, dev);
    cudaDeviceGetAttribute(&info.major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&info.minor, cudaDevAttrComputeCapabilityMinor, dev);
    if (info.sm_count <= 0) info.sm_count = 148;
  });
  return info;
}

}  // namespace lg

extern "C" {

const char* lg_last_error(void) { return lg::g_last_error.c_str(); }

int lg_version(void) { return 100; }

int lg_device_info(int* sm_count, int* l2_bytes, int* cc_major, int* cc_minor) {
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return lg::fail(LG_ECUDA, std::string("no CUDA device: ") +
                                  cudaGetErrorString(e));
  const lg::DevInfo& d = lg::dev_info();
  if (sm_count) *sm_count = d.sm_count;
  if (l2_bytes) *l2_bytes = d.l2_bytes;
  if (cc_major) *cc_major = d.major;
  if (cc_minor) *cc_minor = d.minor;
  return LG_OK;
}

int lg_readback(const void* dev, void* host_pinned, int64_t bytes, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  LG_CUDA(cudaMemcpyAsync(host_pinned, dev, (size_t)bytes,
                          cudaMemcpyDeviceToHost, s));
  LG_CUDA(cudaStreamSynchronize(s));
  return LG_OK;
}

int lg_upload(void* dev, const void* host, int64_t bytes, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  LG_CUDA(cudaMemcpyAsync(dev, host, (size_t)bytes, cudaMemcpyHostToDevice, s));
  return LG_OK;
}

// ---- CUDA graphs: capture a fixed launch sequence once, replay it --------
int lg_capture_begin(void* stream) {
  if (!stream) return lg::fail(LG_EINVAL, "lg_capture_begin: needs a non-legacy stream");
  LG_CUDA(cudaStreamBeginCapture((cudaStream_t)stream, cudaStreamCaptureModeThreadLocal));
  return LG_OK;
}

int lg_capture_end(void* stream, void** exec_out) {
  if (!exec_out) return lg::fail(LG_EINVAL, "lg_capture_end: exec_out is NULL");
  cudaGraph_t g = nullptr;
  LG_CUDA(cudaStreamEndCapture((cudaStream_t)stream, &g));
  cudaGraphExec_t e = nullptr;
  cudaError_t err = cudaGraphInstantiate(&e, g, 0);
  cudaGraphDestroy(g);
  if (err != cudaSuccess)
    return lg::fail(LG_ECUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(err));
  *exec_out = (void*)e;
  return LG_OK;
}

int lg_graph_launch(void* exec, void* stream) {
  LG_CUDA(cudaGraphLaunch((cudaGraphExec_t)exec, (cudaStream_t)stream));
  return LG_OK;
}

int lg_graph_destroy(void* exec) {
  if (exec) cudaGraphExecDestroy((cudaGraphExec_t)exec);
  return LG_OK;
}

int lg_ws_create(lg_ws** out) {
  if (!out) return lg::fail(LG_EINVAL, "lg_ws_create: out is NULL");
  lg_ws* ws = new lg_ws();
  size_t pbytes = sizeof(double) * (size_t)lg::kMaxRedBlocks * lg::kMaxRedVals;
  if (cudaMalloc(&ws->partial, pbytes) != cudaSuccess ||
      cudaMalloc(&ws->ticket, sizeof(unsigned)) != cudaSuccess) {
    cudaFree(ws->partial);
    delete ws;
    return lg::fail(LG_ENOMEM, "lg_ws_create: cudaMalloc failed");
  }
  cudaMemset(ws->ticket, 0, sizeof(unsigned));
  cudaDeviceSynchronize();
  *out = ws;
  return LG_OK;
}

int lg_ws_destroy(lg_ws* ws) {
  if (!ws) return LG_OK;
  cudaFree(ws->partial);
  cudaFree(ws->ticket);
  cudaFree(ws->long_dots);
  cudaFree(ws->long_ticket);
  cudaFree(ws->long_part);
  cudaFree(ws->mm_part);
  delete ws;
  return LG_OK;
}

}  // extern "C"
