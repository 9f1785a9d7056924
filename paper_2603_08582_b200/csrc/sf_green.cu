// sf_green.cu -- optional spatial partition of the SMs (green contexts).
//
// The cfg1 FISTA chain is latency-bound while the operator phase of later
// pulses (K~ build, power iteration) runs beside it on the pipeline streams
// and competes for SMs.  With SF_GREEN_SMS=K the engine creates two green
// contexts over disjoint SM sets -- K SMs for the FISTA replay stream, the
// rest for the pipeline and state streams -- so the two phases stop stealing
// each other's SMs (they still share L2 and HBM).  Driver entry points are
// resolved with dlopen (libcuda.so.1 is already loaded by the runtime).
#include <cuda.h>
#include <dlfcn.h>

#include <string>

#include "sf_common.cuh"
#include "sf_kernels.cuh"

namespace sf {

namespace {
struct GreenApi {
  bool ok = false;
  CUresult (*deviceGet)(CUdevice *, int) = nullptr;
  CUresult (*getDevResource)(CUdevice, CUdevResource *, CUdevResourceType) = nullptr;
  CUresult (*split)(CUdevResource *, unsigned int *, const CUdevResource *, CUdevResource *,
                    unsigned int, unsigned int) = nullptr;
  CUresult (*genDesc)(CUdevResourceDesc *, CUdevResource *, unsigned int) = nullptr;
  CUresult (*create)(CUgreenCtx *, CUdevResourceDesc, CUdevice, unsigned int) = nullptr;
  CUresult (*streamCreate)(CUstream *, CUgreenCtx, unsigned int, int) = nullptr;
};

GreenApi &api() {
  static GreenApi a;
  static bool tried = false;
  if (tried) return a;
  tried = true;
  void *h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libcuda.so.1", RTLD_NOW);
  if (!h) return a;
  a.deviceGet = (decltype(a.deviceGet))dlsym(h, "cuDeviceGet");
  a.getDevResource = (decltype(a.getDevResource))dlsym(h, "cuDeviceGetDevResource");
  a.split = (decltype(a.split))dlsym(h, "cuDevSmResourceSplitByCount");
  a.genDesc = (decltype(a.genDesc))dlsym(h, "cuDevResourceGenerateDesc");
  a.create = (decltype(a.create))dlsym(h, "cuGreenCtxCreate");
  a.streamCreate = (decltype(a.streamCreate))dlsym(h, "cuGreenCtxStreamCreate");
  a.ok = a.deviceGet && a.getDevResource && a.split && a.genDesc && a.create && a.streamCreate;
  return a;
}
}  // namespace

// Streams on two disjoint SM partitions: `fista` on >= k SMs, the returned
// `rest` streams on the remaining SMs.  Returns SF_EUNSUPPORTED when green
// contexts are unavailable (the caller keeps its ordinary streams).
sf_status green_partition(int device, int k, int hi_prio, int lo_prio, cudaStream_t *fista,
                          cudaStream_t *rest, int n_rest, int *sms_fista, int *sms_rest) {
  GreenApi &a = api();
  if (!a.ok) return fail(SF_EUNSUPPORTED, "green contexts unavailable");
  CUdevice dev;
  if (a.deviceGet(&dev, device) != CUDA_SUCCESS) return fail(SF_ECUDA, "cuDeviceGet");
  CUdevResource all{};
  if (a.getDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS)
    return fail(SF_EUNSUPPORTED, "cuDeviceGetDevResource");
  CUdevResource grp{}, remaining{};
  unsigned int n = 1;
  if (a.split(&grp, &n, &all, &remaining, 0, (unsigned)k) != CUDA_SUCCESS || n < 1)
    return fail(SF_EUNSUPPORTED, "cuDevSmResourceSplitByCount");
  CUdevResourceDesc d1, d2;
  if (a.genDesc(&d1, &grp, 1) != CUDA_SUCCESS || a.genDesc(&d2, &remaining, 1) != CUDA_SUCCESS)
    return fail(SF_EUNSUPPORTED, "cuDevResourceGenerateDesc");
  CUgreenCtx g1, g2;
  if (a.create(&g1, d1, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS ||
      a.create(&g2, d2, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS)
    return fail(SF_EUNSUPPORTED, "cuGreenCtxCreate");
  CUstream s;
  if (a.streamCreate(&s, g1, CU_STREAM_NON_BLOCKING, hi_prio) != CUDA_SUCCESS)
    return fail(SF_EUNSUPPORTED, "cuGreenCtxStreamCreate");
  *fista = (cudaStream_t)s;
  for (int i = 0; i < n_rest; ++i) {
    if (a.streamCreate(&s, g2, CU_STREAM_NON_BLOCKING, i == 0 ? hi_prio : lo_prio) != CUDA_SUCCESS)
      return fail(SF_EUNSUPPORTED, "cuGreenCtxStreamCreate");
    rest[i] = (cudaStream_t)s;
  }
  *sms_fista = (int)grp.sm.smCount;
  *sms_rest = (int)remaining.sm.smCount;
  return SF_OK;
}

}  // namespace sf
