// ct_tune.cu -- C ABI of the live measurement path (include/countertune_tune.h):
// NVRTC variant compiler + launcher and CUPTI range-profiler collector.
//
// The reference replays recorded measurements (search.py:197-217) or talks to
// an external runner over a line protocol (search.py:220-275); this library
// is the in-process B200 runner behind CudaMeasurementSource (tuner.py):
//   * every configuration of a tuning space is one NVRTC compilation of the
//     benchmark source with -D<PARAM>=<value> options, for this device's
//     sm_XXXa target, cached by handle;
//   * runtimes come from CUDA events around single launches on the tuner's
//     stream, with an optional L2 flush between launches;
//   * counters come from the CUPTI range profiler (user range, user replay:
//     the kernel is re-launched once per pass; benchmark kernels are
//     idempotent), evaluated on the host to GPU metric values.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nvrtc.h>
#include <cstdio>
#include <cupti_profiler_host.h>
#include <cupti_profiler_target.h>
#include <cupti_range_profiler.h>
#include <cupti_target.h>

#include <algorithm>
#include <chrono>
#include <map>
#include <memory>
#include <atomic>
#include <thread>
#include <cstring>
#include <string>
#include <vector>

#include "countertune_tune.h"

namespace {

// Driver API through the runtime's entry-point table: the library links
// only cudart/NVRTC/CUPTI, so it loads (and reports "no CUDA device") on a
// host without the driver, like libct_b200.so.
struct DriverTable {
#define CT_DRV(fn) decltype(&::fn) fn = nullptr;
    CT_DRV(cuInit) CT_DRV(cuDeviceGet) CT_DRV(cuDevicePrimaryCtxRetain)
    CT_DRV(cuDevicePrimaryCtxRelease) CT_DRV(cuCtxSetCurrent) CT_DRV(cuGetErrorString)
    CT_DRV(cuModuleLoadData) CT_DRV(cuModuleGetFunction) CT_DRV(cuModuleUnload)
    CT_DRV(cuFuncGetAttribute) CT_DRV(cuFuncSetAttribute) CT_DRV(cuLaunchKernel)
    CT_DRV(cuTensorMapEncodeTiled)
#undef CT_DRV
    bool ready = false;
};
DriverTable D;

bool load_driver() {
    if (D.ready) return true;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n < 1) return false;
    bool ok = true;
#define CT_DRV(fn)                                                                           \
    {                                                                                        \
        void* p_ = nullptr;                                                                  \
        cudaDriverEntryPointQueryResult q_;                                                  \
        if (cudaGetDriverEntryPoint(#fn, &p_, cudaEnableDefault, &q_) != cudaSuccess ||      \
            q_ != cudaDriverEntryPointSuccess || !p_)                                        \
            ok = false;                                                                      \
        D.fn = reinterpret_cast<decltype(D.fn)>(p_);                                         \
    }
    CT_DRV(cuInit) CT_DRV(cuDeviceGet) CT_DRV(cuDevicePrimaryCtxRetain)
    CT_DRV(cuDevicePrimaryCtxRelease) CT_DRV(cuCtxSetCurrent) CT_DRV(cuGetErrorString)
    CT_DRV(cuModuleLoadData) CT_DRV(cuModuleGetFunction) CT_DRV(cuModuleUnload)
    CT_DRV(cuFuncGetAttribute) CT_DRV(cuFuncSetAttribute) CT_DRV(cuLaunchKernel)
    CT_DRV(cuTensorMapEncodeTiled)
#undef CT_DRV
    D.ready = ok;
    return ok;
}

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

std::string cu_msg(CUresult r) {
    const char* s = nullptr;
    if (D.cuGetErrorString) D.cuGetErrorString(r, &s);
    return s ? s : "unknown CUDA driver error";
}

#define TU_CU(call)                                                                          \
    do {                                                                                     \
        CUresult r_ = (call);                                                                \
        if (r_ != CUDA_SUCCESS) return fail(CT_TUNE_ERR_CUDA, std::string(#call) + ": " + cu_msg(r_)); \
    } while (0)

#define TU_RT(call)                                                                          \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess)                                                               \
            return fail(CT_TUNE_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define TU_CUPTI(call)                                                                       \
    do {                                                                                     \
        CUptiResult c_ = (call);                                                             \
        if (c_ != CUPTI_SUCCESS) {                                                           \
            const char* m_ = nullptr;                                                        \
            cuptiGetResultString(c_, &m_);                                                   \
            return fail(CT_TUNE_ERR_PROFILER, std::string(#call) + ": " + (m_ ? m_ : "?")); \
        }                                                                                    \
    } while (0)

struct Variant {
    CUmodule mod = nullptr;
    CUfunction fn = nullptr;
    size_t smem_attr = 0;
};

}  // namespace

namespace {
// Host configuration of a metric set: config image + pass count.
struct HostConfig {
    CUpti_Profiler_Host_Object* host = nullptr;
    // the metric names, owned here: every CUPTI call of this configuration
    // gets these pointers, never the caller's (which live for one call)
    std::vector<std::string> names;
    std::vector<const char*> name_ptrs;
    std::vector<uint8_t> image;
    size_t passes = 0;
    std::vector<uint8_t> counter_data;   // one-range counter data image
    ~HostConfig() {
        if (host) {
            CUpti_Profiler_Host_Deinitialize_Params dp = {sizeof(CUpti_Profiler_Host_Deinitialize_Params)};
            dp.pHostObject = host;
            cuptiProfilerHostDeinitialize(&dp);
        }
    }
};

}  // namespace

struct ct_tuner {
    int device = 0;
    CUdevice dev = 0;
    CUcontext ctx = nullptr;
    cudaStream_t stream = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    std::vector<Variant> variants;
    std::vector<void*> allocs;
    void* flush = nullptr;
    size_t flush_bytes = 0;
    std::string arch;
    int sm_count = 0, max_threads_sm = 0;
    // CUPTI
    bool cupti_ready = false;
    std::string chip;
    std::vector<uint8_t> avail;
    CUpti_RangeProfiler_Object* rp = nullptr;
    // the metric set the range-profiler object was last configured with: a
    // SetConfig with another set does not take effect on the same object
    // (it keeps the first set's pass count and leaves the new metrics NaN),
    // so a switch of set re-creates the object
    const void* rp_config = nullptr;
    int32_t rp_ranges = 0;            // ranges per pass it was configured for
    // host configurations by metric set (building one costs milliseconds)
    std::map<std::string, std::unique_ptr<HostConfig>> configs;
    // wall time of ct_tuner_profile by phase (microseconds, accumulated):
    // [0] counter-data init + SetConfig, [1] replay passes (range + launch),
    // [2] stream sync, [3] DecodeData, [4] evaluation, [5] calls, [6] passes,
    // [7] host-config build (first use of a metric set)
    double prof_us[8] = {0, 0, 0, 0, 0, 0, 0, 0};
};

namespace {

int activate(ct_tuner* t) {
    if (!t) return fail(CT_TUNE_ERR_VALUE, "null tuner");
    TU_RT(cudaSetDevice(t->device));
    TU_CU(D.cuCtxSetCurrent(t->ctx));
    return CT_TUNE_OK;
}

int get_variant(ct_tuner* t, int32_t v, Variant** out) {
    if (v < 0 || v >= (int32_t)t->variants.size() || !t->variants[v].fn)
        return fail(CT_TUNE_ERR_VALUE, "unknown variant " + std::to_string(v));
    *out = &t->variants[v];
    return CT_TUNE_OK;
}

// NVRTC: source + -D options -> cubin for this device (thread-safe).
bool compile_cubin(const std::string& arch, const char* source, const char* const* options,
                   int32_t n_options, std::vector<char>* cubin, std::string* log) {
    nvrtcProgram prog;
    nvrtcResult nr = nvrtcCreateProgram(&prog, source, "variant.cu", 0, nullptr, nullptr);
    if (nr != NVRTC_SUCCESS) { *log = nvrtcGetErrorString(nr); return false; }
    std::vector<std::string> opts = {"--gpu-architecture=" + arch, "--std=c++17",
                                     "--device-as-default-execution-space", "-lineinfo"};
    for (int i = 0; i < n_options; ++i) opts.emplace_back(options[i]);
    std::vector<const char*> optp;
    for (auto& o : opts) optp.push_back(o.c_str());
    nr = nvrtcCompileProgram(prog, (int)optp.size(), optp.data());
    size_t log_size = 0;
    nvrtcGetProgramLogSize(prog, &log_size);
    log->assign(log_size, '\0');
    if (log_size) nvrtcGetProgramLog(prog, &(*log)[0]);
    if (!log->empty() && log->back() == '\0') log->pop_back();
    if (nr != NVRTC_SUCCESS) {
        *log = std::string(nvrtcGetErrorString(nr)) + "\n" + *log;
        nvrtcDestroyProgram(&prog);
        return false;
    }
    size_t cubin_size = 0;
    nvrtcGetCUBINSize(prog, &cubin_size);
    cubin->resize(cubin_size);
    nvrtcGetCUBIN(prog, cubin->data());
    nvrtcDestroyProgram(&prog);
    return true;
}

int load_variant(ct_tuner* t, const std::vector<char>& cubin, const char* name, int32_t* variant) {
    Variant v;
    CUresult r = D.cuModuleLoadData(&v.mod, cubin.data());
    if (r != CUDA_SUCCESS) return fail(CT_TUNE_ERR_COMPILE, "cuModuleLoadData: " + cu_msg(r));
    r = D.cuModuleGetFunction(&v.fn, v.mod, name);
    if (r != CUDA_SUCCESS) {
        D.cuModuleUnload(v.mod);
        return fail(CT_TUNE_ERR_COMPILE, std::string("kernel ") + name + " not found: " + cu_msg(r));
    }
    t->variants.push_back(v);
    *variant = (int32_t)t->variants.size() - 1;
    return CT_TUNE_OK;
}

int launch_once(ct_tuner* t, Variant* var, const ct_launch* l) {
    std::vector<void*> params((size_t)std::max(l->n_args, 0));
    for (int i = 0; i < l->n_args; ++i)
        params[i] = const_cast<char*>(static_cast<const char*>(l->args) + l->arg_offsets[i]);
    // the opt-in limit counts dynamic + static shared memory: raise it for any
    // dynamic request (48 KB of dynamic memory on top of static fails otherwise)
    if (l->dynamic_smem > var->smem_attr) {
        TU_CU(D.cuFuncSetAttribute(var->fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES,
                                 (int)l->dynamic_smem));
        var->smem_attr = l->dynamic_smem;
    }
    CUresult r = D.cuLaunchKernel(var->fn, l->grid[0], l->grid[1], l->grid[2], l->block[0],
                                l->block[1], l->block[2], l->dynamic_smem, (CUstream)t->stream,
                                params.data(), nullptr);
    if (r != CUDA_SUCCESS) return fail(CT_TUNE_ERR_LAUNCH, "cuLaunchKernel: " + cu_msg(r));
    return CT_TUNE_OK;
}

int cupti_init(ct_tuner* t) {
    if (t->cupti_ready) return CT_TUNE_OK;
    CUpti_Profiler_Initialize_Params ip = {CUpti_Profiler_Initialize_Params_STRUCT_SIZE};
    TU_CUPTI(cuptiProfilerInitialize(&ip));
    CUpti_Device_GetChipName_Params cp = {CUpti_Device_GetChipName_Params_STRUCT_SIZE};
    cp.deviceIndex = (size_t)t->device;
    TU_CUPTI(cuptiDeviceGetChipName(&cp));
    t->chip = cp.pChipName;
    CUpti_Profiler_GetCounterAvailability_Params ap = {CUpti_Profiler_GetCounterAvailability_Params_STRUCT_SIZE};
    ap.ctx = t->ctx;
    TU_CUPTI(cuptiProfilerGetCounterAvailability(&ap));
    t->avail.assign(ap.counterAvailabilityImageSize, 0);
    ap.pCounterAvailabilityImage = t->avail.data();
    TU_CUPTI(cuptiProfilerGetCounterAvailability(&ap));
    CUpti_RangeProfiler_Enable_Params ep = {CUpti_RangeProfiler_Enable_Params_STRUCT_SIZE};
    ep.ctx = t->ctx;
    TU_CUPTI(cuptiRangeProfilerEnable(&ep));
    t->rp = ep.pRangeProfilerObject;
    t->cupti_ready = true;
    return CT_TUNE_OK;
}

int host_config(ct_tuner* t, const char* const* metrics_in, int32_t n, HostConfig* hc) {
    hc->names.assign(metrics_in, metrics_in + n);
    hc->name_ptrs.clear();
    for (const std::string& m : hc->names) hc->name_ptrs.push_back(m.c_str());
    const char* const* metrics = hc->name_ptrs.data();
    CUpti_Profiler_Host_Initialize_Params hp = {sizeof(CUpti_Profiler_Host_Initialize_Params)};
    hp.profilerType = CUPTI_PROFILER_TYPE_RANGE_PROFILER;
    hp.pChipName = t->chip.c_str();
    hp.pCounterAvailabilityImage = t->avail.data();
    TU_CUPTI(cuptiProfilerHostInitialize(&hp));
    hc->host = hp.pHostObject;
    CUpti_Profiler_Host_ConfigAddMetrics_Params mp = {sizeof(CUpti_Profiler_Host_ConfigAddMetrics_Params)};
    mp.pHostObject = hc->host;
    mp.ppMetricNames = const_cast<const char**>(metrics);
    mp.numMetrics = (size_t)n;
    TU_CUPTI(cuptiProfilerHostConfigAddMetrics(&mp));
    CUpti_Profiler_Host_GetConfigImageSize_Params sp = {sizeof(CUpti_Profiler_Host_GetConfigImageSize_Params)};
    sp.pHostObject = hc->host;
    TU_CUPTI(cuptiProfilerHostGetConfigImageSize(&sp));
    hc->image.assign(sp.configImageSize, 0);
    CUpti_Profiler_Host_GetConfigImage_Params gp = {sizeof(CUpti_Profiler_Host_GetConfigImage_Params)};
    gp.pHostObject = hc->host;
    gp.configImageSize = hc->image.size();
    gp.pConfigImage = hc->image.data();
    TU_CUPTI(cuptiProfilerHostGetConfigImage(&gp));
    CUpti_Profiler_Host_GetNumOfPasses_Params np = {sizeof(CUpti_Profiler_Host_GetNumOfPasses_Params)};
    np.configImageSize = hc->image.size();
    np.pConfigImage = hc->image.data();
    TU_CUPTI(cuptiProfilerHostGetNumOfPasses(&np));
    hc->passes = np.numOfPasses;
    return CT_TUNE_OK;
}

// cached host configuration of a metric set
int host_config_cached(ct_tuner* t, const char* const* metrics, int32_t n, HostConfig** out) {
    std::string key;
    for (int i = 0; i < n; ++i) { key += metrics[i]; key += '\n'; }
    auto it = t->configs.find(key);
    if (it == t->configs.end()) {
        std::unique_ptr<HostConfig> hc(new HostConfig());
        int rc = host_config(t, metrics, n, hc.get()); if (rc) return rc;
        it = t->configs.emplace(key, std::move(hc)).first;
    }
    *out = it->second.get();
    return CT_TUNE_OK;
}

// The range-profiler object serves one collection shape: a SetConfig with
// another metric set does not take effect on it (the first set's pass count
// stays, the new metrics read NaN), and after a k-range collection a 1-range
// counter-data image no longer initialises against it.  A change of (metric
// set, ranges per pass) therefore re-creates the object.
int rp_shape(ct_tuner* t, HostConfig* hc, int32_t ranges) {
    if (!t->rp || (t->rp_config && (t->rp_config != hc || t->rp_ranges != ranges))) {
        if (t->rp) {
            CUpti_RangeProfiler_Disable_Params dp = {CUpti_RangeProfiler_Disable_Params_STRUCT_SIZE};
            dp.pRangeProfilerObject = t->rp;
            TU_CUPTI(cuptiRangeProfilerDisable(&dp));
        }
        CUpti_RangeProfiler_Enable_Params ep = {CUpti_RangeProfiler_Enable_Params_STRUCT_SIZE};
        ep.ctx = t->ctx;
        TU_CUPTI(cuptiRangeProfilerEnable(&ep));
        t->rp = ep.pRangeProfilerObject;
        // counter-data images were sized and initialised against the old
        // object: every configuration re-derives its image under the new one
        for (auto& kv : t->configs) kv.second->counter_data.clear();
    }
    t->rp_config = hc;
    t->rp_ranges = ranges;
    return CT_TUNE_OK;
}

}  // namespace

extern "C" {

int ct_tune_abi_version(void) { return CT_TUNE_ABI_VERSION; }

const char* ct_tune_last_error(void) { return g_err.c_str(); }

int ct_tuner_create(int device, ct_tuner** out) {
    if (!out) return fail(CT_TUNE_ERR_VALUE, "null output");
    *out = nullptr;
    if (!load_driver()) return fail(CT_TUNE_ERR_CUDA, "no CUDA device");
    TU_CU(D.cuInit(0));
    ct_tuner* t = new ct_tuner();
    t->device = device;
    CUresult r = D.cuDeviceGet(&t->dev, device);
    if (r == CUDA_SUCCESS) r = D.cuDevicePrimaryCtxRetain(&t->ctx, t->dev);
    if (r != CUDA_SUCCESS) { delete t; return fail(CT_TUNE_ERR_CUDA, cu_msg(r)); }
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaFree(nullptr);   // bind the runtime to the primary context
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&t->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreate(&t->e0);
    if (e == cudaSuccess) e = cudaEventCreate(&t->e1);
    if (e != cudaSuccess) { delete t; return fail(CT_TUNE_ERR_CUDA, cudaGetErrorString(e)); }
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
    cudaDeviceGetAttribute(&t->sm_count, cudaDevAttrMultiProcessorCount, device);
    cudaDeviceGetAttribute(&t->max_threads_sm, cudaDevAttrMaxThreadsPerMultiProcessor, device);
    t->arch = "sm_" + std::to_string(major * 10 + minor) + (major >= 9 ? "a" : "");
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device);
    t->flush_bytes = std::max<size_t>((size_t)l2 * 2, 64u << 20);
    *out = t;
    return CT_TUNE_OK;
}

int ct_tuner_destroy(ct_tuner* t) {
    if (!t) return CT_TUNE_OK;
    cudaSetDevice(t->device);
    D.cuCtxSetCurrent(t->ctx);
    cudaStreamSynchronize(t->stream);
    t->configs.clear();
    if (t->rp) {
        CUpti_RangeProfiler_Disable_Params dp = {CUpti_RangeProfiler_Disable_Params_STRUCT_SIZE};
        dp.pRangeProfilerObject = t->rp;
        cuptiRangeProfilerDisable(&dp);
    }
    for (auto& v : t->variants)
        if (v.mod) D.cuModuleUnload(v.mod);
    for (void* p : t->allocs) cudaFree(p);
    if (t->flush) cudaFree(t->flush);
    cudaEventDestroy(t->e0);
    cudaEventDestroy(t->e1);
    cudaStreamDestroy(t->stream);
    D.cuDevicePrimaryCtxRelease(t->dev);
    delete t;
    return CT_TUNE_OK;
}

int ct_tuner_device_info(ct_tuner* t, char* arch, int32_t cap, int32_t* sm_count,
                         int32_t* max_threads_sm) {
    if (!t) return fail(CT_TUNE_ERR_VALUE, "null tuner");
    if (arch && cap > 0) {
        std::strncpy(arch, t->arch.c_str(), (size_t)cap - 1);
        arch[cap - 1] = 0;
    }
    if (sm_count) *sm_count = t->sm_count;
    if (max_threads_sm) *max_threads_sm = t->max_threads_sm;
    return CT_TUNE_OK;
}

int ct_tuner_compile(ct_tuner* t, const char* source, const char* name, const char* const* options,
                     int32_t n_options, int32_t* variant, char* log, int64_t log_cap) {
    int rc = activate(t); if (rc) return rc;
    if (!source || !name || !variant || n_options < 0 || (n_options && !options))
        return fail(CT_TUNE_ERR_VALUE, "bad compile arguments");
    std::vector<char> cubin;
    std::string plog;
    bool ok = compile_cubin(t->arch, source, options, n_options, &cubin, &plog);
    if (log && log_cap > 0) {
        std::strncpy(log, plog.c_str(), (size_t)log_cap - 1);
        log[log_cap - 1] = 0;
    }
    if (!ok) return fail(CT_TUNE_ERR_COMPILE, plog);
    return load_variant(t, cubin, name, variant);
}

int ct_tuner_compile_batch(ct_tuner* t, const char* source, const char* name,
                           const char* const* options_flat, const int32_t* n_options,
                           int32_t n_variants, int32_t threads, int32_t* variants,
                           int32_t* status) {
    int rc = activate(t); if (rc) return rc;
    if (!source || !name || n_variants < 0 || (n_variants && (!n_options || !variants || !status)))
        return fail(CT_TUNE_ERR_VALUE, "bad compile_batch arguments");
    std::vector<int64_t> first(n_variants + 1, 0);
    for (int i = 0; i < n_variants; ++i) {
        if (n_options[i] < 0) return fail(CT_TUNE_ERR_VALUE, "negative option count");
        first[i + 1] = first[i] + n_options[i];
    }
    if (first[n_variants] && !options_flat) return fail(CT_TUNE_ERR_VALUE, "null options");
    std::vector<std::vector<char>> cubins(n_variants);
    std::vector<std::string> logs(n_variants);
    std::vector<char> ok(n_variants, 0);
    int nt = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
    nt = std::min(nt, std::max(n_variants, 1));
    std::atomic<int> next{0};
    auto worker = [&]() {
        for (int i = next++; i < n_variants; i = next++)
            ok[i] = compile_cubin(t->arch, source, options_flat + first[i], n_options[i],
                                  &cubins[i], &logs[i]);
    };
    std::vector<std::thread> pool;
    for (int k = 1; k < nt; ++k) pool.emplace_back(worker);
    worker();
    for (auto& th : pool) th.join();
    // modules are loaded on the calling thread, into the tuner's context
    std::string first_err;
    for (int i = 0; i < n_variants; ++i) {
        variants[i] = -1;
        if (!ok[i]) {
            status[i] = CT_TUNE_ERR_COMPILE;
            if (first_err.empty()) first_err = logs[i];
            continue;
        }
        status[i] = load_variant(t, cubins[i], name, &variants[i]);
        if (status[i] && first_err.empty()) first_err = g_err;
    }
    g_err = first_err;
    return CT_TUNE_OK;
}

int ct_tuner_variant_info(ct_tuner* t, int32_t variant, int32_t* regs, int32_t* smem,
                          int32_t* max_threads) {
    int rc = activate(t); if (rc) return rc;
    Variant* v = nullptr;
    rc = get_variant(t, variant, &v); if (rc) return rc;
    int a = 0;
    if (regs) { TU_CU(D.cuFuncGetAttribute(&a, CU_FUNC_ATTRIBUTE_NUM_REGS, v->fn)); *regs = a; }
    if (smem) { TU_CU(D.cuFuncGetAttribute(&a, CU_FUNC_ATTRIBUTE_SHARED_SIZE_BYTES, v->fn)); *smem = a; }
    if (max_threads) {
        TU_CU(D.cuFuncGetAttribute(&a, CU_FUNC_ATTRIBUTE_MAX_THREADS_PER_BLOCK, v->fn));
        *max_threads = a;
    }
    return CT_TUNE_OK;
}

int ct_tuner_unload(ct_tuner* t, int32_t variant) {
    int rc = activate(t); if (rc) return rc;
    Variant* v = nullptr;
    rc = get_variant(t, variant, &v); if (rc) return rc;
    // the range profiler keeps per-module state for the kernels it has
    // instrumented (the SASS-patched instruction-class metrics): unloading
    // a module under a live profiler object crashed a later collection, so
    // the object is released first and re-created by the next collection
    if (t->rp) {
        CUpti_RangeProfiler_Disable_Params dp = {CUpti_RangeProfiler_Disable_Params_STRUCT_SIZE};
        dp.pRangeProfilerObject = t->rp;
        TU_CUPTI(cuptiRangeProfilerDisable(&dp));
        t->rp = nullptr;
        t->rp_config = nullptr;
        for (auto& kv : t->configs) kv.second->counter_data.clear();
    }
    TU_CU(D.cuModuleUnload(v->mod));
    v->mod = nullptr;
    v->fn = nullptr;
    return CT_TUNE_OK;
}

int ct_tuner_alloc(ct_tuner* t, int64_t bytes, uint64_t* dev_ptr) {
    int rc = activate(t); if (rc) return rc;
    if (bytes < 0 || !dev_ptr) return fail(CT_TUNE_ERR_VALUE, "bad allocation");
    void* p = nullptr;
    TU_RT(cudaMalloc(&p, (size_t)std::max<int64_t>(bytes, 1)));
    t->allocs.push_back(p);
    *dev_ptr = (uint64_t)(uintptr_t)p;
    return CT_TUNE_OK;
}

int ct_tuner_free(ct_tuner* t, uint64_t dev_ptr) {
    int rc = activate(t); if (rc) return rc;
    void* p = (void*)(uintptr_t)dev_ptr;
    auto it = std::find(t->allocs.begin(), t->allocs.end(), p);
    if (it == t->allocs.end()) return fail(CT_TUNE_ERR_VALUE, "pointer not owned by the tuner");
    TU_RT(cudaStreamSynchronize(t->stream));
    TU_RT(cudaFree(p));
    t->allocs.erase(it);
    return CT_TUNE_OK;
}

int ct_tuner_h2d(ct_tuner* t, uint64_t dev, const void* host, int64_t bytes) {
    int rc = activate(t); if (rc) return rc;
    TU_RT(cudaMemcpyAsync((void*)(uintptr_t)dev, host, (size_t)bytes, cudaMemcpyHostToDevice, t->stream));
    TU_RT(cudaStreamSynchronize(t->stream));
    return CT_TUNE_OK;
}

int ct_tuner_d2h(ct_tuner* t, void* host, uint64_t dev, int64_t bytes) {
    int rc = activate(t); if (rc) return rc;
    TU_RT(cudaMemcpyAsync(host, (void*)(uintptr_t)dev, (size_t)bytes, cudaMemcpyDeviceToHost, t->stream));
    TU_RT(cudaStreamSynchronize(t->stream));
    return CT_TUNE_OK;
}

int ct_tuner_memset(ct_tuner* t, uint64_t dev, int32_t value, int64_t bytes) {
    int rc = activate(t); if (rc) return rc;
    TU_RT(cudaMemsetAsync((void*)(uintptr_t)dev, value, (size_t)bytes, t->stream));
    TU_RT(cudaStreamSynchronize(t->stream));
    return CT_TUNE_OK;
}

int ct_tuner_time(ct_tuner* t, int32_t variant, const ct_launch* l, int32_t warmup, int32_t reps,
                  int32_t flush_l2, double* times_us) {
    int rc = activate(t); if (rc) return rc;
    if (!l || reps < 0 || warmup < 0 || (reps && !times_us)) return fail(CT_TUNE_ERR_VALUE, "bad timing arguments");
    Variant* v = nullptr;
    rc = get_variant(t, variant, &v); if (rc) return rc;
    if (flush_l2 && !t->flush) TU_RT(cudaMalloc(&t->flush, t->flush_bytes));
    for (int i = 0; i < warmup; ++i) { rc = launch_once(t, v, l); if (rc) return rc; }
    for (int i = 0; i < reps; ++i) {
        if (flush_l2) TU_RT(cudaMemsetAsync(t->flush, i & 0xff, t->flush_bytes, t->stream));
        TU_RT(cudaEventRecord(t->e0, t->stream));
        rc = launch_once(t, v, l); if (rc) return rc;
        TU_RT(cudaEventRecord(t->e1, t->stream));
        cudaError_t e = cudaEventSynchronize(t->e1);
        if (e != cudaSuccess) return fail(CT_TUNE_ERR_LAUNCH, std::string("kernel failed: ") + cudaGetErrorString(e));
        float ms = 0.0f;
        TU_RT(cudaEventElapsedTime(&ms, t->e0, t->e1));
        times_us[i] = (double)ms * 1e3;
    }
    TU_RT(cudaStreamSynchronize(t->stream));
    return CT_TUNE_OK;
}

int ct_tuner_profile_passes(ct_tuner* t, const char* const* metrics, int32_t n, int32_t* passes) {
    int rc = activate(t); if (rc) return rc;
    if (!metrics || n < 1 || !passes) return fail(CT_TUNE_ERR_VALUE, "bad metric list");
    rc = cupti_init(t); if (rc) return rc;
    HostConfig* hc = nullptr;
    rc = host_config_cached(t, metrics, n, &hc); if (rc) return rc;
    *passes = (int32_t)hc->passes;
    return CT_TUNE_OK;
}

int ct_tuner_profile(ct_tuner* t, int32_t variant, const ct_launch* l, const char* const* metrics,
                     int32_t n, double* values, int32_t* passes) {
    int rc = activate(t); if (rc) return rc;
    if (!l || !metrics || n < 1 || !values) return fail(CT_TUNE_ERR_VALUE, "bad profile arguments");
    Variant* v = nullptr;
    rc = get_variant(t, variant, &v); if (rc) return rc;
    rc = cupti_init(t); if (rc) return rc;
    using clk = std::chrono::steady_clock;
    auto us = [](clk::time_point a, clk::time_point b) {
        return std::chrono::duration<double, std::micro>(b - a).count();
    };
    const auto t0 = clk::now();
    HostConfig* hc = nullptr;
    rc = host_config_cached(t, metrics, n, &hc); if (rc) return rc;
    rc = rp_shape(t, hc, 1); if (rc) return rc;
    const auto t1 = clk::now();
    t->prof_us[7] += us(t0, t1);
    // counter data image for one range (re-initialised per collection)
    if (hc->counter_data.empty()) {
        CUpti_RangeProfiler_GetCounterDataSize_Params cs = {CUpti_RangeProfiler_GetCounterDataSize_Params_STRUCT_SIZE};
        cs.pRangeProfilerObject = t->rp;
        cs.pMetricNames = hc->name_ptrs.data();
        cs.numMetrics = (size_t)n;
        cs.maxNumOfRanges = 1;
        cs.maxNumRangeTreeNodes = 1;
        TU_CUPTI(cuptiRangeProfilerGetCounterDataSize(&cs));
        hc->counter_data.assign(cs.counterDataSize, 0);
    }
    std::vector<uint8_t>& data = hc->counter_data;
    CUpti_RangeProfiler_CounterDataImage_Initialize_Params ci = {CUpti_RangeProfiler_CounterDataImage_Initialize_Params_STRUCT_SIZE};
    ci.pRangeProfilerObject = t->rp;
    ci.counterDataSize = data.size();
    ci.pCounterData = data.data();
    TU_CUPTI(cuptiRangeProfilerCounterDataImageInitialize(&ci));
    CUpti_RangeProfiler_SetConfig_Params sc = {CUpti_RangeProfiler_SetConfig_Params_STRUCT_SIZE};
    sc.pRangeProfilerObject = t->rp;
    sc.configSize = hc->image.size();
    sc.pConfig = hc->image.data();
    sc.counterDataImageSize = data.size();
    sc.pCounterDataImage = data.data();
    // user range + user replay: one launch of ours per pass (CUPTI's kernel
    // replay with an auto range returned zeros for every metric here)
    static const bool trace = std::getenv("CT_TUNE_TRACE") != nullptr;
    sc.range = CUPTI_UserRange;
    sc.replayMode = CUPTI_UserReplay;
    sc.maxRangesPerPass = 1;
    sc.numNestingLevels = 1;
    sc.minNestingLevel = 1;
    sc.passIndex = 0;
    sc.targetNestingLevel = 1;
    TU_CUPTI(cuptiRangeProfilerSetConfig(&sc));
    const auto t2 = clk::now();
    int used = 0;
    for (;;) {
        const auto q0 = clk::now();
        CUpti_RangeProfiler_Start_Params st = {CUpti_RangeProfiler_Start_Params_STRUCT_SIZE};
        st.pRangeProfilerObject = t->rp;
        TU_CUPTI(cuptiRangeProfilerStart(&st));
        const auto q1 = clk::now();
        CUpti_RangeProfiler_PushRange_Params pr = {CUpti_RangeProfiler_PushRange_Params_STRUCT_SIZE};
        pr.pRangeProfilerObject = t->rp;
        pr.pRangeName = "variant";
        TU_CUPTI(cuptiRangeProfilerPushRange(&pr));
        rc = launch_once(t, v, l);
        const auto q2 = clk::now();
        CUpti_RangeProfiler_PopRange_Params po = {CUpti_RangeProfiler_PopRange_Params_STRUCT_SIZE};
        po.pRangeProfilerObject = t->rp;
        TU_CUPTI(cuptiRangeProfilerPopRange(&po));
        CUpti_RangeProfiler_Stop_Params sp = {CUpti_RangeProfiler_Stop_Params_STRUCT_SIZE};
        sp.pRangeProfilerObject = t->rp;
        TU_CUPTI(cuptiRangeProfilerStop(&sp));
        const auto q3 = clk::now();
        if (trace)
            std::fprintf(stderr, "[ct_tune] pass %d: start %.1f us, push+launch %.1f us, pop+stop %.1f us%s\n",
                         used, us(q0, q1), us(q1, q2), us(q2, q3),
                         sp.isAllPassSubmitted ? " (all passes submitted)" : "");
        if (rc) return rc;
        ++used;
        if (sp.isAllPassSubmitted) break;
        if (used > 64) return fail(CT_TUNE_ERR_PROFILER, "range profiler did not finish its passes");
    }
    const auto t3 = clk::now();
    TU_RT(cudaStreamSynchronize(t->stream));
    const auto t4 = clk::now();
    CUpti_RangeProfiler_DecodeData_Params dd = {CUpti_RangeProfiler_DecodeData_Params_STRUCT_SIZE};
    dd.pRangeProfilerObject = t->rp;
    TU_CUPTI(cuptiRangeProfilerDecodeData(&dd));
    const auto t5 = clk::now();
    CUpti_Profiler_Host_EvaluateToGpuValues_Params ev = {sizeof(CUpti_Profiler_Host_EvaluateToGpuValues_Params)};
    ev.pHostObject = hc->host;
    ev.pCounterDataImage = data.data();
    ev.counterDataImageSize = data.size();
    ev.rangeIndex = 0;
    ev.ppMetricNames = hc->name_ptrs.data();
    ev.numMetrics = (size_t)n;
    ev.pMetricValues = values;
    TU_CUPTI(cuptiProfilerHostEvaluateToGpuValues(&ev));
    const auto t6 = clk::now();
    t->prof_us[0] += us(t1, t2);
    t->prof_us[1] += us(t2, t3);
    t->prof_us[2] += us(t3, t4);
    t->prof_us[3] += us(t4, t5);
    t->prof_us[4] += us(t5, t6);
    t->prof_us[5] += 1;
    t->prof_us[6] += used;
    if (passes) *passes = used;
    return CT_TUNE_OK;
}

int ct_tuner_profile_batch(ct_tuner* t, int32_t k, const int32_t* variants,
                           const ct_launch* launches, const char* const* metrics, int32_t n,
                           double* values, int32_t* passes) {
    int rc = activate(t); if (rc) return rc;
    if (k < 1 || !variants || !launches || !metrics || n < 1 || !values)
        return fail(CT_TUNE_ERR_VALUE, "bad batch profile arguments");
    std::vector<Variant*> vs((size_t)k);
    for (int i = 0; i < k; ++i) { rc = get_variant(t, variants[i], &vs[i]); if (rc) return rc; }
    rc = cupti_init(t); if (rc) return rc;
    HostConfig* hc = nullptr;
    rc = host_config_cached(t, metrics, n, &hc); if (rc) return rc;
    rc = rp_shape(t, hc, k); if (rc) return rc;
    // a counter-data image for k ranges (per call: k varies)
    CUpti_RangeProfiler_GetCounterDataSize_Params cs = {CUpti_RangeProfiler_GetCounterDataSize_Params_STRUCT_SIZE};
    cs.pRangeProfilerObject = t->rp;
    cs.pMetricNames = hc->name_ptrs.data();
    cs.numMetrics = (size_t)n;
    cs.maxNumOfRanges = (size_t)k;
    cs.maxNumRangeTreeNodes = (size_t)k;
    TU_CUPTI(cuptiRangeProfilerGetCounterDataSize(&cs));
    std::vector<uint8_t> data(cs.counterDataSize, 0);
    CUpti_RangeProfiler_CounterDataImage_Initialize_Params ci = {CUpti_RangeProfiler_CounterDataImage_Initialize_Params_STRUCT_SIZE};
    ci.pRangeProfilerObject = t->rp;
    ci.counterDataSize = data.size();
    ci.pCounterData = data.data();
    TU_CUPTI(cuptiRangeProfilerCounterDataImageInitialize(&ci));
    CUpti_RangeProfiler_SetConfig_Params sc = {CUpti_RangeProfiler_SetConfig_Params_STRUCT_SIZE};
    sc.pRangeProfilerObject = t->rp;
    sc.configSize = hc->image.size();
    sc.pConfig = hc->image.data();
    sc.counterDataImageSize = data.size();
    sc.pCounterDataImage = data.data();
    sc.range = CUPTI_UserRange;
    sc.replayMode = CUPTI_UserReplay;
    sc.maxRangesPerPass = (size_t)k;
    sc.numNestingLevels = 1;
    sc.minNestingLevel = 1;
    sc.passIndex = 0;
    sc.targetNestingLevel = 1;
    TU_CUPTI(cuptiRangeProfilerSetConfig(&sc));
    std::vector<std::string> names((size_t)k);
    for (int i = 0; i < k; ++i) names[i] = "r" + std::to_string(i);
    int used = 0;
    for (;;) {
        CUpti_RangeProfiler_Start_Params st = {CUpti_RangeProfiler_Start_Params_STRUCT_SIZE};
        st.pRangeProfilerObject = t->rp;
        TU_CUPTI(cuptiRangeProfilerStart(&st));
        for (int i = 0; i < k && rc == 0; ++i) {
            CUpti_RangeProfiler_PushRange_Params pr = {CUpti_RangeProfiler_PushRange_Params_STRUCT_SIZE};
            pr.pRangeProfilerObject = t->rp;
            pr.pRangeName = names[i].c_str();
            TU_CUPTI(cuptiRangeProfilerPushRange(&pr));
            rc = launch_once(t, vs[i], &launches[i]);
            CUpti_RangeProfiler_PopRange_Params po = {CUpti_RangeProfiler_PopRange_Params_STRUCT_SIZE};
            po.pRangeProfilerObject = t->rp;
            TU_CUPTI(cuptiRangeProfilerPopRange(&po));
        }
        CUpti_RangeProfiler_Stop_Params sp = {CUpti_RangeProfiler_Stop_Params_STRUCT_SIZE};
        sp.pRangeProfilerObject = t->rp;
        TU_CUPTI(cuptiRangeProfilerStop(&sp));
        if (rc) return rc;
        ++used;
        if (sp.isAllPassSubmitted) break;
        if (used > 64) return fail(CT_TUNE_ERR_PROFILER, "range profiler did not finish its passes");
    }
    TU_RT(cudaStreamSynchronize(t->stream));
    CUpti_RangeProfiler_DecodeData_Params dd = {CUpti_RangeProfiler_DecodeData_Params_STRUCT_SIZE};
    dd.pRangeProfilerObject = t->rp;
    TU_CUPTI(cuptiRangeProfilerDecodeData(&dd));
    for (int i = 0; i < k; ++i) {
        CUpti_Profiler_Host_EvaluateToGpuValues_Params ev = {sizeof(CUpti_Profiler_Host_EvaluateToGpuValues_Params)};
        ev.pHostObject = hc->host;
        ev.pCounterDataImage = data.data();
        ev.counterDataImageSize = data.size();
        ev.rangeIndex = (size_t)i;
        ev.ppMetricNames = hc->name_ptrs.data();
        ev.numMetrics = (size_t)n;
        ev.pMetricValues = values + (size_t)i * n;
        TU_CUPTI(cuptiProfilerHostEvaluateToGpuValues(&ev));
    }
    if (passes) *passes = used;
    return CT_TUNE_OK;
}

int ct_tuner_tensor_map_2d(ct_tuner* t, uint64_t dev_ptr, uint64_t dim0, uint64_t dim1,
                           uint64_t row_stride_bytes, uint32_t box0, uint32_t box1,
                           void* out128) {
    int rc = activate(t); if (rc) return rc;
    if (!dev_ptr || !out128 || !dim0 || !dim1 || !box0 || !box1 || (box0 * 4) % 16 ||
        box0 > 256 || box1 > 256 || row_stride_bytes % 16)
        return fail(CT_TUNE_ERR_VALUE, "bad tensor map geometry");
    CUtensorMap map;
    const cuuint64_t dims[2] = {dim0, dim1};
    const cuuint64_t strides[1] = {row_stride_bytes};
    const cuuint32_t box[2] = {box0, box1};
    const cuuint32_t estr[2] = {1, 1};
    TU_CU(D.cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                                   reinterpret_cast<void*>(dev_ptr), dims, strides, box, estr,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
    std::memcpy(out128, &map, sizeof(map));
    return CT_TUNE_OK;
}

int ct_tuner_profile_timing(ct_tuner* t, double* out8, int32_t reset) {
    if (!t || !out8) return fail(CT_TUNE_ERR_VALUE, "null argument");
    for (int i = 0; i < 8; ++i) out8[i] = t->prof_us[i];
    if (reset)
        for (int i = 0; i < 8; ++i) t->prof_us[i] = 0;
    return CT_TUNE_OK;
}

}  // extern "C"
