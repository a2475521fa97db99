// nvls.cu -- NVLink SHARP (NVSwitch multicast) for the delegate-mask
// OR-reduction of the peer engine (comm.py:75-98; SURVEY §8e option iii).
//
// Each rank's two per-level delegate masks (dnext by parity, d/8 bytes each)
// live in physical memory bound to one multicast object that spans every
// rank's GPU.  A rank writes its own copy through an ordinary (unicast)
// mapping; in F(L) a single `multimem.ld_reduce.or` on the multicast mapping
// returns the OR of all P copies, reduced inside the NVSwitch -- one NVLink
// read per word instead of P-1 peer reads.
//
// Ranks are threads of one process (group.py: the CUmemGenericAllocationHandle
// of the multicast object is shared by value); one-process-per-GPU jobs
// (torchrun) would need the POSIX-fd export passed between processes and keep
// the peer reads.  Opt-in with DBFS_NVLS=1.
#include <cuda.h>

#include <map>
#include <mutex>

#include "internal.h"

namespace dbfs {

// Driver entry points through the runtime (libdbfs does not link libcuda, so
// it still loads on a machine without a driver).
namespace drv {
#define DBFS_DRV_FN(name) static decltype(&::name) name = nullptr;
DBFS_DRV_FN(cuGetErrorString)
DBFS_DRV_FN(cuDeviceGet)
DBFS_DRV_FN(cuDeviceGetAttribute)
DBFS_DRV_FN(cuMulticastGetGranularity)
DBFS_DRV_FN(cuMulticastCreate)
DBFS_DRV_FN(cuMulticastAddDevice)
DBFS_DRV_FN(cuMulticastBindMem)
DBFS_DRV_FN(cuMulticastUnbind)
DBFS_DRV_FN(cuMemCreate)
DBFS_DRV_FN(cuMemRelease)
DBFS_DRV_FN(cuMemAddressReserve)
DBFS_DRV_FN(cuMemAddressFree)
DBFS_DRV_FN(cuMemMap)
DBFS_DRV_FN(cuMemUnmap)
DBFS_DRV_FN(cuMemSetAccess)
#undef DBFS_DRV_FN

static bool load() {
    static int state = 0;  // 0 untried, 1 ok, -1 missing
    if (state) return state > 0;
    bool ok = true;
    auto get = [&](const char *sym, void **fn) {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint(sym, fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !*fn) {
            cudaGetLastError();
            ok = false;
        }
    };
#define DBFS_DRV_GET(name) get(#name, reinterpret_cast<void **>(&name));
    DBFS_DRV_GET(cuGetErrorString)
    DBFS_DRV_GET(cuDeviceGet)
    DBFS_DRV_GET(cuDeviceGetAttribute)
    DBFS_DRV_GET(cuMulticastGetGranularity)
    DBFS_DRV_GET(cuMulticastCreate)
    DBFS_DRV_GET(cuMulticastAddDevice)
    DBFS_DRV_GET(cuMulticastBindMem)
    DBFS_DRV_GET(cuMulticastUnbind)
    DBFS_DRV_GET(cuMemCreate)
    DBFS_DRV_GET(cuMemRelease)
    DBFS_DRV_GET(cuMemAddressReserve)
    DBFS_DRV_GET(cuMemAddressFree)
    DBFS_DRV_GET(cuMemMap)
    DBFS_DRV_GET(cuMemUnmap)
    DBFS_DRV_GET(cuMemSetAccess)
#undef DBFS_DRV_GET
    state = ok ? 1 : -1;
    return ok;
}
}  // namespace drv

#define DBFS_CU(call)                                                                              \
    do {                                                                                           \
        CUresult _r = (call);                                                                      \
        if (_r != CUDA_SUCCESS) {                                                                  \
            const char *_s = nullptr;                                                              \
            drv::cuGetErrorString(_r, &_s);                                                             \
            throw ::dbfs::Error(DBFS_ECUDA, std::string(#call) + ": " + (_s ? _s : "?"));          \
        }                                                                                          \
    } while (0)

// The ranks of a group share one multicast object (by handle value, one
// process): it is released when its last rank lets go.
static std::mutex g_mc_mu;
static std::map<unsigned long long, int> g_mc_refs;

struct NvlsState {
    CUmemGenericAllocationHandle mc = 0, phys = 0;
    CUdeviceptr uc_va = 0, mc_va = 0;
    size_t size = 0;
};

static int agree_all(Ctx &ctx, int v) {
    DArray<uint32_t> f;
    f.alloc(1);
    uint32_t h = v ? 1u : 0u;
    DBFS_CUDA(cudaMemcpy(f.p, &h, 4, cudaMemcpyHostToDevice));
    nccl_allreduce_u32_sum(ctx, f.p, 1);
    DBFS_CUDA(cudaMemcpy(&h, f.p, 4, cudaMemcpyDeviceToHost));
    return (int)h == ctx.nranks;
}

// Collective over the group's ranks.  Returns false (nothing changed) when
// multicast is unavailable; on success masks[0..1] are this rank's unicast
// mask buffers and mc[0..1] the multicast addresses of the same words.
bool nvls_setup(Graph &g, int64_t mask_words, uint32_t **masks, const uint32_t **mc) {
    Ctx &ctx = *g.ctx;
    if (!ctx.local_group || ctx.nranks < 2) return false;
    if (!drv::load()) return false;
    CUdevice dev;
    int ok = drv::cuDeviceGet(&dev, ctx.device) == CUDA_SUCCESS;
    int mcs = 0;
    if (ok && drv::cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev) != CUDA_SUCCESS) mcs = 0;
    if (!agree_all(ctx, ok && mcs)) return false;
    auto *st = new NvlsState();
    CUmulticastObjectProp prop = {};
    prop.numDevices = (unsigned)ctx.nranks;
    prop.handleTypes = CU_MEM_HANDLE_TYPE_NONE;
    size_t gran = 0;
    DBFS_CU(drv::cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    const size_t bytes = (size_t)2 * mask_words * 4;
    st->size = (bytes + gran - 1) / gran * gran;
    prop.size = st->size;
    // rank 0 creates the object; every rank adds its device before any bind
    uint64_t hv = 0;
    if (ctx.rank == 0) {
        DBFS_CU(drv::cuMulticastCreate(&st->mc, &prop));
        hv = (uint64_t)st->mc;
    }
    {
        DArray<uint64_t> b;
        b.alloc(1);
        DBFS_CUDA(cudaMemcpy(b.p, &hv, 8, cudaMemcpyHostToDevice));
        nccl_allreduce_i64(ctx, (int64_t *)b.p, 1, 0);  // only rank 0 contributes
        DBFS_CUDA(cudaMemcpy(&hv, b.p, 8, cudaMemcpyDeviceToHost));
        st->mc = (CUmemGenericAllocationHandle)hv;
    }
    {
        std::lock_guard<std::mutex> lock(g_mc_mu);
        g_mc_refs[(unsigned long long)st->mc]++;
    }
    DBFS_CU(drv::cuMulticastAddDevice(st->mc, dev));
    nccl_barrier(ctx);
    CUmemAllocationProp pp = {};
    pp.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    pp.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    pp.location.id = ctx.device;
    DBFS_CU(drv::cuMemCreate(&st->phys, st->size, &pp, 0));
    DBFS_CU(drv::cuMulticastBindMem(st->mc, 0, st->phys, 0, st->size, 0));
    CUmemAccessDesc acc = {};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = ctx.device;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    DBFS_CU(drv::cuMemAddressReserve(&st->uc_va, st->size, gran, 0, 0));
    DBFS_CU(drv::cuMemMap(st->uc_va, st->size, 0, st->phys, 0));
    DBFS_CU(drv::cuMemSetAccess(st->uc_va, st->size, &acc, 1));
    DBFS_CU(drv::cuMemAddressReserve(&st->mc_va, st->size, gran, 0, 0));
    DBFS_CU(drv::cuMemMap(st->mc_va, st->size, 0, st->mc, 0));
    DBFS_CU(drv::cuMemSetAccess(st->mc_va, st->size, &acc, 1));
    DBFS_CUDA(cudaMemset((void *)st->uc_va, 0, st->size));
    DBFS_CUDA(cudaDeviceSynchronize());
    nccl_barrier(ctx);
    masks[0] = reinterpret_cast<uint32_t *>(st->uc_va);
    masks[1] = masks[0] + mask_words;
    mc[0] = reinterpret_cast<const uint32_t *>(st->mc_va);
    mc[1] = mc[0] + mask_words;
    g.nvls = st;
    return true;
}

void nvls_release(Graph &g) {
    auto *st = static_cast<NvlsState *>(g.nvls);
    if (!st) return;
    cudaDeviceSynchronize();
    if (st->mc_va) {
        drv::cuMemUnmap(st->mc_va, st->size);
        drv::cuMemAddressFree(st->mc_va, st->size);
    }
    if (st->uc_va) {
        drv::cuMemUnmap(st->uc_va, st->size);
        drv::cuMemAddressFree(st->uc_va, st->size);
    }
    CUdevice dev;
    if (drv::cuDeviceGet(&dev, g.ctx->device) == CUDA_SUCCESS && st->mc) {
        drv::cuMulticastUnbind(st->mc, dev, 0, st->size);
    }
    if (st->phys) drv::cuMemRelease(st->phys);
    if (st->mc) {
        std::lock_guard<std::mutex> lock(g_mc_mu);
        if (--g_mc_refs[(unsigned long long)st->mc] == 0) {
            g_mc_refs.erase((unsigned long long)st->mc);
            drv::cuMemRelease(st->mc);
        }
    }
    delete st;
    g.nvls = nullptr;
}

}  // namespace dbfs
