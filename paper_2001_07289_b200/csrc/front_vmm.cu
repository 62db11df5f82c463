// Coarse front memory with aliased update blocks (CUDA virtual memory management).
//
// A multifrontal front of node v is one column-major (ld x f) block: the s separator columns
// (the factor panel, read by every coarse solve) and the b = f - s update columns, whose
// lower triangle only lives from v's first task (extend-add of its children, trailing
// updates) to the extend-add of v into its parent. Kept resident, the update blocks dominate
// the coarse memory at cfg5 (Σ b² = 112 GB of Σ f² = 158 GB). Here the update columns of
// every large front are mapped onto pages of a shared pool such that two blocks share a page
// only if their lifetimes are ordered by the dataflow dependencies:
//   U_u and U_v (u in the subtree of v) may alias iff parent(u) is a proper descendant of v
//   (u's consumer finishes before any task of v starts). Unrelated subtrees never alias.
// Page assignment (bottom-up): children of v get consecutive sub-pools, U_v takes the first
// free pages of v's pool that no child's U occupies; need(v) = max(Σ need(c), Σ u(c) + u(v)).
// The extend-add zeroes the entries it consumes, so the pool is all-zero again when a block
// is reused (upper-triangle / padding entries are never written). The virtual range stays
// contiguous per front, so the factorization and solve kernels address fronts unchanged.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <exception>
#include <thread>

#include "bddc_internal.cuh"

namespace bddc {

namespace {

struct Drv {
  decltype(&cuMemCreate) create = nullptr;
  decltype(&cuMemRelease) release = nullptr;
  decltype(&cuMemAddressReserve) reserve = nullptr;
  decltype(&cuMemAddressFree) vfree = nullptr;
  decltype(&cuMemMap) map = nullptr;
  decltype(&cuMemUnmap) unmap = nullptr;
  decltype(&cuMemSetAccess) access = nullptr;
  decltype(&cuMemGetAllocationGranularity) gran = nullptr;
};

// driver entry points through the runtime (no link-time dependency on libcuda)
const Drv& drv() {
  static Drv d;
  static bool done = false;
  if (!done) {
    auto get = [](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult q;
      BDDC_CUDA(cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q));
      if (q != cudaDriverEntryPointSuccess || !*fn) throw CudaError(std::string("driver entry point ") + name);
    };
    get("cuMemCreate", (void**)&d.create);
    get("cuMemRelease", (void**)&d.release);
    get("cuMemAddressReserve", (void**)&d.reserve);
    get("cuMemAddressFree", (void**)&d.vfree);
    get("cuMemMap", (void**)&d.map);
    get("cuMemUnmap", (void**)&d.unmap);
    get("cuMemSetAccess", (void**)&d.access);
    get("cuMemGetAllocationGranularity", (void**)&d.gran);
    done = true;
  }
  return d;
}

void cu_check(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS) throw CudaError(std::string("front memory: ") + what + " failed (CUresult " + std::to_string((int)r) + ")");
}

}  // namespace

struct FrontVmm {
  CUdeviceptr va = 0, pview = 0, uview = 0;  // fronts, persistent view, pool view
  size_t va_bytes = 0, p_bytes = 0, u_bytes = 0;
  std::vector<CUmemGenericAllocationHandle> handles;  // each mapped whole (cuMemMap offset 0)
  std::vector<std::pair<size_t, size_t>> maps;  // (va, bytes) mapped ranges to unmap
  // the driver calls that back the reserved ranges (create / map / access: seconds at cfg5)
  // run on this thread while the setup builds its schedules; front_vmm_wait joins it
  std::thread worker;
  std::exception_ptr error;
  // every extend-add zeroes the update entries it consumes, so after a factorization that ran
  // to completion the pool is all zero again and the next setup need not clear it
  bool pool_clean = false;
};

void front_pool_mark_clean(Ctx& c) {
  if (c.vmm) c.vmm->pool_clean = true;
}

void front_vmm_wait(Ctx& c) {
  FrontVmm* v = c.vmm;
  if (!v || !v->worker.joinable()) return;
  v->worker.join();
  if (v->error) {
    std::exception_ptr e = v->error;
    v->error = nullptr;
    std::rethrow_exception(e);
  }
}

void front_vmm_release(Ctx& c) {
  FrontVmm* v = c.vmm;
  if (!v) return;
  if (v->worker.joinable()) v->worker.join();
  const Drv& d = drv();
  cudaDeviceSynchronize();
  for (auto& m : v->maps) d.unmap((CUdeviceptr)m.first, m.second);
  if (v->va) d.vfree(v->va, v->va_bytes);
  if (v->pview) d.vfree(v->pview, v->p_bytes);
  if (v->uview) d.vfree(v->uview, v->u_bytes);
  for (auto h : v->handles) d.release(h);
  delete v;
  c.vmm = nullptr;
}

// 0: off, 1: on, -1: automatic (when the resident fronts would take > 25% of free memory)
static int alias_mode() {
  const char* e = getenv("BDDC_FRONT_ALIAS");
  return e ? atoi(e) : -1;
}

bool front_alias_layout(Ctx& c) {
  FrontPlan& fp = c.fp;
  const int N = fp.nnodes;
  const int mode = alias_mode();
  if (mode == 0) return false;
  if (mode < 0) {
    size_t free_b = 0, total_b = 0;
    BDDC_CUDA(cudaMemGetInfo(&free_b, &total_b));
    if ((double)fp.front_pool * 8.0 <= 0.25 * (double)free_b) return false;
  }
  const Drv& d = drv();
  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = c.device;
  size_t g = 0;
  cu_check(d.gran(&g, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "granularity");
  // Page size: every mapping costs a cuMemMap + its share of cuMemSetAccess (~0.2 ms each,
  // serialized in the driver: tools/vmm_probe.cu), while larger pages waste more of each
  // aliased block's last page (cfg5: 75.5 GB resident at 2 MB, 86 GB at 8 MB, and the local
  // setup then runs in 4x more memory-bound chunks). Default 2 MB (BDDC_FRONT_PAGE_MB
  // overrides); the mapping count is cut by merging pool runs below instead.
  size_t free_b = 0, total_b = 0;
  BDDC_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const char* pe = getenv("BDDC_FRONT_PAGE_MB");
  const char* te = getenv("BDDC_FRONT_ALIAS_MIN_MB");  // aliasing threshold (default: one page)
  std::vector<long long> cands;
  if (pe) cands.push_back((long long)atoi(pe) << 20);
  else cands.push_back(2LL << 20);
  long long PG = 0, vpages = 0, upages = 0;
  std::vector<long long> u, upage, need, choff, front_off;
  using Runs = std::vector<std::pair<long long, long long>>;  // (first page, count)
  std::vector<Runs> urun;
  for (size_t ci = 0; ci < cands.size(); ++ci) {
    PG = std::max<long long>(cands[ci], (long long)g) / 8;  // doubles per page
    const double thr = te ? atof(te) * 1e6 : 8.0 * (double)PG;
    // (1) virtual layout: aliased fronts start so that their update columns are page aligned
    u.assign(N, 0);
    upage.assign(N, -1);
    front_off.assign(N, 0);
    long long off = 0;
    for (int i = 0; i < N; ++i) {
      const long long s = fp.sep_size[i], b = fp.bnd_size[i], f = s + b, ld = fp.ld[i];
      if (b > 0 && 8.0 * (double)(ld * b) >= thr) {
        const long long fo = round_up(off + s * ld, PG) - s * ld;
        const long long ue = round_up(fo + f * ld, PG);
        front_off[i] = fo;
        upage[i] = (fo + s * ld) / PG;
        u[i] = ue / PG - upage[i];
        off = ue;
      } else {
        front_off[i] = off;
        off = round_up(off + ld * f, 2);
      }
    }
    vpages = std::max<long long>(1, (off + PG - 1) / PG);
    // (2) pool pages, bottom-up (nodes are in postorder): runs relative to the node's sub-pool
    urun.assign(N, Runs());
    need.assign(N, 0);
    choff.assign(N, 0);
    for (int v = 0; v < N; ++v) {
      long long sum_need = 0, sum_u = u[v];
      Runs occ;
      for (int k = fp.child_ptr[v]; k < fp.child_ptr[v + 1]; ++k) {
        const int ch = fp.child_list[k];
        choff[ch] = sum_need;
        for (auto& r : urun[ch]) occ.push_back({r.first + sum_need, r.second});
        sum_need += need[ch];
        sum_u += u[ch];
      }
      need[v] = std::max(sum_need, sum_u);
      std::sort(occ.begin(), occ.end());
      long long want = u[v], p = 0;
      for (size_t k = 0; k <= occ.size() && want > 0; ++k) {
        const long long gap_end = k < occ.size() ? occ[k].first : need[v];
        if (gap_end > p) {
          const long long take = std::min(want, gap_end - p);
          urun[v].push_back({p, take});
          want -= take;
        }
        if (k < occ.size()) p = std::max(p, occ[k].first + occ[k].second);
      }
      if (want > 0) throw CudaError("front alias planner: pool too small");
    }
    upages = 0;
    for (int v = 0; v < N; ++v)
      if (fp.parent[v] < 0) upages += need[v];
    long long na = 0;
    for (int i = 0; i < N; ++i) na += u[i];
    const double resident = 8.0 * (double)PG * (double)(vpages - na + std::max(upages, 1LL));
    if (resident <= 0.5 * (double)free_b || ci + 1 == cands.size()) break;
  }
  for (int i = 0; i < N; ++i) fp.front_off[i] = front_off[i];
  // absolute pool positions, top-down (parents after children in index order)
  std::vector<long long> base(N, 0);
  upages = 0;
  for (int v = N - 1; v >= 0; --v) {
    if (fp.parent[v] < 0) {
      base[v] = upages;
      upages += need[v];
    } else {
      base[v] = base[fp.parent[v]] + choff[v];
    }
  }
  upages = std::max(upages, 1LL);
  HostTimer ht;
  ht.mark("alias: page plan");
  // (3) physical memory: persistent pages (everything outside aliased update columns) + pool
  std::vector<char> aliased(vpages, 0);
  long long na = 0;
  for (int i = 0; i < N; ++i)
    for (long long k = 0; k < u[i]; ++k) aliased[upage[i] + k] = 1, ++na;
  const long long ppages = std::max(1LL, vpages - na);
  const size_t PB = (size_t)PG * 8;
  FrontVmm* vm = new FrontVmm;
  c.vmm = vm;
  vm->va_bytes = (size_t)vpages * PB;
  vm->p_bytes = (size_t)ppages * PB;
  vm->u_bytes = (size_t)upages * PB;
  cu_check(d.reserve(&vm->va, vm->va_bytes, PB, 0, 0), "reserve");
  cu_check(d.reserve(&vm->pview, vm->p_bytes, PB, 0, 0), "reserve");
  cu_check(d.reserve(&vm->uview, vm->u_bytes, PB, 0, 0), "reserve");
  fp.front_pool = vpages * PG;
  fp.alias = true;
  fp.alias_resident_bytes = (long long)(vm->p_bytes + vm->u_bytes);
  fp.ualias.assign(N, 0);
  for (int i = 0; i < N; ++i) fp.ualias[i] = u[i] > 0;
  fp.d.fronts = (double*)vm->va;
  const int dev = c.device;
  long long nal = 0;
  for (int i = 0; i < N; ++i) nal += u[i] > 0;
  vm->worker = std::thread([vm, d, prop, PB, PG, vpages, ppages, upages, N, nal, dev, aliased = std::move(aliased),
                            upage = std::move(upage), urun = std::move(urun), base = std::move(base)]() {
    try {
      BDDC_CUDA(cudaSetDevice(dev));
      HostTimer ht;
      auto create = [&](size_t bytes) {
        CUmemGenericAllocationHandle h;
        cu_check(d.create(&h, bytes, &prop, 0), "cuMemCreate");
        vm->handles.push_back(h);
        return h;
      };
      auto map = [&](CUdeviceptr va, size_t bytes, CUmemGenericAllocationHandle h) {
        cu_check(d.map(va, bytes, 0, h, 0), "cuMemMap");
        vm->maps.push_back({(size_t)va, bytes});
      };
      // persistent runs: one allocation each, mapped in place and into the persistent view
      long long pnext = 0;
      for (long long p = 0; p < vpages;) {
        long long q = p;
        while (q < vpages && aliased[q] == aliased[p]) ++q;
        if (!aliased[p]) {
          const size_t bytes = (size_t)(q - p) * PB;
          const CUmemGenericAllocationHandle h = create(bytes);
          map(vm->va + (size_t)p * PB, bytes, h);
          map(vm->pview + (size_t)pnext * PB, bytes, h);
          pnext += q - p;
        }
        p = q;
      }
      ht.mark("alias: persistent runs");
      // pool: consecutive pages used by exactly the same update blocks at consecutive virtual
      // pages form one allocation (every mapping costs a driver call: ~3.5x fewer at cfg5),
      // mapped into the pool view and under each of those update blocks
      std::vector<std::vector<std::pair<int, long long>>> users(upages);  // (front, virtual page)
      for (int i = 0; i < N; ++i) {
        long long vp = upage[i];
        for (auto& r : urun[i])
          for (long long k = 0; k < r.second; ++k, ++vp) users[base[i] + r.first + k].push_back({i, vp});
      }
      long long nruns = 0, nmaps = 0;
      for (long long p0 = 0; p0 < upages;) {
        long long p1 = p0 + 1;
        auto same = [&](long long q) {
          if (users[q].size() != users[p0].size()) return false;
          for (size_t j = 0; j < users[q].size(); ++j)
            if (users[q][j].first != users[p0][j].first || users[q][j].second != users[p0][j].second + (q - p0))
              return false;
          return true;
        };
        while (p1 < upages && same(p1)) ++p1;
        const size_t bytes = (size_t)(p1 - p0) * PB;
        const CUmemGenericAllocationHandle h = create(bytes);
        map(vm->uview + (size_t)p0 * PB, bytes, h);
        for (auto& us : users[p0]) map(vm->va + (size_t)us.second * PB, bytes, h);
        ++nruns;
        nmaps += 1 + (long long)users[p0].size();
        p0 = p1;
      }
      ht.mark("alias: pool runs + update-block maps");
      if (ht.on) {
        fprintf(stderr, "bddc_setup host: alias: page %lld MB, %lld virtual / %lld persistent / %lld pool pages, "
                "%lld aliased fronts, %lld pool runs, %lld pool mappings, %zu allocations\n", PG * 8 >> 20, vpages,
                ppages, upages, nal, nruns, nmaps, vm->handles.size());
      }
      CUmemAccessDesc acc{};
      acc.location = prop.location;
      acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
      cu_check(d.access(vm->va, vm->va_bytes, &acc, 1), "cuMemSetAccess");
      cu_check(d.access(vm->pview, vm->p_bytes, &acc, 1), "cuMemSetAccess");
      cu_check(d.access(vm->uview, vm->u_bytes, &acc, 1), "cuMemSetAccess");
      ht.mark("alias: access");
    } catch (...) {
      vm->error = std::current_exception();
    }
  });
  return true;
}

// Zero every front (setup start): the persistent pages and (unless the last factorization left
// it clean) the pool, each through its own contiguous view (the aliased virtual range would
// zero shared pages many times over).
void front_memset(Ctx& c, cudaStream_t s) {
  front_vmm_wait(c);  // the fronts' physical pages are mapped
  if (!c.vmm) {
    BDDC_CUDA(cudaMemsetAsync(c.fp.d.fronts, 0, sizeof(double) * c.fp.front_pool, s));
    return;
  }
  BDDC_CUDA(cudaMemsetAsync((void*)c.vmm->pview, 0, c.vmm->p_bytes, s));
  if (!c.vmm->pool_clean) BDDC_CUDA(cudaMemsetAsync((void*)c.vmm->uview, 0, c.vmm->u_bytes, s));
  c.vmm->pool_clean = false;  // dirty until the factorization completes (front_pool_mark_clean)
}

}  // namespace bddc
