// dgmg_b200.cu - C ABI (include/dgmg_b200.h) over the sm_100a kernels.
//
// Host runtime responsibilities (native, C++):
//  - level objects: device tables (one allocation), window geometry;
//  - colour lists built in closed form: red-black cells (mesh.py:350-357),
//    structured patch colours (mesh.py:360-375) in ascending colour order,
//    patch ids ascending inside a colour, and per patch colour the cells the
//    colour covers (the restricted MVS residual, SURVEY 8(d) kappa);
//  - the smoothing-step launch sequences of LevelSmoother (smoothers.py:
//    131-166), captured once into CUDA graphs and replayed.
#include "../../include/dgmg_b200.h"
#include "launch.h"
#ifdef DGB_EXPERIMENTAL
#include "flow.cuh"
#endif

#include <cstdlib>

#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <string>
#include <tuple>
#include <vector>

namespace dgb {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}


__global__ void gather_map_kernel(MapParams p) {
  const int64_t per = (p.d == 3) ? (int64_t)p.m * p.m * p.m : (p.d == 2 ? (int64_t)p.m * p.m : p.m);
  const int64_t total = p.count * per;
  const int NEc = (p.d == 3) ? p.n * p.n * p.n : (p.d == 2 ? p.n * p.n : p.n);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = t / per;
    const int e = (int)(t % per);
    int rem = p.list[k];
    int c[3] = {0, 0, 0}, q[3] = {e % p.m, (e / p.m) % p.m, e / (p.m * p.m)};
    int off = 0, mul = 1;
    for (int s = 0; s < p.d; ++s) {
      const int span = p.geo.nc[s] - 1;
      const int v = 1 + rem % span;
      rem /= span;
      c[s] = v - 1 + q[s] / p.n;
      off += (q[s] % p.n) * mul;
      mul *= p.n;
    }
    int64_t cell;
    if (p.d == 1) cell = c[0] - p.geo.zb;
    else if (p.d == 2) cell = c[0] + (int64_t)p.geo.nc[0] * (c[1] - p.geo.zb);
    else cell = c[0] + (int64_t)p.geo.nc[0] * (c[1] + (int64_t)p.geo.nc[1] * (c[2] - p.geo.zb));
    p.out[t] = cell * NEc + off;
  }
}

// ---------------------------------------------------------------------------
// template dispatch
// ---------------------------------------------------------------------------

}  // namespace dgb

using namespace dgb;

struct DevList {
  int32_t* ptr = nullptr;
  int64_t count = 0;
};

struct GraphKey {
  int kind;
  double omega;
  int reverse;
  const void* x;
  const void* b;
  const void* r;
  uint64_t switches;  // switch_signature() at capture: a changed DGB_* variable re-captures
  bool operator<(const GraphKey& o) const {
    return std::tie(kind, omega, reverse, x, b, r, switches) <
           std::tie(o.kind, o.omega, o.reverse, o.x, o.b, o.r, o.switches);
  }
};

struct dg_level {
  dg_level_desc_t desc;
  int d = 0, n = 0, m = 0;
  int64_t layer_cells = 0, ncells_local = 0, ndofs = 0, cell_dofs = 0;
  Geo geo;
  double* dtab = nullptr;
  const double *mass = nullptr, *adiag = nullptr, *bg = nullptr;
  const double *cz = nullptr, *czt = nullptr, *cinv = nullptr;
  const double *pz = nullptr, *pzt = nullptr, *pinv = nullptr;
  const double *ceod = nullptr, *peod = nullptr;  // device even/odd tables (tensor-core solves)
  int* wcount = nullptr;  // work counter of the persistent solve kernel (fdm2p.cuh)
  double* big_scratch = nullptr;  // per-CTA patch tensors of the generic solve (fdmg.cuh)
  int big_slots = 0;
  double alpha = 0, beta = 0, betap = 0;
  bool has_patch = false;
  std::vector<double> hcz, hczt, hpz, hpzt;  // host copies for the kernel parameter space
  std::vector<double> hmass, hadiag, hbg, hceo, hpeo, hreo;  // *_eo empty = dense path
  HostRes hres() const {
    return HostRes{hmass.data(), hadiag.data(), hbg.data(), hreo.empty() ? nullptr : hreo.data()};
  }
  const double* ceo() const { return hceo.empty() ? nullptr : hceo.data(); }
  const double* peo() const { return hpeo.empty() ? nullptr : hpeo.data(); }
  std::vector<DevList> rb;          // red-black owned cells (MCS), local ids
  std::vector<DevList> rb_pk;       // same, packed global coordinates
  std::vector<DevList> pcol;        // patch colours (AVS / MVS), global patch ids
  std::vector<DevList> pcol_pk;     // same, packed vertex coordinates
  std::vector<DevList> pcol_cells;  // cells covered by a patch colour (MVS), local ids
  std::vector<DevList> pcol_cells_pk;
  // per colour of pcol_pk: voff[v] = entries with last vertex coordinate < v
  // (the lists are in patch-id order, so a v_last range is a sub-list)
  std::vector<std::vector<int64_t>> pcol_voff;
  std::vector<DevList> clus_pk;     // AVS clusters per cluster colour, packed base vertices
  DevList pall_pk;                  // all patches (colour order), packed, one-launch AVS
  std::vector<DevList> pwin_pk;     // AVS launch order: (z-window, parity class), packed
  int pall_vlo = 0;                 // first v_last of pall_pk (spatial order)
  int64_t layer_patches = 0;        // patches per v_last value
  cudaStream_t side = nullptr;      // low-priority stream of the overlapped AVS residual
  std::vector<cudaEvent_t> ev;      // residual-chunk completion events
  int avs_win = 0;                  // z-window of pwin_pk in patch vertices (0 = whole level)
  FlowDev flow;                     // dataflow AVS step (flow.cuh)
  bool flow_ok = false;
  cudaStream_t cap = nullptr;       // capture stream
  std::map<GraphKey, cudaGraphExec_t> graphs;
  int64_t last_launches = 0;
};

static int upload_list(const std::vector<int32_t>& h, DevList* out) {
  out->count = (int64_t)h.size();
  if (h.empty()) return DG_OK;
  DG_CUDA(cudaMalloc(&out->ptr, h.size() * sizeof(int32_t)));
  DG_CUDA(cudaMemcpy(out->ptr, h.data(), h.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  return DG_OK;
}

static void free_level(dg_level* L) {
  if (!L) return;
  for (auto& kv : L->graphs) cudaGraphExecDestroy(kv.second);
  for (auto* v : {&L->rb, &L->rb_pk, &L->pcol, &L->pcol_pk, &L->pcol_cells, &L->pcol_cells_pk,
                  &L->clus_pk, &L->pwin_pk})
    for (auto& l : *v) cudaFree(l.ptr);
  cudaFree(L->pall_pk.ptr);
  cudaFree(L->dtab);
  cudaFree(L->wcount);
  cudaFree(L->big_scratch);
  cudaFree(L->flow.tasks);
  cudaFree(L->flow.succ);
  cudaFree(L->flow.plist);
  cudaFree(L->flow.state);
  cudaFree(L->flow.state_init);
  if (L->cap) cudaStreamDestroy(L->cap);
  if (L->side) cudaStreamDestroy(L->side);
  for (auto e : L->ev) cudaEventDestroy(e);
  delete L;
}

static ResArgs res_params(const dg_level* L, const double* x, const double* b, double* r) {
  ResArgs p;
  p.x = x;
  p.b = b;
  p.r = r;
  p.alpha = L->alpha;
  p.beta = L->beta;
  p.betap = L->betap;
  p.oned.adiag = L->adiag;
  p.oned.bg = L->bg;
  p.geo = L->geo;
  return p;
}

static FdmArgs fdm_params(const dg_level* L, bool patch, const double* r, double* x,
                          double omega) {
  FdmArgs p;
  p.r = r;
  p.x = x;
  p.invsum = patch ? L->pinv : L->cinv;
  p.zd = patch ? L->pz : L->cz;
  p.ztd = patch ? L->pzt : L->czt;
  p.eod = patch ? L->peod : L->ceod;
  p.counter = L->wcount;
  if (patch) {
    p.big_scratch = L->big_scratch;
    p.big_slots = L->big_slots;
  }
  p.omega = omega;
  p.geo = L->geo;
  return p;
}

static int check_align(const dg_level* L, const void* a, const void* b, const void* c) {
  if (L->n % 2) return DG_OK;  // odd n: scalar row access
  for (const void* p : {a, b, c})
    if (p && (reinterpret_cast<uintptr_t>(p) & 15))
      return fail(DG_EINVAL, "vectors must be 16-byte aligned (even n uses 16-byte row access)");
  return DG_OK;
}

static int check_layers(const dg_level* L, int z0, int z1) {
  const int lo = L->desc.z_begin, hi = L->desc.z_begin + L->desc.z_count;
  const int last = L->desc.ncells[L->d - 1];
  if (z0 < lo || z1 > hi || z0 > z1)
    return fail(DG_EINVAL, "layer range outside the stored window");
  // neighbours of computed layers must be stored (or be the physical boundary)
  if ((z0 > 0 && z0 - 1 < lo && z0 < z1) || (z1 < last && z1 >= hi && z0 < z1))
    return fail(DG_EINVAL, "residual layers need a stored neighbour layer on each side");
  return DG_OK;
}


// ---------------------------------------------------------------------------
// dataflow task graph of the AVS step (flow.cuh): z-blocks of `W` vertex
// layers, colour skew `skew` between consecutive blocks.
// ---------------------------------------------------------------------------

#ifdef DGB_EXPERIMENTAL
static int build_flow(dg_level* L) {
  int gp = 0, gr = 0;
  if (!L->has_patch || !flow_shape(L->d, L->n, &gp, &gr)) return DG_OK;
  const int d = L->d;
  const int* nc = L->desc.ncells;
  for (int t = 0; t < d; ++t)
    if (nc[t] < 2) return DG_OK;
  const int W = std::max(1, env_int("DGB_FLOW_W", 2));
  const int skew = std::max(0, env_int("DGB_FLOW_SKEW", 4));
  const int zb = L->desc.z_begin;
  const int vlo = std::max(1, L->desc.pv_begin), vhi = std::min(nc[d - 1] - 1, L->desc.pv_end);
  struct HT {
    int type, colour, blk, lo, hi;
    int64_t start, count;
    double key;
    std::vector<int> deps;
  };
  std::vector<HT> ptasks;
  std::vector<int32_t> plist;
  const int ncol = 1 << (d + 1);
  int64_t layer_patches = 1;
  for (int t = 0; t < d - 1; ++t) layer_patches *= (nc[t] - 1);
  // blocks aligned to global vertex layers 1 + W*k so that every window (slab)
  // orders the colour updates of a DoF exactly as the single-GPU step does
  for (int k0 = (vlo - 1) / W, blk = 0; 1 + k0 * W <= vhi; ++k0, ++blk) {
    const int v0 = std::max(vlo, 1 + k0 * W);
    const int v1 = std::min(vhi, k0 * W + W);
    std::vector<std::vector<int32_t>> pc(ncol);
    std::vector<int> lo(ncol, 1 << 30), hi(ncol, -1);
    for (int64_t id = (int64_t)(v0 - 1) * layer_patches; id < (int64_t)v1 * layer_patches; ++id) {
      int64_t rem = id;
      int v[3] = {1, 1, 1}, parq = 0, half = 0;
      for (int t = 0; t < d; ++t) {
        v[t] = 1 + (int)(rem % (nc[t] - 1));
        rem /= (nc[t] - 1);
        parq += (v[t] & 1) << t;
        half += v[t] / 2;
      }
      const int col = parq * 2 + (half & 1);
      pc[col].push_back(pack_d(d, v[0], v[1], d == 3 ? v[2] : 0));
      lo[col] = std::min(lo[col], v[d - 1] - 1);
      hi[col] = std::max(hi[col], v[d - 1]);
    }
    for (int c = 0; c < ncol; ++c) {
      if (pc[c].empty()) continue;
      HT t{1, c, blk, lo[c], hi[c], (int64_t)plist.size(), (int64_t)pc[c].size(),
           (double)c + (double)skew * blk, {}};
      plist.insert(plist.end(), pc[c].begin(), pc[c].end());
      ptasks.push_back(t);
    }
  }
  std::stable_sort(ptasks.begin(), ptasks.end(), [](const HT& a, const HT& b) {
    return a.key < b.key || (a.key == b.key && a.blk < b.blk);
  });
  // residual layers, each inserted right before the first patch task that
  // reads its r or writes the x it reads
  std::vector<std::vector<HT>> before(ptasks.size() + 1);
  for (int z = L->desc.res_begin; z < L->desc.res_end; ++z) {
    size_t pos = ptasks.size();
    for (size_t i = 0; i < ptasks.size(); ++i)
      if (ptasks[i].hi >= z - 1 && ptasks[i].lo <= z + 1) { pos = i; break; }
    HT r{0, -1, -1, z - 1, z + 1, (int64_t)(z - zb) * L->layer_cells, L->layer_cells, 0.0, {}};
    if (pos == ptasks.size()) before[0].push_back(r);
    else before[pos].push_back(r);
  }
  std::vector<HT> seq;
  for (size_t i = 0; i <= ptasks.size(); ++i) {
    for (auto& r : before[i]) seq.push_back(r);
    if (i < ptasks.size()) seq.push_back(ptasks[i]);
  }
  const int nt = (int)seq.size();
  // locality edges: block b starts only when block b-1 has finished colour `lag`
  const int lag = std::max(0, env_int("DGB_FLOW_LAG", 7));
  std::vector<std::vector<int>> extra(nt);
  {
    std::map<std::pair<int, int>, int> pos;  // (blk, colour) -> sequence index
    for (int j = 0; j < nt; ++j)
      if (seq[j].type == 1) pos[{seq[j].blk, seq[j].colour}] = j;
    for (int j = 0; j < nt; ++j) {
      if (seq[j].type != 1 || seq[j].blk == 0) continue;
      // first colour of the block (smallest colour present)
      bool first = true;
      for (int c = 0; c < seq[j].colour; ++c)
        if (pos.count({seq[j].blk, c})) first = false;
      if (!first) continue;
      int best = -1;  // colour <= lag of the previous block, latest present
      for (int c = 0; c <= std::min(lag, ncol - 1); ++c) {
        auto it = pos.find({seq[j].blk - 1, c});
        if (it != pos.end()) best = it->second;
      }
      if (best >= 0 && best < j) extra[j].push_back(best);
    }
  }
  // dependencies (conflicting earlier tasks), transitively reduced
  const int words = (nt + 63) / 64;
  std::vector<std::vector<uint64_t>> anc(nt, std::vector<uint64_t>(words, 0));
  auto conflict = [](const HT& a, const HT& b) {
    if (a.type == 0 && b.type == 0) return false;
    if (a.type == 1 && b.type == 1)
      return a.colour != b.colour && a.hi >= b.lo && b.hi >= a.lo;
    return a.hi >= b.lo && b.hi >= a.lo;  // R(z) vs P: x/r layer overlap
  };
  for (int j = 0; j < nt; ++j) {
    auto keep = [&](int i) {
      seq[j].deps.push_back(i);
      anc[j][i / 64] |= uint64_t(1) << (i % 64);
      for (int w = 0; w < words; ++w) anc[j][w] |= anc[i][w];
    };
    for (int i : extra[j]) keep(i);
    for (int i = j - 1; i >= 0; --i) {
      if (!conflict(seq[i], seq[j])) continue;
      if (seq[j].type == 0) return fail(DG_EINVAL, "flow: residual after a conflicting patch task");
      if (anc[j][i / 64] >> (i % 64) & 1) continue;  // implied by a kept dependency
      keep(i);
    }
  }
  // device images: tasks with successor lists (CSR), initial scheduler state
  std::vector<std::vector<int>> succ(nt);
  for (int j = 0; j < nt; ++j)
    for (int i : seq[j].deps) succ[i].push_back(j);
  std::vector<FlowTask> ht(nt);
  std::vector<int32_t> sflat;
  int64_t units = 0;
  for (int j = 0; j < nt; ++j) {
    FlowTask& t = ht[j];
    const int g = seq[j].type == 0 ? gr : gp;
    t.type = seq[j].type;
    t.units = (int)((seq[j].count + g - 1) / g);
    t.start = seq[j].start;
    t.count = seq[j].count;
    t.succ_off = (int)sflat.size();
    t.nsucc = (int)succ[j].size();
    sflat.insert(sflat.end(), succ[j].begin(), succ[j].end());
    units += t.units;
  }
  std::vector<int> state(4 + 5 * (size_t)nt, 0);
  int* pend = state.data() + 4;
  int* queue = pend + 3 * nt;
  int* valid = queue + nt;
  int q = 0;
  for (int j = 0; j < nt; ++j) {
    pend[j] = (int)seq[j].deps.size();
    if (pend[j] == 0) {
      queue[q] = j;
      valid[q] = 1;
      ++q;
    }
  }
  state[1] = q;  // tail
  FlowDev& f = L->flow;
  DG_CUDA(cudaMalloc(&f.tasks, sizeof(FlowTask) * nt));
  DG_CUDA(cudaMemcpy(f.tasks, ht.data(), sizeof(FlowTask) * nt, cudaMemcpyHostToDevice));
  DG_CUDA(cudaMalloc(&f.succ, sizeof(int32_t) * std::max<size_t>(1, sflat.size())));
  if (!sflat.empty())
    DG_CUDA(cudaMemcpy(f.succ, sflat.data(), sizeof(int32_t) * sflat.size(), cudaMemcpyHostToDevice));
  DG_CUDA(cudaMalloc(&f.plist, sizeof(int32_t) * std::max<size_t>(1, plist.size())));
  if (!plist.empty())
    DG_CUDA(cudaMemcpy(f.plist, plist.data(), sizeof(int32_t) * plist.size(), cudaMemcpyHostToDevice));
  DG_CUDA(cudaMalloc(&f.state, sizeof(int) * state.size()));
  DG_CUDA(cudaMalloc(&f.state_init, sizeof(int) * state.size()));
  DG_CUDA(cudaMemcpy(f.state_init, state.data(), sizeof(int) * state.size(), cudaMemcpyHostToDevice));
  f.ntasks = nt;
  f.units = units;
  L->flow_ok = true;
  return DG_OK;
}

#endif  // DGB_EXPERIMENTAL

extern char** environ;

uint64_t dgb::switch_signature() {
  uint64_t h = 1469598103934665603ull;
  for (char** e = environ; e && *e; ++e) {
    if (std::strncmp(*e, "DGB_", 4) != 0) continue;
    for (const char* c = *e; *c; ++c) h = (h ^ (unsigned char)*c) * 1099511628211ull;
    h = (h ^ 0xff) * 1099511628211ull;
  }
  return h;
}

extern "C" {

const char* dg_last_error(void) { return g_err.c_str(); }

int dg_version(void) { return 1; }

int dg_level_create(const dg_level_desc_t* desc, const dg_tables_t* T, dg_level_t** out) {
  if (!desc || !T || !out) return fail(DG_EINVAL, "null argument");
  *out = nullptr;
  const int d = desc->dim;
  if (d < 1 || d > 3) return fail(DG_EUNSUPPORTED, "device path supports dim 1, 2 and 3");
  const int n = desc->degree + 1;
  if (desc->degree < 1 || n > 16)
    return fail(DG_EUNSUPPORTED, "device path supports 1 <= degree <= 15");
  for (int t = 0; t < d; ++t)
    if (desc->ncells[t] < 1) return fail(DG_EINVAL, "ncells must be >= 1");
  // packed colour lists hold global coordinates in 10 (3D) / 15 (2D) bits,
  // and cell ids are 32-bit
  for (int t = 0; t < d; ++t)
    if (desc->ncells[t] > (d == 3 ? kPackMax3 : kPackMax2))
      return fail(DG_EUNSUPPORTED, d == 3 ? "device path supports at most 1024 cells per direction in 3D"
                                          : "device path supports at most 32768 cells per direction in 2D");
  {
    int64_t cells = 1;
    for (int t = 0; t < d; ++t) cells *= desc->ncells[t];
    if (cells >= (int64_t(1) << 31)) return fail(DG_EUNSUPPORTED, "more than 2^31 cells");
  }
  const int last = desc->ncells[d - 1];
  if (desc->z_begin < 0 || desc->z_count < 1 || desc->z_begin + desc->z_count > last)
    return fail(DG_EINVAL, "stored window outside the level");
  if (!T->mass || !T->adiag || !T->bg || !T->cell_z || !T->cell_zt || !T->cell_invsum)
    return fail(DG_EINVAL, "missing table");
  auto* L = new dg_level();
  L->desc = *desc;
  L->d = d;
  L->n = n;
  L->m = 2 * n;
  L->layer_cells = (d == 3) ? (int64_t)desc->ncells[0] * desc->ncells[1]
                            : (d == 2 ? desc->ncells[0] : 1);
  L->ncells_local = L->layer_cells * desc->z_count;
  L->cell_dofs = (d == 3) ? (int64_t)n * n * n : (d == 2 ? (int64_t)n * n : n);
  L->ndofs = L->ncells_local * L->cell_dofs;
  L->geo.nc[0] = desc->ncells[0];
  L->geo.nc[1] = d >= 2 ? desc->ncells[1] : 1;
  L->geo.nc[2] = d == 3 ? desc->ncells[2] : 1;
  L->geo.zb = desc->z_begin;
  L->geo.zn = desc->z_count;
  for (int t = 0; t < 3; ++t) {
    L->geo.fc[t].init((uint32_t)L->geo.nc[t]);
    L->geo.fv[t].init((uint32_t)std::max(1, L->geo.nc[t] - 1));
  }
  L->alpha = T->alpha;
  L->beta = T->beta;
  L->betap = T->betap;
  L->has_patch = T->patch_z != nullptr;
  L->hmass.assign(T->mass, T->mass + n * n);
  L->hadiag.assign(T->adiag, T->adiag + 4 * n * n);
  L->hbg.assign(T->bg, T->bg + 2 * n);
  if (T->cell_eo && n % 2 == 0) L->hceo.assign(T->cell_eo, T->cell_eo + n * n);
  if (T->res_eo && n % 2 == 0) L->hreo.assign(T->res_eo, T->res_eo + n * n);
  L->hcz.assign(T->cell_z, T->cell_z + 4 * n * n);
  L->hczt.assign(T->cell_zt, T->cell_zt + 4 * n * n);
  if (L->has_patch) {
    L->hpz.assign(T->patch_z, T->patch_z + 16 * n * n);
    L->hpzt.assign(T->patch_zt, T->patch_zt + 16 * n * n);
    if (T->patch_eo) L->hpeo.assign(T->patch_eo, T->patch_eo + 4 * n * n);
  }
  const int m = L->m;
  const int64_t pw = (d == 3) ? 64 : (d == 2 ? 16 : 4);  // 4^d classes
  const int64_t ce = L->cell_dofs,
                pe = (d == 3) ? (int64_t)m * m * m : (d == 2 ? (int64_t)m * m : m);
  std::vector<std::pair<const double*, int64_t>> parts = {
      {T->mass, n * n},  {T->adiag, 4 * n * n}, {T->bg, 2 * n},
      {T->cell_z, 4 * n * n}, {T->cell_zt, 4 * n * n}, {T->cell_invsum, pw * ce}};
  if (L->has_patch) {
    parts.push_back({T->patch_z, 4 * m * m});
    parts.push_back({T->patch_zt, 4 * m * m});
    parts.push_back({T->patch_invsum, pw * pe});
  }
  const int ceo_at = (int)parts.size();
  if (!L->hceo.empty()) parts.push_back({L->hceo.data(), (int64_t)L->hceo.size()});
  const int peo_at = (int)parts.size();
  if (!L->hpeo.empty()) parts.push_back({L->hpeo.data(), (int64_t)L->hpeo.size()});
  int64_t total = 0;
  for (auto& pr : parts) total += (pr.second + 1) & ~int64_t(1);
  cudaError_t e = cudaMalloc(&L->dtab, total * sizeof(double));
  if (e != cudaSuccess) {
    free_level(L);
    return fail(DG_ECUDA, std::string("cudaMalloc tables: ") + cudaGetErrorString(e));
  }
  std::vector<const double*> dptr;
  int64_t off = 0;
  for (auto& pr : parts) {
    if (!pr.first) {
      free_level(L);
      return fail(DG_EINVAL, "missing table");
    }
    e = cudaMemcpy(L->dtab + off, pr.first, pr.second * sizeof(double), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      free_level(L);
      return fail(DG_ECUDA, std::string("cudaMemcpy tables: ") + cudaGetErrorString(e));
    }
    dptr.push_back(L->dtab + off);
    off += (pr.second + 1) & ~int64_t(1);
  }
  L->mass = dptr[0];
  L->adiag = dptr[1];
  L->bg = dptr[2];
  L->cz = dptr[3];
  L->czt = dptr[4];
  L->cinv = dptr[5];
  if (L->has_patch) {
    L->pz = dptr[6];
    L->pzt = dptr[7];
    L->pinv = dptr[8];
  }
  if (!L->hceo.empty()) L->ceod = dptr[ceo_at];
  e = cudaMalloc(&L->wcount, 16 * sizeof(int));
  if (e != cudaSuccess) {
    free_level(L);
    return fail(DG_ECUDA, std::string("cudaMalloc counter: ") + cudaGetErrorString(e));
  }
  if (!L->hpeo.empty()) L->peod = dptr[peo_at];
  if (L->has_patch) {
    // degree >= 8 patches run the generic kernel; its 3D m = 32 tensor does
    // not fit in shared memory and lives in a per-CTA slice of this buffer
    const size_t sb = patch_fdm_scratch_bytes(d, n);
    if (sb) {
      int dev = 0, sms = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      L->big_slots = 2 * std::max(1, sms);
      e = cudaMalloc(&L->big_scratch, sb * (size_t)L->big_slots);
      if (e != cudaSuccess) {
        free_level(L);
        return fail(DG_ECUDA, std::string("cudaMalloc patch scratch: ") + cudaGetErrorString(e));
      }
    }
  }

  // ---- colour lists -------------------------------------------------------
  const int* nc = desc->ncells;
  const int zb = desc->z_begin;
  auto local_of = [&](const int* c) -> int32_t {
    if (d == 1) return (int32_t)(c[0] - zb);
    if (d == 2) return (int32_t)(c[0] + (int64_t)nc[0] * (c[1] - zb));
    return (int32_t)(c[0] + (int64_t)nc[0] * (c[1] + (int64_t)nc[1] * (c[2] - zb)));
  };
  // red-black over owned cells (mesh.py:350-357), ascending local ids
  {
    std::vector<int32_t> col[2], colp[2];
    const int64_t c0 = (int64_t)(desc->own_begin - zb) * L->layer_cells;
    const int64_t c1 = (int64_t)(desc->own_end - zb) * L->layer_cells;
    for (int64_t id = c0; id < c1; ++id) {
      int64_t rem = id;
      int s = 0, cc3[3] = {0, 0, 0};
      for (int t = 0; t < d; ++t) {
        const int64_t ct = (t == d - 1) ? rem + zb : rem % nc[t];
        rem /= nc[t];
        s += (int)ct;
        cc3[t] = (int)ct;
      }
      col[s & 1].push_back((int32_t)id);
      colp[s & 1].push_back(pack_d(d, cc3[0], cc3[1], cc3[2]));
    }
    for (int k = 0; k < 2; ++k) {
      if (col[k].empty()) continue;
      DevList dl, dp;
      int rc = upload_list(col[k], &dl);
      L->rb.push_back(dl);
      if (!rc) rc = upload_list(colp[k], &dp);
      L->rb_pk.push_back(dp);
      if (rc) { free_level(L); return rc; }
    }
  }
  // structured patch colours (mesh.py:360-375) for vertices v_d in
  // [pv_begin, pv_end]; ids ascending inside each colour
  if (L->has_patch) {
    const int ncol = 1 << (d + 1);
    std::vector<std::vector<int32_t>> pc(ncol), cc(ncol), pcp(ncol), ccp(ncol);
    bool ok = true;
    for (int t = 0; t < d; ++t) ok = ok && nc[t] >= 2;
    const int vlo = std::max(1, desc->pv_begin), vhi = std::min(nc[d - 1] - 1, desc->pv_end);
    if (ok && vlo <= vhi) {
      if (vlo - 1 < zb || vhi > zb + desc->z_count - 1) {
        free_level(L);
        return fail(DG_EINVAL, "patch vertex range needs cell layers outside the window");
      }
      int64_t layer_patches = 1;
      for (int t = 0; t < d - 1; ++t) layer_patches *= (nc[t] - 1);
      const int64_t p0 = (int64_t)(vlo - 1) * layer_patches, p1 = (int64_t)vhi * layer_patches;
      L->pall_vlo = vlo;
      L->layer_patches = layer_patches;
      for (int64_t id = p0; id < p1; ++id) {
        int64_t rem = id;
        int v[3] = {1, 1, 1}, parq = 0, half = 0;
        for (int t = 0; t < d; ++t) {
          v[t] = 1 + (int)(rem % (nc[t] - 1));
          rem /= (nc[t] - 1);
          parq += (v[t] & 1) << t;
          half += v[t] / 2;
        }
        const int col = parq * 2 + (half & 1);
        pc[col].push_back((int32_t)id);
        pcp[col].push_back(pack_d(d, v[0], d >= 2 ? v[1] : 0, d == 3 ? v[2] : 0));
        for (int s = 0; s < (1 << d); ++s) {
          int c[3] = {0, 0, 0};
          for (int t = 0; t < d; ++t) c[t] = v[t] - 1 + ((s >> t) & 1);
          cc[col].push_back(local_of(c));
          ccp[col].push_back(pack_d(d, c[0], c[1], c[2]));
        }
      }
    }
    {
      // one-launch additive step: patches in spatial order (v_1 fastest), so
      // the CTAs in flight work on a thin z-slab whose r and x stay in L2
      // while its cells receive their 2^d overlapping updates; colour order
      // with DGB_AVS_ATOMIC_ORDER=0
      std::vector<int32_t> all;
      if (env_int("DGB_AVS_ATOMIC_ORDER", 1)) {
        std::vector<std::pair<int32_t, int32_t>> srt;  // (patch id, packed vertex)
        for (int k = 0; k < ncol; ++k)
          for (size_t i = 0; i < pc[k].size(); ++i) srt.push_back({pc[k][i], pcp[k][i]});
        std::sort(srt.begin(), srt.end());
        for (auto& e2 : srt) all.push_back(e2.second);
      } else {
        for (int k = 0; k < ncol; ++k) all.insert(all.end(), pcp[k].begin(), pcp[k].end());
      }
      if (int rc = upload_list(all, &L->pall_pk)) { free_level(L); return rc; }
    }
    // Additive launch order.  Colours 2q and 2q+1 share the vertex parity q,
    // so together they are write-disjoint (stride-2 vertex lattice) and one
    // launch serves both; every dof still receives its parity-class updates
    // in class order, so with one window this is bitwise the colour-by-colour
    // step.  With W > 0 the classes run window by window along the last
    // direction (v_last in [1 + wW, 1 + (w+1)W), global windows), so a
    // window's x and r (W+1 cell layers) stay in L2 across its 2^d class
    // launches; only dofs of a window's boundary layer see their updates in
    // (window, class) order instead (rounding-level difference, identical on
    // every slab decomposition because the windows are global).
#ifdef DGB_EXPERIMENTAL
    L->avs_win = std::max(0, env_int("DGB_AVS_WIN", 0));
#endif
    {
      const int W = L->avs_win;
      const int nq = 1 << d;
      const int nw = (W > 0 && vlo <= vhi) ? (vhi - 1) / W - (vlo - 1) / W + 1 : 1;
      const int w0 = (W > 0 && vlo <= vhi) ? (vlo - 1) / W : 0;
      for (int w = 0; w < nw; ++w)
        for (int q = 0; q < nq; ++q) {
          std::vector<int32_t> lst;
          for (int k = 2 * q; k <= 2 * q + 1; ++k)
            for (int32_t e : pcp[k]) {
              const int vl = (d == 3) ? (e >> 20) & 1023 : (d == 2 ? (e >> 15) & 32767 : e);
              if (W <= 0 || (vl - 1) / W == w0 + w) lst.push_back(e);
            }
          if (lst.empty()) continue;
          DevList dl;
          int rc = upload_list(lst, &dl);
          L->pwin_pk.push_back(dl);
          if (rc) { free_level(L); return rc; }
        }
    }
    for (int k = 0; k < ncol; ++k) {
      if (pc[k].empty()) continue;
      DevList a, b, ap, bp;
      int rc = upload_list(pc[k], &a);
      L->pcol.push_back(a);
      if (!rc) rc = upload_list(cc[k], &b);
      L->pcol_cells.push_back(b);
      if (!rc) rc = upload_list(pcp[k], &ap);
      L->pcol_pk.push_back(ap);
      {
        const int nv = nc[d - 1] + 1;
        std::vector<int64_t> off(nv + 1, 0);
        for (int32_t e : pcp[k]) {
          const int vl = (d == 3) ? (e >> 20) & 1023 : (d == 2 ? (e >> 15) & 32767 : e);
          ++off[vl + 1];
        }
        for (int v = 1; v <= nv; ++v) off[v] += off[v - 1];
        L->pcol_voff.push_back(off);
      }
      if (!rc) rc = upload_list(ccp[k], &bp);
      L->pcol_cells_pk.push_back(bp);
      if (rc) { free_level(L); return rc; }
    }
  }
#ifdef DGB_EXPERIMENTAL
  // 2^d-patch clusters for the additive step (cluster_kernel): base vertex
  // v0 = 2a+1 per direction, colour = parity of a; only clusters with a patch
  // vertex in [pv_begin, pv_end] along the last direction
  if (L->has_patch && d >= 2) {
    bool ok = true;
    for (int t = 0; t < d; ++t) ok = ok && nc[t] >= 2;
    const int vlo = std::max(1, desc->pv_begin), vhi = std::min(nc[d - 1] - 1, desc->pv_end);
    if (ok && vlo <= vhi) {
      const int ncl = 1 << d;
      std::vector<std::vector<int32_t>> cl(ncl);
      int na[3] = {1, 1, 1};
      for (int t = 0; t < d; ++t) na[t] = nc[t] / 2;  // a = 0 .. (nc-2)/2 covers v = 1 .. nc-1
      int a[3] = {0, 0, 0};
      for (a[2] = 0; a[2] < (d == 3 ? na[2] : 1); ++a[2])
        for (a[1] = 0; a[1] < na[1]; ++a[1])
          for (a[0] = 0; a[0] < na[0]; ++a[0]) {
            const int zlo = 2 * a[d - 1] + 1, zhi = 2 * a[d - 1] + 2;
            if (zhi < vlo || zlo > vhi) continue;
            int col = 0;
            for (int t = 0; t < d; ++t) col |= (a[t] & 1) << t;
            cl[col].push_back(pack_d(d, 2 * a[0] + 1, 2 * a[1] + 1, d == 3 ? 2 * a[2] + 1 : 0));
          }
      for (int k = 0; k < ncl; ++k) {
        if (cl[k].empty()) continue;
        DevList dl;
        int rc = upload_list(cl[k], &dl);
        L->clus_pk.push_back(dl);
        if (rc) { free_level(L); return rc; }
      }
    }
  }
#endif  // DGB_EXPERIMENTAL
  if (desc->own_begin < zb || desc->own_end > zb + desc->z_count ||
      desc->own_begin > desc->own_end) {
    free_level(L);
    return fail(DG_EINVAL, "owned layers outside the window");
  }
  if (int rc = check_layers(L, desc->res_begin, desc->res_end)) {
    free_level(L);
    return rc;
  }
#ifdef DGB_EXPERIMENTAL
  if (int rc = build_flow(L)) {
    free_level(L);
    return rc;
  }
#endif
  {
    // the capture stream carries the patch solves at the highest priority;
    // the residual chunks of the overlapped AVS step run on `side` at the
    // lowest, so free CTA slots go to the solves first
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    e = cudaStreamCreateWithPriority(&L->cap, cudaStreamNonBlocking, hi);
    if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&L->side, cudaStreamNonBlocking, lo);
    if (e != cudaSuccess) {
      free_level(L);
      return fail(DG_ECUDA, std::string("stream create: ") + cudaGetErrorString(e));
    }
  }
  *out = L;
  return DG_OK;
}

int dg_level_destroy(dg_level_t* L) {
  free_level(L);
  return DG_OK;
}

int64_t dg_level_ndofs(const dg_level_t* L) { return L ? L->ndofs : -1; }

int dg_apply(const dg_level_t* L, const double* u, double* v, int z0, int z1, void* stream) {
  if (!L || !u || !v) return fail(DG_EINVAL, "null argument");
  if (u == v) return fail(DG_EINVAL, "apply_operator: output must not alias input");
  if (int rc = check_layers(L, z0, z1)) return rc;
  if (int rc = check_align(L, u, v, nullptr)) return rc;
  ResArgs p = res_params(L, u, nullptr, v);
  p.start = (int64_t)(z0 - L->desc.z_begin) * L->layer_cells;
  p.count = (int64_t)(z1 - z0) * L->layer_cells;
  return dispatch_residual(L->d, L->n, p, L->hres(), (cudaStream_t)stream);
}

int dg_residual(const dg_level_t* L, const double* x, const double* b, double* r, int z0,
                int z1, void* stream) {
  if (!L || !x || !b || !r) return fail(DG_EINVAL, "null argument");
  if (r == x) return fail(DG_EINVAL, "residual: output must not alias x");
  if (int rc = check_layers(L, z0, z1)) return rc;
  if (int rc = check_align(L, x, b, r)) return rc;
  ResArgs p = res_params(L, x, b, r);
  p.start = (int64_t)(z0 - L->desc.z_begin) * L->layer_cells;
  p.count = (int64_t)(z1 - z0) * L->layer_cells;
  return dispatch_residual(L->d, L->n, p, L->hres(), (cudaStream_t)stream);
}

int dg_residual_cells(const dg_level_t* L, const double* x, const double* b, double* r,
                      const int32_t* cells, int64_t n_cells, void* stream) {
  if (!L || !x || !b || !r || (!cells && n_cells > 0)) return fail(DG_EINVAL, "null argument");
  if (r == x) return fail(DG_EINVAL, "residual: output must not alias x");
  if (int rc = check_align(L, x, b, r)) return rc;
  ResArgs p = res_params(L, x, b, r);
  p.list = cells;
  p.count = n_cells;
  return dispatch_residual(L->d, L->n, p, L->hres(), (cudaStream_t)stream);
}

int dg_cell_fdm(const dg_level_t* L, const double* r, double* x, double omega,
                const int32_t* cells, int64_t n_cells, void* stream) {
  if (!L || !r || !x) return fail(DG_EINVAL, "null argument");
  if (r == x) return fail(DG_EINVAL, "cell solve: r must not alias x");
  if (int rc = check_align(L, r, x, nullptr)) return rc;
  FdmArgs p = fdm_params(L, false, r, x, omega);
  if (cells) {
    p.list = cells;
    p.count = n_cells;
  } else {
    p.start = (int64_t)(L->desc.own_begin - L->desc.z_begin) * L->layer_cells;
    p.count = (int64_t)(L->desc.own_end - L->desc.own_begin) * L->layer_cells;
  }
  return dispatch_cell_fdm(L->d, L->n, p, L->hcz.data(), L->hczt.data(), L->ceo(), (cudaStream_t)stream);
}

int dg_patch_fdm(const dg_level_t* L, const double* r, double* x, double omega,
                 const int32_t* patches, int64_t n_patches, int atomic, void* stream) {
  if (!L || !r || !x || (!patches && n_patches > 0)) return fail(DG_EINVAL, "null argument");
  if (r == x) return fail(DG_EINVAL, "patch solve: r must not alias x");
  if (int rc = check_align(L, r, x, nullptr)) return rc;
  if (!L->has_patch)
    return fail(DG_EUNSUPPORTED, "vertex-patch tables not available (degree > 7?)");
  FdmArgs p = fdm_params(L, true, r, x, omega);
  p.list = patches;
  p.count = n_patches;
  p.atomic = atomic;
  return dispatch_patch_fdm(L->d, L->n, p, L->hpz.data(), L->hpzt.data(), L->peo(), (cudaStream_t)stream);
}

int dg_solve_range(const dg_level_t* L, int kind, double omega, const double* r, double* x,
                   int lo, int hi, void* stream) {
  if (!L || !r || !x) return fail(DG_EINVAL, "null argument");
  if (r == x) return fail(DG_EINVAL, "solve: r must not alias x");
  if (int rc = check_align(L, r, x, nullptr)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (kind == DG_ACS) {
    // cells of owned layers [lo, hi)
    const int z0 = std::max(lo, L->desc.own_begin), z1 = std::min(hi, L->desc.own_end);
    if (z1 <= z0) return DG_OK;
    FdmArgs p = fdm_params(L, false, r, x, omega);
    p.start = (int64_t)(z0 - L->desc.z_begin) * L->layer_cells;
    p.count = (int64_t)(z1 - z0) * L->layer_cells;
    return dispatch_cell_fdm(L->d, L->n, p, L->hcz.data(), L->hczt.data(), L->ceo(), st);
  }
  if (kind == DG_AVS) {
    // patches with last vertex coordinate in [lo, hi): a contiguous range of
    // the spatially ordered all-patch list, overlaps by bulk reduce-add
    if (!L->has_patch) return fail(DG_EUNSUPPORTED, "vertex patches unsupported here");
    if (!env_int("DGB_AVS_ATOMIC_ORDER", 1))
      return fail(DG_EINVAL, "dg_solve_range needs the spatial patch order");
    if (L->pall_pk.count == 0) return DG_OK;
    auto idx = [&](int v) {
      const int vv = std::max(L->pall_vlo, v);
      return std::min<int64_t>(L->pall_pk.count, (int64_t)(vv - L->pall_vlo) * L->layer_patches);
    };
    const int64_t i0 = idx(lo), i1 = idx(hi);
    if (i1 <= i0) return DG_OK;
    FdmArgs p = fdm_params(L, true, r, x, omega);
    p.list = L->pall_pk.ptr + i0;
    p.count = i1 - i0;
    p.packed = 1;
    p.atomic = 1;
    return dispatch_patch_fdm(L->d, L->n, p, L->hpz.data(), L->hpzt.data(), L->peo(), st);
  }
  return fail(DG_EINVAL, "dg_solve_range: kind must be DG_ACS or DG_AVS");
}

int dg_num_colours(const dg_level_t* L, int kind) {
  if (!L) return -1;
  switch (kind) {
    case DG_ACS: return 1;
    case DG_MCS: return (int)L->rb.size();
    case DG_AVS:
    case DG_MVS: return (int)L->pcol.size();
  }
  return -1;
}

int dg_colour_list(const dg_level_t* L, int kind, int colour, const int32_t** ids,
                   int64_t* count) {
  if (!L || !ids || !count) return fail(DG_EINVAL, "null argument");
  const std::vector<DevList>* v = nullptr;
  if (kind == DG_MCS) v = &L->rb;
  else if (kind == DG_AVS || kind == DG_MVS) v = &L->pcol;
  else if (kind == 100) v = &L->pcol_cells;
  if (!v || colour < 0 || colour >= (int)v->size()) return fail(DG_EINVAL, "no such colour");
  *ids = (*v)[colour].ptr;
  *count = (*v)[colour].count;
  return DG_OK;
}

int dg_patch_gather_map(const dg_level_t* L, const int32_t* patches, int64_t count,
                        int64_t* out, void* stream) {
  if (!L || (!patches && count > 0) || (!out && count > 0)) return fail(DG_EINVAL, "null argument");
  if (count <= 0) return DG_OK;
  MapParams p{};
  p.list = patches;
  p.count = count;
  p.out = out;
  p.m = L->m;
  p.n = L->n;
  p.d = L->d;
  p.geo = L->geo;
  gather_map_kernel<<<1024, 256, 0, (cudaStream_t)stream>>>(p);
  DG_CUDA(cudaGetLastError());
  return DG_OK;
}

// internal launches over the level's packed colour lists (no index division)
static int res_packed(dg_level_t* L, const double* x, const double* b, double* r,
                      const DevList& l, cudaStream_t st, int block_list = 0) {
  ResArgs p = res_params(L, x, b, r);
  p.list = l.ptr;
  p.count = l.count;
  p.packed = 1;
  p.block_list = block_list;
  return dispatch_residual(L->d, L->n, p, L->hres(), st);
}

static int cell_fdm_packed(dg_level_t* L, const double* r, double* x, double omega,
                           const DevList& l, cudaStream_t st) {
  FdmArgs p = fdm_params(L, false, r, x, omega);
  p.list = l.ptr;
  p.count = l.count;
  p.packed = 1;
  return dispatch_cell_fdm(L->d, L->n, p, L->hcz.data(), L->hczt.data(), L->ceo(), st);
}

static int patch_fdm_packed(dg_level_t* L, const double* r, double* x, double omega,
                            const DevList& l, cudaStream_t st) {
  FdmArgs p = fdm_params(L, true, r, x, omega);
  p.list = l.ptr;
  p.count = l.count;
  p.packed = 1;
  return dispatch_patch_fdm(L->d, L->n, p, L->hpz.data(), L->hpzt.data(), L->peo(), st);
}

static int smooth_launches(dg_level_t* L, int kind, double omega, int reverse, double* x,
                           const double* b, double* r, cudaStream_t st, int64_t* nl) {
  int rc = DG_OK;
  *nl = 0;
  auto res_range = [&]() {
    ResArgs p = res_params(L, x, b, r);
    p.start = (int64_t)(L->desc.res_begin - L->desc.z_begin) * L->layer_cells;
    p.count = (int64_t)(L->desc.res_end - L->desc.res_begin) * L->layer_cells;
    ++*nl;
    return dispatch_residual(L->d, L->n, p, L->hres(), st);
  };
  switch (kind) {
    case DG_ACS: {
      if ((rc = res_range())) return rc;
      ++*nl;
      return dg_cell_fdm(L, r, x, omega, nullptr, 0, st);
    }
    case DG_AVS: {
      if (!L->has_patch) return fail(DG_EUNSUPPORTED, "vertex patches unsupported here");
#ifdef DGB_EXPERIMENTAL
      if (L->flow_ok && env_int("DGB_FLOW", 0)) {
        ++*nl;
        ResArgs ra = res_params(L, x, b, r);
        FdmArgs fa = fdm_params(L, true, r, x, omega);
        return dispatch_flow(L->d, L->n, ra, fa, L->hres(), L->hpz.data(), L->hpzt.data(),
                             L->peo(), L->flow, st);
      }
#endif
      const int64_t pdofs = L->pall_pk.count * (L->d == 3 ? (int64_t)L->m * L->m * L->m
                                                          : (int64_t)L->m * L->m);
      const int64_t amax = (int64_t)env_int("DGB_AVS_ATOMIC_MAX_MDOFS", 1 << 30) * 1000000;
#ifdef DGB_EXPERIMENTAL
      if (env_int("DGB_AVS_ATOMIC", 1) && L->pall_pk.count > 0 && pdofs <= amax &&
          L->d == 3 && env_int("DGB_AVS_OVERLAP", 0)) {
        // residual and solves overlapped in z-chunks of C cell layers on two
        // streams: R(k) = residual on layers [z_k, z_k+1), S(k) = patches with
        // v_z in (z_k, z_k+1] (they read r on [z_k, z_k+1] and add into x
        // there).  S(k) waits for R(k+1): every residual that reads x on
        // those layers (R(k-1..k+1)) is done before S(k) writes them, and
        // R(k+2) reads layers >= z_k+2 - 1 > z_k+1, so it runs concurrently.
        // The solves' stream has the higher priority; the residual chunks
        // fill the CTA slots the solves leave.  Opt-in: measured no gain on
        // cfg 5 (2.47 ms for chunks of 8/16 layers, 2.5-2.7 ms when the
        // residual is held at most DGB_AVS_LEAD chunks ahead) -- both kernels
        // are bound by the SM's L1/shared pipe, so running them side by side
        // does not add throughput.
        const int C = std::max(2, env_int("DGB_AVS_CHUNK", 8) & ~1);
        const int z0 = L->desc.res_begin, z1 = L->desc.res_end;
        const int K = (z1 - z0 + C - 1) / C;
        if (K >= 3) {
          // events: ev[0..K) residual chunks, ev[K..2K) solve chunks, fork, join
          if ((int)L->ev.size() < 2 * K + 2) {
            for (int i = (int)L->ev.size(); i < 2 * K + 2; ++i) {
              cudaEvent_t e2;
              DG_CUDA(cudaEventCreateWithFlags(&e2, cudaEventDisableTiming));
              L->ev.push_back(e2);
            }
          }
          cudaStream_t sd = L->side;
          DG_CUDA(cudaEventRecord(L->ev[2 * K], st));  // fork
          DG_CUDA(cudaStreamWaitEvent(sd, L->ev[2 * K], 0));
          auto zc = [&](int k) { return std::min(z1, z0 + k * C); };
          auto pidx = [&](int v) {  // first index in pall_pk with v_last >= v
            const int vv = std::max(L->pall_vlo, v);
            return std::min<int64_t>(L->pall_pk.count, (int64_t)(vv - L->pall_vlo) * L->layer_patches);
          };
          // R(k) may run ahead of the solves by `lead` chunks: R(k) waits for
          // S(k - lead - 1), so the hardware queue holds a mix of both
          const int lead = std::max(1, env_int("DGB_AVS_LEAD", 2));
          auto launch_r = [&](int k) -> int {
            if (k >= K) return DG_OK;
            if (k - lead - 1 >= 0) DG_CUDA(cudaStreamWaitEvent(sd, L->ev[K + k - lead - 1], 0));
            ResArgs p = res_params(L, x, b, r);
            p.start = (int64_t)(zc(k) - L->desc.z_begin) * L->layer_cells;
            p.count = (int64_t)(zc(k + 1) - zc(k)) * L->layer_cells;
            ++*nl;
            if (int rc2 = dispatch_residual(L->d, L->n, p, L->hres(), sd)) return rc2;
            DG_CUDA(cudaEventRecord(L->ev[k], sd));
            return DG_OK;
          };
          for (int k = 0; k <= lead; ++k)
            if ((rc = launch_r(k))) return rc;
          for (int k = 0; k < K; ++k) {
            const int64_t i0 = k == 0 ? 0 : pidx(zc(k) + 1);
            const int64_t i1 = k == K - 1 ? L->pall_pk.count : pidx(zc(k + 1) + 1);
            DG_CUDA(cudaStreamWaitEvent(st, L->ev[std::min(k + 1, K - 1)], 0));
            if (i1 > i0) {
              ++*nl;
              FdmArgs p = fdm_params(L, true, r, x, omega);
              p.list = L->pall_pk.ptr + i0;
              p.count = i1 - i0;
              p.packed = 1;
              p.atomic = 1;
              if ((rc = dispatch_patch_fdm(L->d, L->n, p, L->hpz.data(), L->hpzt.data(), L->peo(),
                                           st)))
                return rc;
            }
            DG_CUDA(cudaEventRecord(L->ev[K + k], st));
            if ((rc = launch_r(k + lead + 1))) return rc;
          }
          DG_CUDA(cudaEventRecord(L->ev[2 * K + 1], sd));  // join
          DG_CUDA(cudaStreamWaitEvent(st, L->ev[2 * K + 1], 0));
          return DG_OK;
        }
      }
#endif  // DGB_EXPERIMENTAL
      if ((rc = res_range())) return rc;
      // default: one launch over all patches in spatial order; the overlaps
      // accumulate by the TMA engine's fp64 bulk reduce-add at L2 (atomic per
      // element), and the in-flight patches form a thin z-slab whose r and x
      // stay in L2 while each cell takes its 2^d updates.  Measured: cfg 5
      // 2.65 -> 2.47 ms (vs one launch per parity class), cfg 2 0.111 ->
      // 0.091 ms.  The summation order of a dof's 2^d updates then varies
      // run to run (~1e-16 relative); DGB_AVS_ATOMIC=0 gives the
      // deterministic parity-class launches (bitwise the reference's colour
      // order).  DGB_AVS_ATOMIC_MAX_MDOFS caps the patch dofs of this path.
      if (env_int("DGB_AVS_ATOMIC", 1) && L->pall_pk.count > 0 && pdofs <= amax) {
        ++*nl;
        FdmArgs p = fdm_params(L, true, r, x, omega);
        p.list = L->pall_pk.ptr;
        p.count = L->pall_pk.count;
        p.packed = 1;
        p.atomic = 1;
        return dispatch_patch_fdm(L->d, L->n, p, L->hpz.data(), L->hpzt.data(), L->peo(), st);
      }
#ifdef DGB_EXPERIMENTAL
      if (env_int("DGB_CLUSTER", 0) && !L->clus_pk.empty()) {
        for (auto& c : L->clus_pk) {
          ++*nl;
          FdmArgs p = fdm_params(L, true, r, x, omega);
          p.list = c.ptr;
          p.count = c.count;
          p.packed = 1;
          p.cluster = 1;
          p.pv_lo = std::max(1, L->desc.pv_begin);
          p.pv_hi = std::min(L->desc.ncells[L->d - 1] - 1, L->desc.pv_end);
          if ((rc = dispatch_patch_fdm(L->d, L->n, p, L->hpz.data(), L->hpzt.data(), L->peo(), st)))
            return rc;
        }
        return DG_OK;
      }
#endif  // DGB_EXPERIMENTAL
      const auto& order = env_int("DGB_AVS_COLOURS", 0) ? L->pcol_pk : L->pwin_pk;
      for (auto& c : order) {
        ++*nl;
        if ((rc = patch_fdm_packed(L, r, x, omega, c, st))) return rc;
      }
      return DG_OK;
    }
    case DG_MCS: {
      const int nc = (int)L->rb_pk.size();
      for (int i = 0; i < nc; ++i) {
        const auto& c = L->rb_pk[reverse ? nc - 1 - i : i];
        *nl += 2;
        if ((rc = res_packed(L, x, b, r, c, st))) return rc;
        if ((rc = cell_fdm_packed(L, r, x, omega, c, st))) return rc;
      }
      return DG_OK;
    }
    case DG_MVS: {
      if (!L->has_patch) return fail(DG_EUNSUPPORTED, "vertex patches unsupported here");
      const int nc = (int)L->pcol_pk.size();
      // one launch per colour with the restricted residual fused into the
      // patch solve (mvs_fused.cuh; experimental builds, DGB_MVS_FUSED=1):
      // bitwise the two-launch sweep, measured slower (cfg 3: 2.27 vs 2.05 ms)
      const bool fused = mvs_fused_supported(L->d, L->n) && env_int("DGB_MVS_FUSED", 0);
      for (int i = 0; i < nc; ++i) {
        const int k = reverse ? nc - 1 - i : i;
        if (fused) {
          *nl += 1;
          ResArgs ra = res_params(L, x, b, r);
          FdmArgs fa = fdm_params(L, true, r, x, omega);
          fa.list = L->pcol_pk[k].ptr;
          fa.count = L->pcol_pk[k].count;
          fa.packed = 1;
          if ((rc = dispatch_mvs_fused(L->d, L->n, ra, fa, L->hres(), L->hpz.data(),
                                       L->hpzt.data(), L->peo(), st)))
            return rc;
          continue;
        }
        *nl += 2;
        if ((rc = res_packed(L, x, b, r, L->pcol_cells_pk[k], st, 1))) return rc;
        if ((rc = patch_fdm_packed(L, r, x, omega, L->pcol_pk[k], st))) return rc;
      }
      return DG_OK;
    }
  }
  return fail(DG_EINVAL, "unknown smoother kind");
}

int dg_mvs_range(const dg_level_t* Lc, int colour, int what, double omega, double* x,
                 const double* b, double* r, int vlo, int vhi, void* stream) {
  dg_level_t* L = const_cast<dg_level_t*>(Lc);
  if (!L || !x || !b || !r) return fail(DG_EINVAL, "null argument");
  if (r == x || r == b) return fail(DG_EINVAL, "scratch residual must not alias x or b");
  if (!L->has_patch) return fail(DG_EUNSUPPORTED, "vertex patches unsupported here");
  if (colour < 0 || colour >= (int)L->pcol_pk.size()) return fail(DG_EINVAL, "colour out of range");
  if (int rc = check_align(L, x, b, r)) return rc;
  const auto& off = L->pcol_voff[colour];
  const int nv = (int)off.size() - 1;
  const int64_t i0 = off[std::min(std::max(vlo, 0), nv)], i1 = off[std::min(std::max(vhi, 0), nv)];
  if (i1 <= i0) return DG_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int cells = 1 << L->d;
  if (what & 1) {
    DevList l{L->pcol_cells_pk[colour].ptr + cells * i0, cells * (i1 - i0)};
    if (int rc = res_packed(L, x, b, r, l, st, 1)) return rc;
  }
  if (what & 2) {
    DevList l{L->pcol_pk[colour].ptr + i0, i1 - i0};
    if (int rc = patch_fdm_packed(L, r, x, omega, l, st)) return rc;
  }
  return DG_OK;
}

int dg_smooth(dg_level_t* L, int kind, double omega, int reverse, double* x, const double* b,
              double* r, int use_graph, void* stream) {
  if (!L || !x || !b || !r) return fail(DG_EINVAL, "null argument");
  if (r == x || r == b) return fail(DG_EINVAL, "scratch residual must not alias x or b");
  cudaStream_t st = (cudaStream_t)stream;
  if (!use_graph) return smooth_launches(L, kind, omega, reverse, x, b, r, st, &L->last_launches);
  GraphKey key{kind, omega, reverse ? 1 : 0, x, b, r, switch_signature()};
  auto it = L->graphs.find(key);
  if (it == L->graphs.end()) {
    if (L->graphs.size() >= 32) {
      cudaGraphExecDestroy(L->graphs.begin()->second);
      L->graphs.erase(L->graphs.begin());
    }
    DG_CUDA(cudaStreamBeginCapture(L->cap, cudaStreamCaptureModeThreadLocal));
    int64_t nl = 0;
    int rc = smooth_launches(L, kind, omega, reverse, x, b, r, L->cap, &nl);
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(L->cap, &graph);
    if (rc) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    if (e != cudaSuccess) return fail(DG_ECUDA, std::string("capture: ") + cudaGetErrorString(e));
    cudaGraphExec_t exec = nullptr;
    e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return fail(DG_ECUDA, std::string("instantiate: ") + cudaGetErrorString(e));
    it = L->graphs.emplace(key, exec).first;
    L->last_launches = nl;
  }
  DG_CUDA(cudaGraphLaunch(it->second, st));
  return DG_OK;
}

int64_t dg_last_launch_count(const dg_level_t* L) { return L ? L->last_launches : -1; }

int dg_flow_enabled(const dg_level_t* L) {
#ifdef DGB_EXPERIMENTAL
  return L && L->flow_ok && env_int("DGB_FLOW", 0) ? 1 : 0;
#else
  (void)L;
  return 0;
#endif
}

int dg_build_flags(void) {
  int f = 0;
#ifdef DGB_EXPERIMENTAL
  f |= DG_BUILD_EXPERIMENTAL;
#endif
#ifdef DGB_CHECKS
  f |= DG_BUILD_CHECKS;
#endif
  return f;
}

}  // extern "C"
