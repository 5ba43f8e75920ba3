// lopc_slab.cuh — multi-GPU slab mode; included by lopc_api.cu.
//
// Ranks own contiguous, chunk-aligned element ranges [e0, e1) of the linear
// order.  Each rank works on a "box": the whole z-planes (3D) / rows (2D)
// covering [e0 - H, e1 + H), H = d1 d2 + d2 + 1 (3D) / d2 + 1 (2D) = the
// largest linear distance of a star neighbour.  Points of the box outside
// [e0, e1) get no incoming arcs (k_quant_flags own range); those within H of
// the range are ghosts whose subbins come from the neighbour ranks:
//
//   round 1  : k_quant_flags + k_tiles (the single-GPU tile engine on the
//              box), ghosts = 0
//   round i+1: exchange the H boundary subbins with rank r-1 / r+1,
//              k_ghost_inject_tiles (raise ghosts in the planes, mark the
//              tiles of their successors), sum of raised ghosts over
//              ranks == 0 -> done, else k_tiles from the marked tiles (q0 = 2)
//
// A subbin above 8 planes (kErrPlanes; very long chains) makes every rank
// re-run the call on the u32 engine (k_sweep dense + sparse passes, ghosts
// injected by k_ghost_inject into its point worklist), same result.
//
// Every round only raises subbins toward the least fixpoint (all start at 0
// and every raise is a valid relaxation), and at termination every owned
// point satisfies its Bellman equation with the exact neighbour values, so
// the result is the unique least fixpoint of the whole grid (O9): identical
// to the single-GPU subbins, hence identical chunk payloads.  The payload
// offsets come from one allgather of the per-rank payload sizes.
//
// Transport: NCCL (dlopen'ed libnccl.so.2, the one torch loaded) between
// processes, or device copies between the slabs of one process
// (lopc_compress_slabs_local, the single-GPU test hook of the same code).
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <vector>

namespace {

struct SlabGeo {
  Shape g;                 // global grid
  Shape box;               // the rank's box (local grid)
  uint64_t e0, e1, P, H;   // owned range, slab unit (plane / row), halo
  uint64_t B0;             // global index of box element 0
  uint64_t glo, ghi;       // ghost points below e0 / above e1
  uint64_t send_lo, send_hi;  // boundary points sent to rank r-1 / r+1
  uint64_t C_local;
};

int slab_geo(const Shape& g, uint64_t e0, uint64_t e1, bool has_lo, bool has_hi, SlabGeo& s) {
  s = SlabGeo{};
  s.g = g;
  s.e0 = e0;
  s.e1 = e1;
  const uint64_t W = kChunkBytes / g.k;
  if (e0 >= e1 || e1 > g.n) return LOPC_E_SHAPE;
  if (e0 % W) return LOPC_E_SHAPE;
  if (e1 != g.n && e1 % W) return LOPC_E_SHAPE;
  const bool three = g.ndims == 3;
  s.P = three ? g.d1 * g.d2 : g.d2;
  s.H = three ? g.d1 * g.d2 + g.d2 + 1 : g.d2 + 1;
  const uint64_t lo = e0 > s.H ? e0 - s.H : 0, hi = e1 + s.H < g.n ? e1 + s.H : g.n;
  const uint64_t ulo = lo / s.P, uhi = (hi + s.P - 1) / s.P;
  s.B0 = ulo * s.P;
  s.box = g;
  if (three) {
    s.box.d0 = uhi - ulo;
  } else {
    s.box.d1 = uhi - ulo;
  }
  s.box.n = s.box.d0 * s.box.d1 * s.box.d2;
  s.box.C = (s.box.n + W - 1) / W;
  s.glo = has_lo ? (e0 < s.H ? e0 : s.H) : 0;
  s.ghi = has_hi ? (g.n - e1 < s.H ? g.n - e1 : s.H) : 0;
  // what the neighbours need from us (their ghosts), within our range
  s.send_lo = has_lo ? (g.n - e0 < s.H ? g.n - e0 : s.H) : 0;
  s.send_hi = has_hi ? (e1 < s.H ? e1 : s.H) : 0;
  if (s.send_lo > e1 - e0 || s.send_hi > e1 - e0) return LOPC_E_SHAPE;  // a middle range shorter than H
  s.C_local = (e1 - e0 + W - 1) / W;
  return LOPC_OK;
}

struct SlabLayout {
  CLayout L;  // repair + encode regions of the box
  size_t xbox, recv_lo, recv_hi, ctr_sum, total;
};

SlabLayout slab_layout(const SlabGeo& s) {
  SlabLayout S{};
  S.L = compress_layout(s.box, false, false);
  size_t o = S.L.total;
  S.xbox = o;
  o += al(s.box.k * s.box.n);
  S.recv_lo = o;
  o += al((size_t)s.g.k * s.H);  // x halo first (k bytes), then u32 subbins
  S.recv_hi = o;
  o += al((size_t)s.g.k * s.H);
  S.ctr_sum = o;
  o += al(16 * 1024);  // collective scratch: allreduce sum, status allgathers (<= 680 ranks)
  S.total = o;
  return S;
}

// One rank's (or one local slab's) state through a compress call.
struct Slab {
  SlabGeo geo;
  SlabLayout lay;
  uint8_t* ws;
  const void* x_own;  // device, e1 - e0 values
  double eps;
  cudaStream_t st;
  RepairArgs ra;
  bool tiles = true;  // repair engine: k_tiles (planes) or k_sweep (u32)
  uint64_t passes = 0, sparse_points = 0, rounds = 0;

  uint8_t* xbox() const { return ws + lay.xbox; }
  uint32_t* s() const { return reinterpret_cast<uint32_t*>(ws + lay.L.s); }
  Counters* dctr() const { return reinterpret_cast<Counters*>(ws + lay.L.ctr); }
  uint64_t own_lo() const { return geo.e0 - geo.B0; }
  uint64_t own_hi() const { return geo.e1 - geo.B0; }

  // x: own values into the box; everything else 0 until the halo arrives
  int setup() {
    CK(cudaMemsetAsync(ws, 0, lay.L.zero_end, st));
    CK(cudaMemsetAsync(xbox(), 0, geo.box.k * geo.box.n, st));
    CK(cudaMemcpyAsync(xbox() + geo.g.k * own_lo(), x_own, geo.g.k * (geo.e1 - geo.e0), cudaMemcpyDeviceToDevice, st));
    ra = make_repair_args(geo.box, xbox(), eps, ws, lay.L);
    ra.own_lo = (int64_t)own_lo();
    ra.own_hi = (int64_t)own_hi();
    ra.engine = 0;  // slab rounds build on the dense pass
    return LOPC_OK;
  }
  // halo pointers (element size esz: k for x, 4 for s)
  uint8_t* send_lo_ptr(uint8_t* base, size_t esz) const { return base + esz * own_lo(); }
  uint8_t* send_hi_ptr(uint8_t* base, size_t esz) const { return base + esz * (own_hi() - geo.send_hi); }
  uint8_t* ghost_lo_ptr(uint8_t* base, size_t esz) const { return base + esz * (own_lo() - geo.glo); }
  uint8_t* ghost_hi_ptr(uint8_t* base, size_t esz) const { return base + esz * own_hi(); }
  uint8_t* recv_lo() const { return ws + lay.recv_lo; }
  uint8_t* recv_hi() const { return ws + lay.recv_hi; }

  // the repair of round 1 (after k_quant_flags); with tiles the subbins stay
  // in the planes (the encoder reads them; the halo exchange widens only
  // the points it sends, widen_send)
  int repair1() {
    if (tiles) return launch_tiles(geo.box, ra, ws, lay.L, st, false);
    ra.skip_dense = 0;
    return launch_sweep(geo.box, ra, lay.L, st);
  }
  int round1() {
    int rc = launch_quant_flags(geo.box, ra, lay.L, st);
    if (rc) return rc;
    return repair1();
  }
  // after recv_lo/recv_hi hold the neighbours' boundary subbins
  int inject() {
    CK(cudaMemsetAsync(&dctr()->ghost_changed, 0, sizeof(uint64_t), st));
    if (tiles) {
      CK(cudaMemsetAsync(&dctr()->tl_count[0], 0, sizeof(dctr()->tl_count) + sizeof(dctr()->tl_ticket), st));
      const TileArgs ta = make_tile_args(geo.box, ra, ws, lay.L);
      auto gi = [&](const uint8_t* buf, uint64_t g0, uint64_t cnt) {
        const unsigned gb = (unsigned)((cnt + 255) / 256 < 1184 ? (cnt + 255) / 256 : 1184);
        if (geo.box.ndims == 3)
          k_ghost_inject_tiles<3><<<gb, 256, 0, st>>>(ta, reinterpret_cast<const uint32_t*>(buf), (int64_t)g0, (int64_t)cnt);
        else
          k_ghost_inject_tiles<2><<<gb, 256, 0, st>>>(ta, reinterpret_cast<const uint32_t*>(buf), (int64_t)g0, (int64_t)cnt);
      };
      if (geo.glo) gi(recv_lo(), own_lo() - geo.glo, geo.glo);
      if (geo.ghi) gi(recv_hi(), own_hi(), geo.ghi);
      CK(cudaGetLastError());
      return LOPC_OK;
    }
    CK(cudaMemsetAsync(&dctr()->list_count[0], 0, sizeof(dctr()->list_count), st));
    const bool i32 = use_i32(geo.box);
#define GI(ND, IX, BUF, G0, CNT)                                                                                   \
  k_ghost_inject<ND, IX><<<(unsigned)((CNT + 255) / 256 < 1184 ? (CNT + 255) / 256 : 1184), 256, 0, st>>>(       \
      ra, reinterpret_cast<const uint32_t*>(BUF), (int64_t)(G0), (int64_t)(CNT))
    if (geo.glo) {
      if (geo.box.ndims == 3) {
        if (i32) GI(3, int32_t, recv_lo(), own_lo() - geo.glo, geo.glo); else GI(3, int64_t, recv_lo(), own_lo() - geo.glo, geo.glo);
      } else {
        if (i32) GI(2, int32_t, recv_lo(), own_lo() - geo.glo, geo.glo); else GI(2, int64_t, recv_lo(), own_lo() - geo.glo, geo.glo);
      }
    }
    if (geo.ghi) {
      if (geo.box.ndims == 3) {
        if (i32) GI(3, int32_t, recv_hi(), own_hi(), geo.ghi); else GI(3, int64_t, recv_hi(), own_hi(), geo.ghi);
      } else {
        if (i32) GI(2, int32_t, recv_hi(), own_hi(), geo.ghi); else GI(2, int64_t, recv_hi(), own_hi(), geo.ghi);
      }
    }
#undef GI
    CK(cudaGetLastError());
    return LOPC_OK;
  }
  // tiles: the u32 subbins of the boundary points this slab sends
  int widen_send() {
    if (!tiles) return LOPC_OK;
    const uint32_t* sp = reinterpret_cast<const uint32_t*>(ws + lay.L.sp);
    auto wr = [&](uint64_t start, uint64_t cnt) {
      if (!cnt) return;
      const unsigned gb = (unsigned)((cnt + 255) / 256 < 1184 ? (cnt + 255) / 256 : 1184);
      k_planes_range<<<gb, 256, 0, st>>>(sp, s(), (int64_t)geo.box.d2, (int64_t)lay.L.nseg, (int64_t)start, (int64_t)cnt);
    };
    wr(own_lo(), geo.send_lo);
    wr(own_hi() - geo.send_hi, geo.send_hi);
    CK(cudaGetLastError());
    return LOPC_OK;
  }
  int sweep_sparse() {
    if (tiles) return launch_tiles(geo.box, ra, ws, lay.L, st, false, 2);
    ra.skip_dense = 1;
    return launch_sweep(geo.box, ra, lay.L, st);
  }
  // encode the owned chunks; out_local = table slice (8 C_local) ‖ payloads
  int encode(uint8_t* out_local, size_t cap, Timer* tm = nullptr) {
    const Shape& g = geo.g;
    EncodeArgs ea{};
    ea.x = x_own;
    ea.s = s() + own_lo();
    if (tiles) {  // planes mode: the box's planes and flags, offset by the owned range
      ea.sp = reinterpret_cast<const uint32_t*>(ws + lay.L.sp);
      ea.flags = reinterpret_cast<const uint32_t*>(ws + lay.L.flags);
      ea.nseg = (int64_t)lay.L.nseg;
      ea.sw = geo.box.ndims == 3 ? Geo<3>::SW : Geo<2>::SW;
      ea.sp_off = own_lo();
      ea.cesc = nullptr;  // its chunk bits are per box chunk: read every escape word
    }
    ea.stage = ws + lay.L.stage;
    ea.sizes = reinterpret_cast<uint32_t*>(ws + lay.L.sizes);
    ea.ctr = dctr();
    ea.eps = eps;
    ea.inv = 1.0 / eps;
    ea.inv32 = inv32_of(eps);
    ea.n = geo.e1 - geo.e0;
    ea.C = (uint32_t)geo.C_local;
    ea.ndims = g.ndims;
    ea.vec = ((uintptr_t)ea.x % 16 == 0) && ((uintptr_t)ea.s % 16 == 0);
    ea.prof = 0;
    ea.d0 = g.d0;
    ea.d1 = g.d1;
    ea.d2 = g.d2;
    set_escape_limits(ea, g.dtype == LOPC_F64, eps);
    const size_t smem = sizeof(EncSmem);
    launch_encode(ea, g.dtype == LOPC_F64, 1, (unsigned)geo.C_local, smem, st);
    launch_encode(ea, g.dtype == LOPC_F64, 2, (unsigned)geo.C_local, smem, st);
    CK(cudaGetLastError());
    if (tm) tm->mark();
    ScanArgs sa{};
    sa.sizes = ea.sizes;
    sa.C = (uint32_t)geo.C_local;
    sa.off = reinterpret_cast<uint64_t*>(ws + lay.L.off);
    sa.state = reinterpret_cast<uint64_t*>(ws + lay.L.state);
    sa.ctr = dctr();
    sa.base = 0;
    k_chunk_scan<<<(unsigned)((geo.C_local + kScanTile - 1) / kScanTile), kScanThreads, 0, st>>>(sa);
    CK(cudaGetLastError());
    PlaceArgs pa{};
    pa.stage = ea.stage;
    pa.sizes = ea.sizes;
    pa.off = sa.off;
    pa.table = out_local;
    pa.out = out_local + 8 * geo.C_local;
    pa.header = 0;
    pa.out_cap = cap > 8 * geo.C_local ? cap - 8 * geo.C_local : 0;
    pa.ctr = dctr();
    pa.C = (uint32_t)geo.C_local;
    DevInfo* di;
    int rc = dev_info(di);
    if (rc) return rc;
    uint64_t pg = (geo.C_local + 7) / 8;
    const uint64_t pmax = (uint64_t)di->sms * 8;
    if (pg > pmax) pg = pmax;
    k_place<<<(unsigned)pg, 256, 0, st>>>(pa);
    CK(cudaGetLastError());
    return LOPC_OK;
  }
};

// ---- NCCL through dlopen ---------------------------------------------------
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  const char* (*GetErrorString)(ncclResult_t);
};
NcclApi g_nccl;

int nccl_load() {
  if (g_nccl.h) return LOPC_OK;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the copy torch already loaded, if any
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
  if (!h) {
    snprintf(g_errmsg, sizeof(g_errmsg), "dlopen(libnccl.so.2): %s", dlerror());
    return LOPC_E_NCCL;
  }
#define SYM(F)                                                                   \
  g_nccl.F = reinterpret_cast<decltype(g_nccl.F)>(dlsym(h, "nccl" #F));          \
  if (!g_nccl.F) {                                                               \
    snprintf(g_errmsg, sizeof(g_errmsg), "libnccl.so.2 lacks nccl%s", #F);       \
    return LOPC_E_NCCL;                                                          \
  }
  SYM(GetUniqueId) SYM(CommInitRank) SYM(CommDestroy) SYM(Send) SYM(Recv) SYM(GroupStart) SYM(GroupEnd)
  SYM(AllReduce) SYM(AllGather) SYM(GetErrorString)
#undef SYM
  g_nccl.h = h;
  return LOPC_OK;
}

#define NK(call)                                                                                   \
  do {                                                                                             \
    ncclResult_t r_ = (call);                                                                      \
    if (r_ != ncclSuccess) {                                                                       \
      snprintf(g_errmsg, sizeof(g_errmsg), "%s: %s", #call, g_nccl.GetErrorString(r_));           \
      return LOPC_E_NCCL;                                                                          \
    }                                                                                              \
  } while (0)

int err_rank(int rc) { return rc < 0 ? -rc : 0; }

// Test hook: LOPC_FAULT_RANK=r and LOPC_FAULT_ROUND=k make rank r fail
// locally after repair round k (0 = after the first sweep), to exercise the
// slab mode's error agreement.  Off unless both are set.
bool fault_injected(int rank, int round) {
  static const int fr = getenv("LOPC_FAULT_RANK") ? atoi(getenv("LOPC_FAULT_RANK")) : -1;
  static const int fk = getenv("LOPC_FAULT_ROUND") ? atoi(getenv("LOPC_FAULT_ROUND")) : -1;
  return fr >= 0 && fk >= 0 && rank == fr && round == fk;
}

}  // namespace

struct lopc_comm {
  int world, rank;
  ncclComm_t comm;
};

extern "C" {

int lopc_comm_unique_id(void* id128) {
  if (!id128) return LOPC_E_ARG;
  int rc = nccl_load();
  if (rc) return rc;
  ncclUniqueId id;
  NK(g_nccl.GetUniqueId(&id));
  memcpy(id128, &id, sizeof(id));
  return LOPC_OK;
}

int lopc_comm_create(lopc_comm** comm, int world, int rank, const void* id128) {
  if (!comm || !id128 || world < 1 || rank < 0 || rank >= world) return LOPC_E_ARG;
  int rc = nccl_load();
  if (rc) return rc;
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  lopc_comm* c = new lopc_comm{world, rank, nullptr};
  ncclResult_t r = g_nccl.CommInitRank(&c->comm, world, id, rank);
  if (r != ncclSuccess) {
    snprintf(g_errmsg, sizeof(g_errmsg), "ncclCommInitRank: %s", g_nccl.GetErrorString(r));
    delete c;
    return LOPC_E_NCCL;
  }
  *comm = c;
  return LOPC_OK;
}

int lopc_comm_destroy(lopc_comm* comm) {
  if (!comm) return LOPC_OK;
  if (comm->comm) g_nccl.CommDestroy(comm->comm);
  delete comm;
  return LOPC_OK;
}

int lopc_slab_partition(int ndims, const uint64_t* dims, int dtype, int world, uint64_t* bounds) {
  Shape g;
  int rc = make_shape(ndims, dims, dtype, g);
  if (rc) return rc;
  if (world < 1 || !bounds) return LOPC_E_ARG;
  const uint64_t W = kChunkBytes / g.k;
  for (int r = 0; r <= world; ++r) {
    const uint64_t c = (g.C * (uint64_t)r) / (uint64_t)world;  // chunk-balanced split
    bounds[r] = c * W < g.n ? c * W : g.n;
  }
  for (int r = 0; r < world; ++r) {
    SlabGeo s;
    if (bounds[r] >= bounds[r + 1] || slab_geo(g, bounds[r], bounds[r + 1], r > 0, r + 1 < world, s))
      return LOPC_E_SHAPE;
  }
  return LOPC_OK;
}

int lopc_slab_info(int ndims, const uint64_t* dims, int dtype, uint64_t e_begin, uint64_t e_end, int has_lo,
                   int has_hi, uint64_t* info8) {
  Shape g;
  int rc = make_shape(ndims, dims, dtype, g);
  if (rc) return rc;
  SlabGeo s;
  if ((rc = slab_geo(g, e_begin, e_end, has_lo != 0, has_hi != 0, s))) return rc;
  if (info8) {
    const uint64_t v[8] = {s.B0, s.box.n, s.H, s.glo, s.ghi, s.send_lo, s.send_hi, s.C_local};
    memcpy(info8, v, sizeof(v));
  }
  return LOPC_OK;
}

size_t lopc_slab_workspace_bytes(int ndims, const uint64_t* dims, int dtype, uint64_t e_begin, uint64_t e_end) {
  Shape g;
  if (make_shape(ndims, dims, dtype, g)) return 0;
  SlabGeo s;
  if (slab_geo(g, e_begin, e_end, true, true, s)) {
    if (slab_geo(g, e_begin, e_end, false, false, s)) return 0;
  }
  return slab_layout(s).total;
}

size_t lopc_slab_bound(int ndims, const uint64_t* dims, int dtype, uint64_t e_begin, uint64_t e_end) {
  Shape g;
  if (make_shape(ndims, dims, dtype, g) || e_end <= e_begin) return 0;
  const uint64_t W = kChunkBytes / g.k;
  const uint64_t C = (e_end - e_begin + W - 1) / W;
  return 8 * C + 2ull * kChunkBytes * C;
}

int lopc_write_header(void* hdr64, int ndims, const uint64_t* dims, int dtype, double eps, uint64_t total_bytes) {
  Shape g;
  int rc = make_shape(ndims, dims, dtype, g);
  if (rc) return rc;
  if (!hdr64) return LOPC_E_ARG;
  write_header_host(static_cast<uint8_t*>(hdr64), g, eps, total_bytes);
  return LOPC_OK;
}

constexpr int kSlabRetryU32 = -1000;  // internal (never returned): a subbin above 8 planes on some rank

int compress_slab_impl(lopc_comm* comm, const void* in_slab, int ndims, const uint64_t* dims, int dtype, double eps,
                       uint64_t e_begin, uint64_t e_end, void* out_local, size_t* out_local_bytes,
                       uint64_t* payload_offset, uint64_t* total_bytes, void* workspace, size_t workspace_bytes,
                       void* stream, bool tiles) {
  if (!in_slab || !out_local || !out_local_bytes) return LOPC_E_ARG;
  Shape g;
  int rc = make_shape(ndims, dims, dtype, g);
  if (rc) return rc;
  if ((rc = check_eps(eps))) return rc;
  if (!is_device_ptr(in_slab) || !is_device_ptr(out_local)) return LOPC_E_ARG;
  const int world = comm ? comm->world : 1, rank = comm ? comm->rank : 0;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // every rank checks the global partition (allgather of the ranges), so
  // that all ranks return the same code
  uint64_t* dscratch = nullptr;
  Slab sl{};
  rc = slab_geo(g, e_begin, e_end, rank > 0, rank + 1 < world, sl.geo);
  sl.lay = slab_layout(sl.geo);
  if (!rc && (!workspace || workspace_bytes < sl.lay.total)) rc = LOPC_E_NOSPACE;
  Counters* hc;
  int rc2;
  if ((rc2 = host_ctr(hc))) return rc2;
  g_stats = lopc_stats{};
  g_stats.n_elems = g.n;
  g_stats.n_chunks = g.C;
  if (world > 1) {
    // status exchange: (rc, e_begin, e_end) of every rank
    if (!workspace || workspace_bytes < 24ull * (world + 1)) return LOPC_E_NOSPACE;  // cannot even talk
    if (world > 680) return LOPC_E_ARG;
    dscratch = reinterpret_cast<uint64_t*>(static_cast<uint8_t*>(workspace) + (rc ? 0 : sl.lay.ctr_sum));
    std::vector<uint64_t> mine = {(uint64_t)err_rank(rc), e_begin, e_end}, all(3 * world);
    CK(cudaMemcpyAsync(dscratch, mine.data(), 24, cudaMemcpyHostToDevice, st));
    NK(g_nccl.AllGather(dscratch, dscratch + 3, 3, ncclUint64, comm->comm, st));
    CK(cudaMemcpyAsync(all.data(), dscratch + 3, 24ull * world, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    uint64_t worst = 0;
    for (int r = 0; r < world; ++r) {
      worst = all[3 * r] > worst ? all[3 * r] : worst;
      const uint64_t b = all[3 * r + 1], e = all[3 * r + 2];
      if ((r == 0 && b != 0) || (r + 1 == world && e != g.n) || (r + 1 < world && e != all[3 * (r + 1) + 1]))
        worst = worst > (uint64_t)-LOPC_E_SHAPE ? worst : (uint64_t)-LOPC_E_SHAPE;
    }
    if (worst) return -(int)worst;
  } else {
    if (rc) return rc;
    if (e_begin != 0 || e_end != g.n) return LOPC_E_SHAPE;
  }
  sl.ws = static_cast<uint8_t*>(workspace);
  sl.x_own = in_slab;
  sl.eps = eps;
  sl.st = st;
  sl.tiles = tiles;
  Timer tm;
  if ((rc = tm.init(st))) return rc;
  tm.mark();  // 0
  if ((rc = sl.setup())) return rc;
  const SlabGeo& G = sl.geo;
  const int lo = rank - 1, hi = rank + 1;
  auto halo = [&](uint8_t* base, size_t esz, ncclDataType_t dt) -> int {
    NK(g_nccl.GroupStart());
    if (G.send_lo) NK(g_nccl.Send(sl.send_lo_ptr(base, esz), G.send_lo * esz / (dt == ncclUint8 ? 1 : esz), dt, lo,
                                  comm->comm, st));
    if (G.glo) NK(g_nccl.Recv(sl.recv_lo(), G.glo * esz / (dt == ncclUint8 ? 1 : esz), dt, lo, comm->comm, st));
    if (G.send_hi) NK(g_nccl.Send(sl.send_hi_ptr(base, esz), G.send_hi * esz / (dt == ncclUint8 ? 1 : esz), dt, hi,
                                  comm->comm, st));
    if (G.ghi) NK(g_nccl.Recv(sl.recv_hi(), G.ghi * esz / (dt == ncclUint8 ? 1 : esz), dt, hi, comm->comm, st));
    NK(g_nccl.GroupEnd());
    return LOPC_OK;
  };
  if (world > 1) {  // x halo, once
    if ((rc = halo(sl.xbox(), g.k, ncclUint8))) return rc;
    if (G.glo) CK(cudaMemcpyAsync(sl.ghost_lo_ptr(sl.xbox(), g.k), sl.recv_lo(), G.glo * g.k, cudaMemcpyDeviceToDevice, st));
    if (G.ghi) CK(cudaMemcpyAsync(sl.ghost_hi_ptr(sl.xbox(), g.k), sl.recv_hi(), G.ghi * g.k, cudaMemcpyDeviceToDevice, st));
  }
  tm.mark();  // 1
  // From here on every rank takes part in every collective of the schedule
  // whatever happens locally: a local failure (lrc) skips this rank's work,
  // is summed into the round's allreduce (all ranks leave the loop together)
  // and reaches every rank's return code through the final allgather.  Only
  // a failing NCCL call itself returns at once (the communicator is then
  // unusable; the caller must tear the job down).
  int lrc = launch_quant_flags(G.box, sl.ra, sl.lay.L, st);
  tm.mark();  // 2
  if (!lrc) lrc = sl.repair1();
  if (!lrc && fault_injected(rank, 0)) lrc = LOPC_E_INTERNAL;
  uint64_t rounds = 1;
  bool broke_on_failure = false;
  while (world > 1) {
    if (!lrc) lrc = sl.widen_send();
    if ((rc = halo(reinterpret_cast<uint8_t*>(sl.s()), 4, ncclUint32))) return rc;
    if (!lrc) lrc = sl.inject();
    if (!lrc && fault_injected(rank, (int)rounds)) lrc = LOPC_E_INTERNAL;
    // round agreement: sum over ranks of (ghosts raised, local failures)
    uint64_t* sum = reinterpret_cast<uint64_t*>(sl.ws + sl.lay.ctr_sum);  // [0, 1] in, [2, 3] out
    // (a device-side error bit of this rank, e.g. kErrPlanes, counts as a failure too)
    if (cudaMemcpyAsync(sum, &sl.dctr()->ghost_changed, 8, cudaMemcpyDeviceToDevice, st) != cudaSuccess ||
        cudaMemsetAsync(sum + 1, 0, 8, st) != cudaSuccess ||
        cudaMemcpyAsync(sum + 1, &sl.dctr()->err, 4, cudaMemcpyDeviceToDevice, st) != cudaSuccess ||
        (lrc && cudaMemsetAsync(sum + 1, 1, 1, st) != cudaSuccess))
      lrc = lrc ? lrc : LOPC_E_CUDA;
    NK(g_nccl.AllReduce(sum, sum + 2, 2, ncclUint64, ncclSum, comm->comm, st));
    uint64_t hs[2] = {0, 1};
    if (cudaMemcpyAsync(hs, sum + 2, 16, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return set_cuda_error(cudaGetLastError(), "slab round agreement");
    if (hs[1] != 0) {  // some rank failed: everyone stops here
      // (the failing rank's own code reaches every rank through the final
      // allgather; a rank whose trouble is a device error bit reports it there)
      broke_on_failure = true;
      break;
    }
    if (hs[0] == 0) break;
    if (!lrc) lrc = sl.sweep_sparse();
    ++rounds;
  }
  tm.mark();  // 3
  if (!lrc) lrc = sl.encode(static_cast<uint8_t*>(out_local), *out_local_bytes, &tm);  // mark 4
  tm.mark();  // 5
  CK(cudaMemcpyAsync(hc, sl.dctr(), sizeof(Counters), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (tm.on) {
    g_stats.timing_valid = 1;
    g_stats.ms_quant_repair = tm.ms(1, 2);
    g_stats.ms_sweep = tm.ms(2, 3);  // all repair rounds, halo exchanges included
    g_stats.ms_encode = tm.ms(3, 4);
    g_stats.ms_place = tm.ms(4, 5);
    g_stats.ms_total = tm.ms(0, 5);
  }
  uint32_t herr = hc->err;
  if (hc->passes >= (unsigned long long)sl.ra.max_passes && hc->list_count[(hc->passes + 1) % 3] != 0)
    herr |= kErrPassCap;  // a repair that did not converge is never encoded silently
  int local = lrc ? lrc : map_err(herr & ~kErrNoSpace);
  if (!lrc && (herr & kErrPlanes)) local = kSlabRetryU32;  // every rank re-runs on the u32 engine
  if (!local && world > 1 && broke_on_failure) local = LOPC_E_INTERNAL;  // another rank failed
  uint64_t mine[2] = {hc->total_bytes, (uint64_t)err_rank(local)};
  std::vector<uint64_t> all(2 * world);
  if (world > 1) {
    uint64_t* d = reinterpret_cast<uint64_t*>(sl.ws + sl.lay.ctr_sum);
    CK(cudaMemcpyAsync(d, mine, 16, cudaMemcpyHostToDevice, st));
    NK(g_nccl.AllGather(d, d + 2, 2, ncclUint64, comm->comm, st));
    CK(cudaMemcpyAsync(all.data(), d + 2, 16ull * world, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  } else {
    all[0] = mine[0];
    all[1] = mine[1];
  }
  uint64_t off = kHdrBytes + 8 * g.C, worst = 0;
  for (int r = 0; r < world; ++r) {
    if (r == rank) *payload_offset = off;
    off += all[2 * r];
    worst = all[2 * r + 1] > worst ? all[2 * r + 1] : worst;
  }
  if (total_bytes) *total_bytes = off;
  g_stats.sweep_passes = hc->passes;
  g_stats.max_subbin = hc->max_s;
  g_stats.bin_bytes = hc->bin_bytes;
  g_stats.sub_bytes = hc->sub_bytes;
  g_stats.total_bytes = off;
  g_stats.inner_iters = rounds;  // slab mode: repair rounds (halo exchanges + 1)
  // quant_flags + repair, per further round: (tiles: 2 boundary widens +) up
  // to 2 injections + repair; 2 encoder grids, scan, place
  g_stats.launches = (uint32_t)(2 + (tiles ? 5 : 3) * (rounds - 1) + 2 + 2);
  const uint64_t need = 8 * G.C_local + mine[0];
  if (worst == (uint64_t)-kSlabRetryU32) return kSlabRetryU32;
  if (worst) {
    if (-(int)worst == LOPC_E_NOSPACE) *out_local_bytes = need;  // lopc.h: NOSPACE reports the size needed
    return -(int)worst;
  }
  if (need > *out_local_bytes) {
    *out_local_bytes = need;
    return LOPC_E_NOSPACE;
  }
  *out_local_bytes = need;
  return LOPC_OK;
}

int lopc_compress_slab(lopc_comm* comm, const void* in_slab, int ndims, const uint64_t* dims, int dtype, double eps,
                       uint64_t e_begin, uint64_t e_end, void* out_local, size_t* out_local_bytes,
                       uint64_t* payload_offset, uint64_t* total_bytes, void* workspace, size_t workspace_bytes,
                       void* stream) {
  const size_t cap = out_local_bytes ? *out_local_bytes : 0;
  int rc = compress_slab_impl(comm, in_slab, ndims, dims, dtype, eps, e_begin, e_end, out_local, out_local_bytes,
                              payload_offset, total_bytes, workspace, workspace_bytes, stream, g_engine == 0);
  if (rc == kSlabRetryU32) {  // agreed by every rank: a subbin above 8 planes somewhere
    *out_local_bytes = cap;
    rc = compress_slab_impl(comm, in_slab, ndims, dims, dtype, eps, e_begin, e_end, out_local, out_local_bytes,
                            payload_offset, total_bytes, workspace, workspace_bytes, stream, false);
  }
  return rc;
}

// Single-device test hook: the slab algorithm over `nslabs` ranges in one
// call, with the halo exchanges done by device copies between the slabs.
// Writes the whole stream.  Allocates its own workspaces (diagnostic only).
int compress_slabs_local_impl(const void* in, int ndims, const uint64_t* dims, int dtype, double eps, int nslabs,
                              const uint64_t* bounds, void* out, size_t* out_bytes, bool tiles) {
  if (!in || !out || !out_bytes || !bounds || nslabs < 1) return LOPC_E_ARG;
  Shape g;
  int rc = make_shape(ndims, dims, dtype, g);
  if (rc) return rc;
  if ((rc = check_eps(eps))) return rc;
  if (!is_device_ptr(in) || !is_device_ptr(out)) return LOPC_E_ARG;
  if (bounds[0] != 0 || bounds[nslabs] != g.n) return LOPC_E_SHAPE;
  std::vector<Slab> sl(nslabs);
  std::vector<void*> mem;
  auto cleanup = [&]() {
    for (void* p : mem) cudaFree(p);
  };
  cudaStream_t st = nullptr;
  for (int r = 0; r < nslabs; ++r) {
    if ((rc = slab_geo(g, bounds[r], bounds[r + 1], r > 0, r + 1 < nslabs, sl[r].geo))) {
      cleanup();
      return rc;
    }
    sl[r].lay = slab_layout(sl[r].geo);
    void* w = nullptr;
    if (cudaMalloc(&w, sl[r].lay.total) != cudaSuccess) {
      cleanup();
      return LOPC_E_CUDA;
    }
    mem.push_back(w);
    sl[r].ws = static_cast<uint8_t*>(w);
    sl[r].x_own = static_cast<const uint8_t*>(in) + g.k * bounds[r];
    sl[r].eps = eps;
    sl[r].st = st;
    sl[r].tiles = tiles;
    if ((rc = sl[r].setup())) {
      cleanup();
      return rc;
    }
  }
  auto exchange = [&](bool xs) -> int {
    const size_t esz = xs ? g.k : 4;
    for (int r = 0; r < nslabs; ++r) {
      Slab& a = sl[r];
      uint8_t* base_lo = r > 0 ? (xs ? sl[r - 1].xbox() : reinterpret_cast<uint8_t*>(sl[r - 1].s())) : nullptr;
      uint8_t* base_hi = r + 1 < nslabs ? (xs ? sl[r + 1].xbox() : reinterpret_cast<uint8_t*>(sl[r + 1].s())) : nullptr;
      if (a.geo.glo) CK(cudaMemcpyAsync(a.recv_lo(), sl[r - 1].send_hi_ptr(base_lo, esz), a.geo.glo * esz, cudaMemcpyDeviceToDevice, st));
      if (a.geo.ghi) CK(cudaMemcpyAsync(a.recv_hi(), sl[r + 1].send_lo_ptr(base_hi, esz), a.geo.ghi * esz, cudaMemcpyDeviceToDevice, st));
    }
    return LOPC_OK;
  };
  if (nslabs > 1) {
    if ((rc = exchange(true))) { cleanup(); return rc; }
    for (auto& a : sl) {
      if (a.geo.glo) CK(cudaMemcpyAsync(a.ghost_lo_ptr(a.xbox(), g.k), a.recv_lo(), a.geo.glo * g.k, cudaMemcpyDeviceToDevice, st));
      if (a.geo.ghi) CK(cudaMemcpyAsync(a.ghost_hi_ptr(a.xbox(), g.k), a.recv_hi(), a.geo.ghi * g.k, cudaMemcpyDeviceToDevice, st));
    }
  }
  for (auto& a : sl)
    if ((rc = a.round1())) { cleanup(); return rc; }
  uint64_t rounds = 1;
  Counters* hc;
  if ((rc = host_ctr(hc))) { cleanup(); return rc; }
  while (nslabs > 1) {
    for (auto& a : sl)
      if ((rc = a.widen_send())) { cleanup(); return rc; }
    if ((rc = exchange(false))) { cleanup(); return rc; }
    for (auto& a : sl)
      if ((rc = a.inject())) { cleanup(); return rc; }
    uint64_t changed = 0;
    uint32_t errs = 0;
    for (auto& a : sl) {
      uint64_t v = 0;
      uint32_t e = 0;
      CK(cudaMemcpyAsync(&v, &a.dctr()->ghost_changed, 8, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(&e, &a.dctr()->err, 4, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      changed += v;
      errs |= e;
    }
    if (errs & kErrPlanes) {
      cleanup();
      return kSlabRetryU32;
    }
    if (!changed) break;
    for (auto& a : sl)
      if ((rc = a.sweep_sparse())) { cleanup(); return rc; }
    ++rounds;
  }
  // encode each slab into a scratch area, then assemble header ‖ tables ‖ payloads
  const size_t cap = *out_bytes;
  uint64_t off = kHdrBytes + 8 * g.C, worst = 0;
  std::vector<uint64_t> pay(nslabs);
  std::vector<void*> locals(nslabs);
  uint64_t max_s = 0;
  for (int r = 0; r < nslabs; ++r) {
    const size_t lcap = 8 * sl[r].geo.C_local + 2ull * kChunkBytes * sl[r].geo.C_local;
    if (cudaMalloc(&locals[r], lcap) != cudaSuccess) { cleanup(); return LOPC_E_CUDA; }
    mem.push_back(locals[r]);
    if ((rc = sl[r].encode(static_cast<uint8_t*>(locals[r]), lcap))) { cleanup(); return rc; }
    CK(cudaMemcpyAsync(hc, sl[r].dctr(), sizeof(Counters), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    pay[r] = hc->total_bytes;
    if (hc->err & kErrPlanes) {
      cleanup();
      return kSlabRetryU32;
    }
    worst = (uint64_t)err_rank(map_err(hc->err)) > worst ? (uint64_t)err_rank(map_err(hc->err)) : worst;
    max_s = hc->max_s > max_s ? hc->max_s : max_s;
  }
  uint64_t total = off;
  for (int r = 0; r < nslabs; ++r) total += pay[r];
  if (worst) { cleanup(); return -(int)worst; }
  if (total > cap) {
    *out_bytes = total;
    cleanup();
    return LOPC_E_NOSPACE;
  }
  uint8_t h[kHdrBytes];
  write_header_host(h, g, eps, total);
  uint8_t* o = static_cast<uint8_t*>(out);
  CK(cudaMemcpyAsync(o, h, kHdrBytes, cudaMemcpyHostToDevice, st));
  uint64_t toff = kHdrBytes;
  for (int r = 0; r < nslabs; ++r) {
    const uint64_t tb = 8 * sl[r].geo.C_local;
    CK(cudaMemcpyAsync(o + toff, locals[r], tb, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(o + off, static_cast<uint8_t*>(locals[r]) + tb, pay[r], cudaMemcpyDeviceToDevice, st));
    toff += tb;
    off += pay[r];
  }
  CK(cudaStreamSynchronize(st));
  g_stats = lopc_stats{};
  g_stats.n_elems = g.n;
  g_stats.n_chunks = g.C;
  g_stats.total_bytes = total;
  g_stats.inner_iters = rounds;
  g_stats.max_subbin = (uint32_t)max_s;
  *out_bytes = total;
  cleanup();
  return LOPC_OK;
}

int lopc_compress_slabs_local(const void* in, int ndims, const uint64_t* dims, int dtype, double eps, int nslabs,
                              const uint64_t* bounds, void* out, size_t* out_bytes) {
  const size_t cap = out_bytes ? *out_bytes : 0;
  int rc = compress_slabs_local_impl(in, ndims, dims, dtype, eps, nslabs, bounds, out, out_bytes, g_engine == 0);
  if (rc == kSlabRetryU32) {
    *out_bytes = cap;
    rc = compress_slabs_local_impl(in, ndims, dims, dtype, eps, nslabs, bounds, out, out_bytes, false);
  }
  return rc;
}

size_t lopc_decompress_slab_workspace_bytes(uint64_t n_chunks_local) {
  return al(sizeof(Counters)) + al(8 * (n_chunks_local / kScanTile + 1)) + al(8 * n_chunks_local) + al(64);
}

int lopc_decompress_slab(const void* hdr64_host, const void* local, size_t local_bytes, uint64_t e_begin,
                         uint64_t e_end, void* out_slab, size_t out_capacity, void* workspace, size_t workspace_bytes,
                         void* stream) {
  if (!hdr64_host || !local || !out_slab) return LOPC_E_ARG;
  int nd, dt;
  uint64_t d3[3], n;
  double eps;
  uint32_t C;
  int rc = lopc_stream_info(hdr64_host, kHdrBytes, &nd, d3, &dt, &eps, &n, &C);
  if (rc) return rc;
  if (!is_device_ptr(local) || !is_device_ptr(out_slab)) return LOPC_E_ARG;
  const uint64_t k = dt ? 8 : 4, W = kChunkBytes / k;
  if (e_begin >= e_end || e_end > n || e_begin % W || (e_end != n && e_end % W)) return LOPC_E_SHAPE;
  if ((uint64_t)C != (n + W - 1) / W) return LOPC_E_CORRUPT;
  const uint64_t CL = (e_end - e_begin + W - 1) / W;
  if (out_capacity < k * (e_end - e_begin)) return LOPC_E_NOSPACE;
  if (local_bytes < 8 * CL) return LOPC_E_CORRUPT;
  if (!workspace || workspace_bytes < lopc_decompress_slab_workspace_bytes(CL)) return LOPC_E_NOSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  const size_t o_state = al(sizeof(Counters)), o_off = o_state + al(8 * (CL / kScanTile + 1));
  CK(cudaMemsetAsync(ws, 0, o_off, st));
  Counters* hc;
  if ((rc = host_ctr(hc))) return rc;
  DevInfo* di;
  if ((rc = dev_info(di))) return rc;
  const uint8_t* src = static_cast<const uint8_t*>(local);
  ScanArgs sa{};
  sa.sizes = reinterpret_cast<const uint32_t*>(src);
  sa.C = (uint32_t)CL;
  sa.off = reinterpret_cast<uint64_t*>(ws + o_off);
  sa.state = reinterpret_cast<uint64_t*>(ws + o_state);
  sa.ctr = reinterpret_cast<Counters*>(ws);
  sa.validate = 1;
  sa.expect_total = local_bytes;
  sa.base = 8 * CL;
  Timer tm;
  if ((rc = tm.init(st))) return rc;
  tm.mark();  // 0
  k_chunk_scan<<<(unsigned)((CL + kScanTile - 1) / kScanTile), kScanThreads, 0, st>>>(sa);
  CK(cudaGetLastError());
  tm.mark();  // 1
  DecodeArgs da{};
  da.in = src;
  da.in_bytes = local_bytes;
  da.out = static_cast<uint8_t*>(out_slab) - k * e_begin;  // chunk c (global) at out + c W
  da.out_cap = out_capacity;
  da.off = sa.off;
  da.table = sa.sizes;
  da.base = src;
  da.c_begin = e_begin / W;
  da.c_count = CL;
  da.state_cap = CL;
  da.ctr = sa.ctr;
  da.slab = 1;
  da.given.dtype = dt;
  da.given.ndims = nd;
  da.given.d0 = d3[0];
  da.given.d1 = d3[1];
  da.given.d2 = d3[2];
  da.given.n = e_end;  // the last chunk of this slice ends at e_end
  da.given.eps = eps;
  da.given.C = C;
  da.given.ok = true;
  da.given.err = 0;
  if ((rc = launch_decode(di, da, CL, st))) return rc;
  tm.mark();  // 2
  CK(cudaMemcpyAsync(hc, ws, sizeof(Counters), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  g_stats = lopc_stats{};
  g_stats.launches = 2;
  if (tm.on) {
    g_stats.timing_valid = 1;
    g_stats.ms_place = tm.ms(0, 1);
    g_stats.ms_decode = tm.ms(1, 2);
    g_stats.ms_total = tm.ms(0, 2);
  }
  return map_err(hc->err);
}

}  // extern "C"
