// Cross-rank transport of the strip-partitioned PCG: one PCG iteration
// needs (a) halo exchanges of the smoother iterate z after every colour phase and after the
// prolongation (one node column per neighbour and realisation) and (b) sum all-reduces of
// the dot products and of the chain-end coarse rhs (K_c is distributed by block chains; the
// interface system is replicated).  The assembly all-reduces the interface blocks of K_c.
//
//   MSF_TRANSPORT_NCCL : one process per GPU; NCCL send/recv + all-reduce on the context's
//                        stream (captured into the per-iteration CUDA graph).  libnccl is
//                        loaded at run time (dlopen), so the library links without it.
//   MSF_TRANSPORT_GROUP: every rank of the group lives in this process on one device; the
//                        host drives all ranks phase by phase on one stream, halos are
//                        device-to-device copies and the all-reduce is one kernel that sums
//                        the ranks' buffers in rank order.  Used to prove the partitioned
//                        path equal to the single-GPU one on a single B200.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>

#include "msf_internal.cuh"

#include <algorithm>

#define MSF_MAX_GROUP 8

struct msf_group {
  int n = 0;
  std::vector<msf_ctx*> ranks;
};

namespace {

struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi load_nccl() {
  NcclApi a;
  // the soname resolves to an already-loaded libnccl (e.g. torch's) before the system copy
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    a.err = std::string("cannot load libnccl: ") + dlerror();
    return a;
  }
#define MSF_SYM(field, name)                                     \
  a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, name)); \
  if (!a.field) {                                                \
    a.err = std::string("libnccl lacks ") + name;                \
    return a;                                                    \
  }
  MSF_SYM(GetUniqueId, "ncclGetUniqueId");
  MSF_SYM(CommInitRank, "ncclCommInitRank");
  MSF_SYM(CommDestroy, "ncclCommDestroy");
  MSF_SYM(AllReduce, "ncclAllReduce");
  MSF_SYM(Send, "ncclSend");
  MSF_SYM(Recv, "ncclRecv");
  MSF_SYM(GroupStart, "ncclGroupStart");
  MSF_SYM(GroupEnd, "ncclGroupEnd");
  MSF_SYM(GetErrorString, "ncclGetErrorString");
#undef MSF_SYM
  a.ok = true;
  return a;
}

NcclApi& nccl() {
  static NcclApi a = load_nccl();
  return a;
}

int nccl_check(msf_ctx* c, ncclResult_t r, const char* where) {
  if (r == ncclSuccess) return MSF_OK;
  return msf_fail(c, MSF_ERR_CUDA, std::string(where) + ": " + nccl().GetErrorString(r));
}

struct GroupPtrs {
  double* p[MSF_MAX_GROUP];
  int n;
};

// in-place sum over the group's buffers, fixed rank order, result written to every rank
__global__ void k_group_sum(GroupPtrs g, size_t count) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < g.n; ++r) s += g.p[r][i];
    for (int r = 0; r < g.n; ++r) g.p[r][i] = s;
  }
}

}  // namespace

// ---------------------------------------------------------------------- strip geometry
int strip_bounds(const Dims& d, int rank, int nranks, StripBounds& b, std::string& msg) {
  if (nranks < 1 || rank < 0 || rank >= nranks) {
    msg = "rank out of range";
    return MSF_ERR_ARG;
  }
  if (nranks > d.ncx) {
    msg = "more ranks than coarse columns (need ncx >= nranks)";
    return MSF_ERR_ARG;
  }
  b.C0 = (int)((long long)rank * d.ncx / nranks);
  b.C1 = (int)((long long)(rank + 1) * d.ncx / nranks);
  b.own0 = b.C0 * d.cx;
  b.own1 = (rank == nranks - 1) ? d.nelx + 1 : b.C1 * d.cx;
  b.e0 = b.C0 * d.cx;
  b.e1 = b.C1 * d.cx;
  // wide halos (streaming sweep) when every strip is at least that wide: a halo then lies
  // wholly inside the neighbouring strip
  int minw = d.nelx + 1;
  for (int r = 0; r < nranks; ++r) {
    const int c0 = (int)((long long)r * d.ncx / nranks), c1 = (int)((long long)(r + 1) * d.ncx / nranks);
    minw = std::min(minw, (c1 - c0) * d.cx);
  }
  b.halo = (nranks > 1 && minw >= MSF_STRIP_HALO) ? MSF_STRIP_HALO : 1;
  int lo = 0;
  if (rank > 0) lo = ((b.own0 - b.halo) % 2 == 0) ? b.own0 - b.halo : b.own0 - b.halo - 1;  // even: same colours
  const int hi = (rank == nranks - 1) ? d.nelx + 1 : b.own1 + b.halo;
  b.gox = lo;
  b.ncols = hi - lo;
  return MSF_OK;
}

// ---------------------------------------------------------------------- transport
int dist_comm_create(msf_ctx* c, int transport, void* handle) {
  msf_comm* m = new msf_comm();
  m->kind = transport;
  if (transport == MSF_TRANSPORT_NCCL) {
    NcclApi& A = nccl();
    if (!A.ok) {
      delete m;
      return msf_fail(c, MSF_ERR_CUDA, A.err);
    }
    ncclUniqueId id;
    std::memcpy(&id, handle, sizeof(id));
    ncclComm_t comm = nullptr;
    ncclResult_t r = A.CommInitRank(&comm, c->nranks, id, c->rank);
    if (r != ncclSuccess) {
      delete m;
      return nccl_check(c, r, "ncclCommInitRank");
    }
    m->nccl = comm;
  } else if (transport == MSF_TRANSPORT_GROUP) {
    msf_group* g = (msf_group*)handle;
    if (g->n != c->nranks) {
      delete m;
      return msf_fail(c, MSF_ERR_ARG, "group size differs from nranks");
    }
    if (g->ranks[c->rank]) {
      delete m;
      return msf_fail(c, MSF_ERR_ARG, "group rank already registered");
    }
    g->ranks[c->rank] = c;
    m->grp = g;
  } else {
    delete m;
    return msf_fail(c, MSF_ERR_ARG, "unknown transport");
  }
  c->comm = m;
  return MSF_OK;
}

void dist_comm_destroy(msf_ctx* c) {
  if (!c->comm) return;
  if (c->comm->kind == MSF_TRANSPORT_NCCL && c->comm->nccl)
    nccl().CommDestroy((ncclComm_t)c->comm->nccl);
  if (c->comm->grp) c->comm->grp->ranks[c->rank] = nullptr;
  delete c->comm;
  c->comm = nullptr;
}

// sum all-reduce of count doubles at (ctx->*buf) + off over the ranks this process drives
int dist_allreduce(const std::vector<msf_ctx*>& cs, double* msf_ctx::*buf, size_t off,
                   size_t count) {
  msf_ctx* c0 = cs[0];
  if (c0->comm->kind == MSF_TRANSPORT_NCCL) {
    double* p = c0->*buf + off;
    return nccl_check(c0, nccl().AllReduce(p, p, count, ncclDouble, ncclSum,
                                           (ncclComm_t)c0->comm->nccl, c0->stream),
                      "ncclAllReduce");
  }
  GroupPtrs g{};
  g.n = (int)cs.size();
  for (int r = 0; r < g.n; ++r) g.p[r] = cs[r]->*buf + off;
  int blocks = (int)std::min<size_t>((count + 255) / 256, 592);
  k_group_sum<<<blocks > 0 ? blocks : 1, 256, 0, c0->stream>>>(g, count);
  MSF_LAUNCHED(c0);
  return msf_cuda_check(c0, cudaGetLastError(), "group all-reduce");
}

// halo exchange of the node vector ctx->*vec for realisations [rhs0, rhs0 + nr): every rank sends its
// first / last w owned node columns to the left / right neighbour's w halo columns
int dist_halo(const std::vector<msf_ctx*>& cs, double* msf_ctx::*vec, int rhs0, int nr, int w) {
  msf_ctx* c0 = cs[0];
  if (c0->comm->kind == MSF_TRANSPORT_NCCL) {
    NcclApi& A = nccl();
    msf_ctx* c = c0;
    const Dims& d = c->dl;
    const size_t col = (size_t)2 * d.nny;   // doubles per node column
    const size_t wc = (size_t)w * col;
    ncclComm_t comm = (ncclComm_t)c->comm->nccl;
    int rc = nccl_check(c, A.GroupStart(), "ncclGroupStart");
    if (rc) return rc;
    for (int k = rhs0; k < rhs0 + nr; ++k) {
      double* v = c->*vec + (size_t)k * 2 * d.nn;
      // every call is checked; on a failure the group is still closed before returning, so
      // the communicator is never left inside an open group
      if (c->rank > 0) {
        if (!rc) rc = nccl_check(c, A.Send(v + (size_t)d.own_lo * col, wc, ncclDouble, c->rank - 1, comm, c->stream), "ncclSend (halo, left)");
        if (!rc) rc = nccl_check(c, A.Recv(v + (size_t)(d.own_lo - w) * col, wc, ncclDouble, c->rank - 1, comm, c->stream), "ncclRecv (halo, left)");
      }
      if (c->rank < c->nranks - 1) {
        if (!rc) rc = nccl_check(c, A.Send(v + (size_t)(d.own_hi - w) * col, wc, ncclDouble, c->rank + 1, comm, c->stream), "ncclSend (halo, right)");
        if (!rc) rc = nccl_check(c, A.Recv(v + (size_t)d.own_hi * col, wc, ncclDouble, c->rank + 1, comm, c->stream), "ncclRecv (halo, right)");
      }
    }
    const int rce = nccl_check(c, A.GroupEnd(), "ncclGroupEnd (halo)");
    return rc ? rc : rce;
  }
  for (size_t r = 0; r + 1 < cs.size(); ++r) {
    msf_ctx* a = cs[r];
    msf_ctx* b = cs[r + 1];
    const size_t colb = (size_t)2 * a->dl.nny * sizeof(double);
    const size_t pa = (size_t)2 * a->dl.nn * sizeof(double), pb = (size_t)2 * b->dl.nn * sizeof(double);
    char* va = (char*)(a->*vec) + (size_t)rhs0 * pa;
    char* vb = (char*)(b->*vec) + (size_t)rhs0 * pb;
    // a's last w owned columns -> b's left halo ; b's first w owned columns -> a's right halo
    cudaError_t e = cudaMemcpy2DAsync(vb + (size_t)(b->dl.own_lo - w) * colb, pb,
                                      va + (size_t)(a->dl.own_hi - w) * colb, pa, w * colb, nr,
                                      cudaMemcpyDeviceToDevice, c0->stream);
    if (e == cudaSuccess)
      e = cudaMemcpy2DAsync(va + (size_t)a->dl.own_hi * colb, pa,
                            vb + (size_t)b->dl.own_lo * colb, pb, w * colb, nr,
                            cudaMemcpyDeviceToDevice, c0->stream);
    int rc = msf_cuda_check(c0, e, "group halo copy");
    if (rc) return rc;
  }
  return MSF_OK;
}

std::vector<msf_ctx*> group_ranks(msf_group* g) { return g->ranks; }

extern "C" {

int msf_nccl_unique_id(uint8_t* id) {
  if (!id) return msf_fail(nullptr, MSF_ERR_ARG, "id is null");
  NcclApi& A = nccl();
  if (!A.ok) return msf_fail(nullptr, MSF_ERR_CUDA, A.err);
  ncclUniqueId u;
  ncclResult_t r = A.GetUniqueId(&u);
  if (r != ncclSuccess) return msf_fail(nullptr, MSF_ERR_CUDA, std::string("ncclGetUniqueId: ") + A.GetErrorString(r));
  std::memcpy(id, &u, sizeof(u));
  return MSF_OK;
}

int msf_group_create(int nranks, msf_group** out) {
  if (!out) return msf_fail(nullptr, MSF_ERR_ARG, "out is null");
  *out = nullptr;
  if (nranks < 1 || nranks > MSF_MAX_GROUP) return msf_fail(nullptr, MSF_ERR_ARG, "group size must be 1..8");
  msf_group* g = new msf_group();
  g->n = nranks;
  g->ranks.assign(nranks, nullptr);
  *out = g;
  return MSF_OK;
}

int msf_group_destroy(msf_group* g) {
  if (!g) return MSF_OK;
  for (msf_ctx* c : g->ranks)
    if (c && c->comm) c->comm->grp = nullptr;
  delete g;
  return MSF_OK;
}

}  // extern "C"
