// fem_dist.cu — element-partitioned multi-GPU support: the interface-DOF halo
// add over NCCL and owned-DOF reductions.  Used only when fem_dist_desc.size > 1.
//
// halo add of a rank-local partial vector y (residual / HVP / SpMV):
//   pack     send[t][c]  = y[nbr_nodes[t]][c]          (segments per neighbour, ascending rank)
//   exchange grouped ncclSend / ncclRecv with every neighbour on the caller's stream
//   combine  y[n][c] = sum over the ranks touching n, in ascending rank order, of their
//            partials (own value or recv[t][c]) — identical bits on every rank.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <vector>

#include "fem_internal.cuh"

namespace fem {

__global__ void k_halo_pack(const double *y, const int32_t *nodes, int64_t n, int dim, double *send) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * dim;
       i += (int64_t)gridDim.x * blockDim.x)
    send[i] = y[(int64_t)nodes[i / dim] * dim + i % dim];
}

__global__ void k_halo_combine(double *y, const double *recv, const int32_t *hnodes, int64_t nh,
                               const int32_t *src_ptr, const int32_t *src, int dim) {
  for (int64_t h = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; h < nh;
       h += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = hnodes[h];
    double acc[3] = {0.0, 0.0, 0.0};
    for (int32_t q = src_ptr[h]; q < src_ptr[h + 1]; ++q) {
      const int32_t t = src[q];
      for (int c = 0; c < dim; ++c) acc[c] += (t < 0) ? y[n * dim + c] : recv[(int64_t)t * dim + c];
    }
    for (int c = 0; c < dim; ++c) y[n * dim + c] = acc[c];
  }
}

static fem_status nccl_status(ncclResult_t r, const char *what) {
  if (r == ncclSuccess) return FEM_OK;
  set_error(std::string(what) + ": " + ncclGetErrorString(r));
  return FEM_ERR_NCCL;
}

fem_status dist_setup(Problem *p, const fem_dist_desc *d, cudaStream_t s) {
  p->rank = d->rank;
  p->size = d->size;
  p->nccl = d->nccl_comm;
  FEM_ARG(d->n_nbr >= 0 && (d->n_nbr == 0 || (d->nbr_rank && d->nbr_offset && d->nbr_nodes)),
          "fem_dist_desc: bad neighbour arrays");
  FEM_ARG(d->owned != nullptr, "fem_dist_desc: owned[] required");
  p->n_nbr = d->n_nbr;
  p->nbr_rank_h.assign(d->nbr_rank, d->nbr_rank + d->n_nbr);
  p->nbr_off_h.assign(d->nbr_offset, d->nbr_offset + d->n_nbr + 1);
  const int64_t nt = p->nbr_off_h.empty() ? 0 : p->nbr_off_h.back();
  p->n_halo_entries = nt;
  for (int k = 0; k < d->n_nbr; ++k) {
    FEM_ARG(d->nbr_rank[k] >= 0 && d->nbr_rank[k] < d->size && d->nbr_rank[k] != d->rank,
            "fem_dist_desc: bad neighbour rank");
    FEM_ARG(k == 0 || d->nbr_rank[k] > d->nbr_rank[k - 1], "fem_dist_desc: nbr_rank not ascending");
  }
  // combine lists: per shared node, sources in ascending rank order (self = -1)
  std::vector<std::pair<int32_t, std::pair<int, int32_t>>> ent;  // (node, (rank, t))
  ent.reserve(nt * 2);
  for (int k = 0; k < d->n_nbr; ++k)
    for (int64_t t = d->nbr_offset[k]; t < d->nbr_offset[k + 1]; ++t) {
      const int32_t n = d->nbr_nodes[t];
      FEM_ARG(n >= 0 && n < p->n_nodes, "fem_dist_desc: nbr node out of range");
      ent.push_back({n, {d->nbr_rank[k], (int32_t)t}});
    }
  std::vector<int32_t> nodes;
  for (auto &x : ent) nodes.push_back(x.first);
  std::sort(nodes.begin(), nodes.end());
  nodes.erase(std::unique(nodes.begin(), nodes.end()), nodes.end());
  for (int32_t n : nodes) ent.push_back({n, {d->rank, -1}});
  std::sort(ent.begin(), ent.end());
  std::vector<int32_t> src_ptr(nodes.size() + 1, 0), src;
  size_t j = 0;
  for (size_t h = 0; h < nodes.size(); ++h) {
    while (j < ent.size() && ent[j].first == nodes[h]) src.push_back(ent[j++].second.second);
    src_ptr[h + 1] = (int32_t)src.size();
  }
  p->n_halo_nodes = (int64_t)nodes.size();
  const size_t hb = sizeof(double) * (size_t)std::max<int64_t>(nt, 1) * p->dim;
  FEM_CUDA(cudaMalloc(&p->halo_send_nodes, sizeof(int32_t) * std::max<int64_t>(nt, 1)));
  FEM_CUDA(cudaMalloc(&p->halo_nodes, sizeof(int32_t) * std::max<size_t>(nodes.size(), 1)));
  FEM_CUDA(cudaMalloc(&p->halo_src_ptr, sizeof(int32_t) * src_ptr.size()));
  FEM_CUDA(cudaMalloc(&p->halo_src, sizeof(int32_t) * std::max<size_t>(src.size(), 1)));
  FEM_CUDA(cudaMalloc(&p->sendbuf, hb));
  FEM_CUDA(cudaMalloc(&p->recvbuf, hb));
  FEM_CUDA(cudaMalloc(&p->owned, p->n_nodes));
  if (nt) FEM_CUDA(cudaMemcpyAsync(p->halo_send_nodes, d->nbr_nodes, sizeof(int32_t) * nt, cudaMemcpyHostToDevice, s));
  if (!nodes.empty()) {
    FEM_CUDA(cudaMemcpyAsync(p->halo_nodes, nodes.data(), sizeof(int32_t) * nodes.size(), cudaMemcpyHostToDevice, s));
    FEM_CUDA(cudaMemcpyAsync(p->halo_src, src.data(), sizeof(int32_t) * src.size(), cudaMemcpyHostToDevice, s));
  }
  FEM_CUDA(cudaMemcpyAsync(p->halo_src_ptr, src_ptr.data(), sizeof(int32_t) * src_ptr.size(), cudaMemcpyHostToDevice, s));
  FEM_CUDA(cudaMemcpyAsync(p->owned, d->owned, p->n_nodes, cudaMemcpyHostToDevice, s));
  std::vector<uint8_t> shared(p->n_nodes, 0);
  for (int32_t n : nodes) shared[n] = 1;
  FEM_CUDA(cudaMalloc(&p->shared, p->n_nodes > 0 ? p->n_nodes : 1));
  if (p->n_nodes) FEM_CUDA(cudaMemcpyAsync(p->shared, shared.data(), p->n_nodes, cudaMemcpyHostToDevice, s));
  FEM_CUDA(cudaStreamSynchronize(s));  // host vectors above go out of scope
  return FEM_OK;
}

void dist_free(Problem *p) {
  void *bufs[] = {p->halo_send_nodes, p->halo_nodes, p->halo_src_ptr, p->halo_src, p->sendbuf,
                  p->recvbuf, p->owned, p->shared};
  for (void *b : bufs)
    if (b) cudaFree(b);
  if (p->ev_part_a) cudaEventDestroy(p->ev_part_a);
  if (p->ev_halo) cudaEventDestroy(p->ev_halo);
  if (p->comm_stream) cudaStreamDestroy(p->comm_stream);
}

static fem_status halo_pack(Problem *p, const double *y, double *send, cudaStream_t s) {
  if (p->n_halo_entries)
    k_halo_pack<<<grid_for(p->n_halo_entries * p->dim), kThreads, 0, s>>>(y, p->halo_send_nodes, p->n_halo_entries, p->dim, send);
  FEM_LAUNCH_CHECK("halo pack");
  return FEM_OK;
}

static fem_status halo_combine(Problem *p, double *y, const double *recv, cudaStream_t s) {
  if (p->n_halo_nodes)
    k_halo_combine<<<grid_for(p->n_halo_nodes), kThreads, 0, s>>>(y, recv, p->halo_nodes, p->n_halo_nodes,
                                                                 p->halo_src_ptr, p->halo_src, p->dim);
  FEM_LAUNCH_CHECK("halo combine");
  return FEM_OK;
}

// pack + grouped send / recv of y's shared-node partials on stream cs
static fem_status halo_exchange(Problem *p, const double *y, cudaStream_t cs) {
  if (!p->nccl) {
    set_error("halo add needs an NCCL communicator (or FEM_LOCAL_ONLY + fem_halo_pack/combine)");
    return FEM_ERR_NCCL;
  }
  fem_status st = halo_pack(p, y, p->sendbuf, cs);
  if (st) return st;
  ncclComm_t comm = (ncclComm_t)p->nccl;
  const int D = p->dim;
  fem_status r = nccl_status(ncclGroupStart(), "ncclGroupStart");
  if (r) return r;
  for (int k = 0; k < p->n_nbr; ++k) {
    const int64_t off = p->nbr_off_h[k] * D, cnt = (p->nbr_off_h[k + 1] - p->nbr_off_h[k]) * D;
    r = nccl_status(ncclSend(p->sendbuf + off, (size_t)cnt, ncclDouble, p->nbr_rank_h[k], comm, cs), "ncclSend");
    if (r) return r;
    r = nccl_status(ncclRecv(p->recvbuf + off, (size_t)cnt, ncclDouble, p->nbr_rank_h[k], comm, cs), "ncclRecv");
    if (r) return r;
  }
  return nccl_status(ncclGroupEnd(), "ncclGroupEnd");
}

fem_status halo_add(Problem *p, double *y, cudaStream_t s) {
  if (p->size <= 1) return FEM_OK;
  fem_status st = halo_exchange(p, y, s);
  if (st) return st;
  return halo_combine(p, y, p->recvbuf, s);
}

// Overlapped form: called after the pass over the tiles that touch interface
// nodes, whose partials are then final.  The exchange runs on the problem's comm stream
// while the caller's stream computes the interior tiles; halo_end joins and combines.
fem_status halo_begin(Problem *p, const double *y, cudaStream_t s) {
  if (p->size <= 1) return FEM_OK;
  if (!p->comm_stream) {
    FEM_CUDA(cudaStreamCreateWithFlags(&p->comm_stream, cudaStreamNonBlocking));
    FEM_CUDA(cudaEventCreateWithFlags(&p->ev_part_a, cudaEventDisableTiming));
    FEM_CUDA(cudaEventCreateWithFlags(&p->ev_halo, cudaEventDisableTiming));
  }
  FEM_CUDA(cudaEventRecord(p->ev_part_a, s));
  FEM_CUDA(cudaStreamWaitEvent(p->comm_stream, p->ev_part_a, 0));
  fem_status st = halo_exchange(p, y, p->comm_stream);
  if (st) return st;
  FEM_CUDA(cudaEventRecord(p->ev_halo, p->comm_stream));
  return FEM_OK;
}

fem_status halo_end(Problem *p, double *y, cudaStream_t s) {
  if (p->size <= 1) return FEM_OK;
  FEM_CUDA(cudaStreamWaitEvent(s, p->ev_halo, 0));
  return halo_combine(p, y, p->recvbuf, s);
}

fem_status allreduce(Problem *p, double *buf, int n, cudaStream_t s) {
  if (p->size <= 1) return FEM_OK;
  if (!p->nccl) {
    set_error("all-reduce needs an NCCL communicator");
    return FEM_ERR_NCCL;
  }
  return nccl_status(ncclAllReduce(buf, buf, (size_t)n, ncclDouble, ncclSum, (ncclComm_t)p->nccl, s),
                     "ncclAllReduce");
}

}  // namespace fem

using namespace fem;

extern "C" {

fem_status fem_nccl_unique_id(unsigned char id[128]) {
  FEM_ARG(id, "fem_nccl_unique_id: null id");
  ncclUniqueId u;
  fem_status st = nccl_status(ncclGetUniqueId(&u), "ncclGetUniqueId");
  if (st) return st;
  static_assert(sizeof(u.internal) == 128, "ncclUniqueId size");
  for (int i = 0; i < 128; ++i) id[i] = (unsigned char)u.internal[i];
  return FEM_OK;
}

fem_status fem_nccl_comm_init(const unsigned char id[128], int rank, int size, void **comm) {
  FEM_NVTX_RANGE("fem_nccl_comm_init");
  FEM_ARG(id && comm && size > 0 && rank >= 0 && rank < size, "fem_nccl_comm_init: bad args");
  ncclUniqueId u;
  for (int i = 0; i < 128; ++i) u.internal[i] = (char)id[i];
  ncclComm_t c = nullptr;
  fem_status st = nccl_status(ncclCommInitRank(&c, size, u, rank), "ncclCommInitRank");
  if (st) return st;
  *comm = (void *)c;
  return FEM_OK;
}

fem_status fem_nccl_comm_count(void *comm, int *count) {
  FEM_NVTX_RANGE("fem_nccl_comm_count");
  FEM_ARG(comm && count, "fem_nccl_comm_count: null argument");
  return nccl_status(ncclCommCount((ncclComm_t)comm, count), "ncclCommCount");
}

fem_status fem_nccl_comm_destroy(void *comm) {
  FEM_NVTX_RANGE("fem_nccl_comm_destroy");
  if (!comm) return FEM_OK;
  return nccl_status(ncclCommDestroy((ncclComm_t)comm), "ncclCommDestroy");
}

fem_status fem_allreduce_sum(fem_problem *h, double *buf, int n, fem_stream stream) {
  FEM_NVTX_RANGE("fem_allreduce_sum");
  FEM_ARG(h && buf && n > 0, "fem_allreduce_sum: bad args");
  return allreduce(&h->p, buf, n, (cudaStream_t)stream);
}

fem_status fem_halo_size(const fem_problem *h, int64_t *n_doubles) {
  FEM_NVTX_RANGE("fem_halo_size");
  FEM_ARG(h && n_doubles, "fem_halo_size: null argument");
  *n_doubles = h->p.n_halo_entries * h->p.dim;
  return FEM_OK;
}

fem_status fem_halo_pack(fem_problem *h, const double *y, double *sendbuf, fem_stream stream) {
  FEM_NVTX_RANGE("fem_halo_pack");
  FEM_ARG(h && y && sendbuf, "fem_halo_pack: null argument");
  return halo_pack(&h->p, y, sendbuf, (cudaStream_t)stream);
}

fem_status fem_halo_combine(fem_problem *h, double *y, const double *recvbuf, fem_stream stream) {
  FEM_NVTX_RANGE("fem_halo_combine");
  FEM_ARG(h && y && recvbuf, "fem_halo_combine: null argument");
  return halo_combine(&h->p, y, recvbuf, (cudaStream_t)stream);
}

}  // extern "C"
