// Slab sharding across the GPUs of one box (include/phiks.h).
#include "host.h"

extern "C" {

// ===========================================================================
// Slab sharding across the GPUs of one box
// ===========================================================================
phiks_status phiks_create_sharded(int d, const int* n, const double* const* A_host, int rank, int world,
                                  phiks_handle* out) {
  return phiks_create_sharded_blocks(1, d, n, A_host, rank, world, out);
}

}  // extern "C"

static phiks_status create_sharded_impl(int nblocks, int d, const int* n, const double* const* A_host, int rank,
                                        int world, bool cplx, phiks_handle* out);

extern "C" {

phiks_status phiks_create_sharded_blocks(int nblocks, int d, const int* n, const double* const* A_host, int rank,
                                         int world, phiks_handle* out) {
  return create_sharded_impl(nblocks, d, n, A_host, rank, world, false, out);
}

phiks_status phiks_create_sharded_complex(int d, const int* n, const double* const* A_host, int rank, int world,
                                          phiks_handle* out) {
  return create_sharded_impl(1, d, n, A_host, rank, world, true, out);
}

phiks_status phiks_create_sharded_blocks_complex(int nblocks, int d, const int* n, const double* const* A_host,
                                                 int rank, int world, phiks_handle* out) {
  return create_sharded_impl(nblocks, d, n, A_host, rank, world, true, out);
}

}  // extern "C"

static phiks_status create_sharded_impl(int nblocks, int d, const int* n, const double* const* A_host, int rank,
                                        int world, bool cplx, phiks_handle* out) {
  if (!out || !n) return fail(PHIKS_ERR_ARG, "null argument");
  *out = nullptr;
  if (world < 1 || world > kMaxRanks || rank < 0 || rank >= world) return fail(PHIKS_ERR_ARG, "rank/world");
  if (world > 1) {
    if (d < 2) return fail(PHIKS_ERR_ARG, "sharding needs d >= 2");
    if (n[d - 1] < world || n[d - 2] < world) return fail(PHIKS_ERR_ARG, "n_d and n_{d-1} must be >= world");
  }
  phiks_handle h = nullptr;
  phiks_status st = cplx ? phiks_create_blocks_complex(nblocks, d, n, A_host, &h)
                         : phiks_create_blocks(nblocks, d, n, A_host, &h);
  if (st != PHIKS_OK) return st;
  h->rank = rank;
  h->world = world;
  if (world > 1) {
    // slabs of mode d (layout S_d) and of mode d-1 (S_{d-1}), block-distributed
    int64_t L0 = 1;
    for (int mu = 0; mu + 2 < d; ++mu) L0 *= n[mu];
    const int64_t na = n[d - 2], nd = n[d - 1];
    h->n[d - 1] = static_cast<int>(blk_cnt(nd, world, rank));
    h->Nc = L0 * na * h->n[d - 1];
    h->N = cplx ? 2 * h->Nc : h->Nc;
    int64_t slot = 0;  // the largest local tensor of either layout on any rank (in doubles)
    for (int k = 0; k < world; ++k)
      slot = std::max({slot, L0 * na * blk_cnt(nd, world, k), L0 * blk_cnt(na, world, k) * nd});
    if (cplx) slot *= 2;
    h->sym_slot = (static_cast<size_t>(slot) * sizeof(double) + 255) & ~size_t(255);
    h->sym_bytes = kCtrlBytes + 2 * kShardChunk * h->sym_slot;
    {  // exponential pool (orchestrate.cpp expm_stage): 12 matrices per distinct factor (q ≤ 12), two halves
      size_t half = 0;
      for (const auto& F : h->factors) half += 12 * ((static_cast<size_t>(F.n) * F.n * sizeof(double) + 255) & ~size_t(255));
      h->xpool_off = h->sym_bytes;
      h->xpool_half = half;
      h->sym_bytes += 2 * half;
    }
    if (!cplx && d >= 3) {  // exponent exchange of the sharded int8 digit stages (host.h shard_digits_ok)
      h->exch_off = h->sym_bytes;
      h->exch_l0 = L0;
      h->sym_bytes += (static_cast<size_t>(world) * kShardChunk * L0 * sizeof(double) + 255) & ~size_t(255);
    }
    if (cudaMalloc(reinterpret_cast<void**>(&h->sym), h->sym_bytes) != cudaSuccess) {
      phiks_destroy(h);
      return fail(PHIKS_ERR_NOMEM, "symmetric region cudaMalloc");
    }
    if (cudaMemset(h->sym, 0, kCtrlBytes) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
      phiks_destroy(h);
      return fail(PHIKS_ERR_CUDA, "symmetric region init");
    }
    h->peer[rank] = h->sym;
  } else {
    h->peers_ready = true;
  }
  *out = h;
  return PHIKS_OK;
}

extern "C" {

phiks_status phiks_shard_info(phiks_handle h, int* rank, int* world, int64_t* local_count, size_t* sym_bytes) {
  if (!h) return fail(PHIKS_ERR_ARG, "null handle");
  if (rank) *rank = h->rank;
  if (world) *world = h->world;
  if (local_count) *local_count = h->Nc;
  if (sym_bytes) *sym_bytes = h->sym_bytes;
  return PHIKS_OK;
}

phiks_status phiks_shard_ipc_handle(phiks_handle h, void* handle_out) {
  if (!h || !handle_out) return fail(PHIKS_ERR_ARG, "null argument");
  std::memset(handle_out, 0, PHIKS_IPC_HANDLE_BYTES);
  if (!h->sharded()) return PHIKS_OK;
  static_assert(sizeof(cudaIpcMemHandle_t) <= PHIKS_IPC_HANDLE_BYTES, "IPC handle size");
  cudaIpcMemHandle_t ih;
  CUDA_TRY(cudaIpcGetMemHandle(&ih, h->sym));
  std::memcpy(handle_out, &ih, sizeof(ih));
  return PHIKS_OK;
}

phiks_status phiks_shard_open_peers(phiks_handle h, const void* handles) {
  if (!h || !handles) return fail(PHIKS_ERR_ARG, "null argument");
  if (!h->sharded()) {
    h->peers_ready = true;
    return PHIKS_OK;
  }
  const char* hb = static_cast<const char*>(handles);
  for (int k = 0; k < h->world; ++k) {
    if (k == h->rank) continue;
    if (h->peer_ipc[k] && h->peer[k]) {
      cudaIpcCloseMemHandle(h->peer[k]);
      h->peer[k] = nullptr;
      h->peer_ipc[k] = false;
    }
    cudaIpcMemHandle_t ih;
    std::memcpy(&ih, hb + static_cast<size_t>(k) * PHIKS_IPC_HANDLE_BYTES, sizeof(ih));
    void* ptr = nullptr;
    CUDA_TRY(cudaIpcOpenMemHandle(&ptr, ih, cudaIpcMemLazyEnablePeerAccess));
    h->peer[k] = static_cast<char*>(ptr);
    h->peer_ipc[k] = true;
  }
  h->peers_ready = true;
  return PHIKS_OK;
}

phiks_status phiks_shard_base(phiks_handle h, void** base) {
  if (!h || !base) return fail(PHIKS_ERR_ARG, "null argument");
  *base = h->sym;
  return PHIKS_OK;
}

phiks_status phiks_shard_set_peer_bases(phiks_handle h, void* const* bases) {
  if (!h || !bases) return fail(PHIKS_ERR_ARG, "null argument");
  if (!h->sharded()) {
    h->peers_ready = true;
    return PHIKS_OK;
  }
  if (bases[h->rank] != h->sym) return fail(PHIKS_ERR_ARG, "bases[rank] must be this handle's region");
  for (int k = 0; k < h->world; ++k) {
    if (!bases[k]) return fail(PHIKS_ERR_ARG, "null peer base");
    h->peer[k] = static_cast<char*>(bases[k]);
  }
  h->peers_ready = true;
  return PHIKS_OK;
}

phiks_status phiks_apply_ranks_serial(const phiks_handle* hs, int world, const phiks_request* req, int n_vecs,
                                      const double* const* vecs, double* const* outs, void* stream) {
  return phiks_apply_ranks_serial_ex(hs, world, req, n_vecs, vecs, outs, stream, 0);
}

phiks_status phiks_apply_ranks_serial_ex(const phiks_handle* hs, int world, const phiks_request* req, int n_vecs,
                                         const double* const* vecs, double* const* outs, void* stream, int which) {
  if (which < 0 || which > 2) return fail(PHIKS_ERR_ARG, "which must be 0, 1 or 2");
  if (!hs || world < 1 || world > kMaxRanks || !req || !vecs || !outs) return fail(PHIKS_ERR_ARG, "bad argument");
  for (int k = 0; k < world; ++k) {
    if (!hs[k] || hs[k]->world != world || hs[k]->rank != k) return fail(PHIKS_ERR_ARG, "hs[k] must be rank k of world");
    if (req->mem_kind != PHIKS_MEM_DEVICE) return fail(PHIKS_ERR_ARG, "ranks_serial takes device memory");
  }
  const bool same = req->mode == PHIKS_MODE_SAME_VECTOR;
  const int nouts = hs[0]->nblocks * (same ? req->n_ells * req->n_scales : req->n_scales);
  std::vector<ApplyRun> runs(world);
  for (int k = 0; k < world; ++k) {
    phiks_status st = runs[k].init(hs[k], req, n_vecs, vecs + static_cast<size_t>(k) * n_vecs,
                                   outs + static_cast<size_t>(k) * nouts, stream, false);
    if (st != PHIKS_OK) return st;
  }
  // plan: norms phase of every rank (no barrier: stream order), then read
  if (runs[0].need_norms) {
    for (int k = 0; k < world; ++k) {
      phiks_status st = runs[k].norms_enqueue(false);
      if (st != PHIKS_OK) return st;
    }
    for (int k = 0; k < world; ++k) {
      phiks_status st = runs[k].norms_finish(hs[0]->sym);
      if (st != PHIKS_OK) return st;
    }
  } else {
    for (int k = 0; k < world; ++k) {
      phiks_status st = runs[k].plan_direct(nullptr);
      if (st != PHIKS_OK) return st;
    }
  }
  std::vector<std::vector<Exec::Op>> ops(world);
  std::vector<size_t> need(world, 0);
  for (int k = 0; k < world; ++k) {
    phiks_status st = runs[k].measure(&need[k]);
    if (st != PHIKS_OK) return st;
    char* base = nullptr;
    st = runs[k].workspace(nullptr, 0, need[k], &base);
    if (st != PHIKS_OK) return st;
    st = runs[k].execute(base, need[k], &ops[k]);
    if (st != PHIKS_OK) return st;
  }
  // replay phase by phase: the segment between two barriers of every rank
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  std::vector<size_t> pos(world, 0);
  bool more = true;
  while (more) {
    more = false;
    for (int k = 0; k < world; ++k) {
      auto& v = ops[k];
      while (pos[k] < v.size() && !v[pos[k]].barrier) {
        if ((which == 1 && !v[pos[k]].pre) || (which == 2 && v[pos[k]].pre)) {  // filtered replay (timing)
          ++pos[k];
          continue;
        }
        cudaError_t e = v[pos[k]].fn(cs);
        if (e != cudaSuccess) return fail(PHIKS_ERR_CUDA, std::string(v[pos[k]].what) + ": " + cudaGetErrorString(e));
        ++pos[k];
      }
      if (pos[k] < v.size()) {
        ++pos[k];  // the barrier itself: implied by stream order
        more = true;
      }
    }
  }
  for (int k = 0; k < world; ++k) runs[k].finish_stats(need[k]);
  return PHIKS_OK;
}


phiks_status phiks_shard_layout(int d, const int* n, int rank, int world, int stage, int64_t* out7) {
  if (!n || !out7 || d < 2 || d > PHIKS_MAX_D || world < 1 || world > kMaxRanks || rank < 0 || rank >= world ||
      (stage != 0 && stage != 1))
    return fail(PHIKS_ERR_ARG, "bad argument");
  if (n[d - 1] % world != 0 || n[d - 2] % world != 0)
    return fail(PHIKS_ERR_ARG, "dims not divisible by world (use phiks_shard_layout_ex)");
  const ShardStage s = shard_stage(d, n, rank, world, stage);
  const int64_t cb = s.n / world;
  const int64_t v[7] = {s.L, s.n, s.R, cb, s.kstride[0], s.kroff[0], s.colstride};
  for (int i = 0; i < 7; ++i) out7[i] = v[i];
  return PHIKS_OK;
}

phiks_status phiks_shard_layout_ex(int d, const int* n, int rank, int world, int stage, int64_t* out) {
  if (!n || !out || d < 2 || d > PHIKS_MAX_D || world < 1 || world > kMaxRanks || rank < 0 || rank >= world ||
      (stage != 0 && stage != 1) || n[d - 1] < world || n[d - 2] < world)
    return fail(PHIKS_ERR_ARG, "bad argument");
  const ShardStage s = shard_stage(d, n, rank, world, stage);
  out[0] = s.L;
  out[1] = s.n;
  out[2] = s.R;
  out[3] = s.colstride;
  for (int k = 0; k < world; ++k) {
    out[4 + k] = s.kstart[k];
    out[4 + world + k] = s.kstride[k];
    out[4 + 2 * world + k] = s.kroff[k];
  }
  return PHIKS_OK;
}


phiks_status phiks_wait(phiks_handle h) {
  if (!h) return fail(PHIKS_ERR_ARG, "null handle");
  for (int k = 0; k < 2; ++k) {
    if (h->ev_d2h[k]) CUDA_TRY(cudaEventSynchronize(h->ev_d2h[k]));
    if (h->ev_cdone[k]) CUDA_TRY(cudaEventSynchronize(h->ev_cdone[k]));
  }
  return check_barrier_flag(h);
}


phiks_status phiks_shard_peer_base(phiks_handle h, int k, void** base) {
  if (!h || !base || k < 0 || k >= h->world) return fail(PHIKS_ERR_ARG, "bad argument");
  *base = h->peer[k];
  return PHIKS_OK;
}

}  // extern "C"
