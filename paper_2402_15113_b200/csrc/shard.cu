// shard.cu — row E: node memory sharded by node id over `world` GPUs.
//
// owner(v) = v mod G, local row = v / G.  Global iteration i covers G·B
// consecutive events; rank g takes the local batch [base + gB, base + (g+1)B)
// ("each GPU worker retrieves a local batch").  The T-CSR is
// replicated, so sampling (A1) and dedup (A2) stay local.  Two exchanges per
// iteration replace the paper's single CPU-resident memory.
//
// Transport: every rank owns a receive WINDOW (one allocation, exported by
// CUDA IPC to the other ranks of the node, or shared directly by in-process
// ranks) and the SENDING kernels store their data straight into the peer's
// window over NVLink — only the real entries, never a padded block:
//
//   fetch (A3):   plan   — the distinct ids each owner must serve, in id order,
//                          written into the owner's window (+ their count);
//                 barrier
//                 serve  — the owner gathers [row | ts (| mail | mail_ts)] of
//                          each request and stores the reply into the
//                          requester's window;
//                 barrier
//                 finish — replies scattered to the dense outputs by position.
//   commit (A7):  pack   — each local winner becomes a record (key, node, ts,
//                          h', mail) stored into its owner's window (+ the
//                          per-sender counts); key = 2·(global event index) +
//                          role, the global pair index, so the merge
//                          reproduces the single-GPU winner of batch G·B;
//                 barrier
//                 merge  — owner: 64-bit atomicMax of key per node, then the
//                          record holding the max key writes the row
//                          (deterministic: independent of arrival order).
//
// The barrier is a one-int NCCL all-reduce on the caller's stream (a fetch
// and a commit communicator, so the two may run on different streams), or
// nothing for in-process ranks (one stream orders the phases).  Windows are
// double-buffered by iteration parity, so a fast rank's next iteration never
// overwrites a slow rank's buffers before that rank has passed the barrier
// that follows its reads.
#include "internal.cuh"

namespace mspipe {

static inline unsigned blocks_for(int64_t threads_total, int per_sm) {
  int64_t b = (threads_total + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * per_sm;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (unsigned)b;
}

// counts region of a window: [3 kinds][world] int32 (FETCH_IDS, -, COMMIT)
constexpr int kCntFetch = 0, kCntCommit = 2;

// ---- fetch plan ---------------------------------------------------------
__global__ void k_shard_mark(const int32_t* __restrict__ ids, int64_t n, int64_t N, uint8_t* __restrict__ needed) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = __ldg(ids + p);
    if (v >= 0 && v < N) needed[v] = 1;
    else if (v != -1) raise_dev(MSPIPE_DEVERR_RANGE);
  }
}

// one CTA: per owner o, compact the needed ids v = o, o+G, ... in id order
// straight into o's window (slot order), then the count
__global__ void __launch_bounds__(1024) k_shard_plan(uint8_t* __restrict__ needed, int64_t N, int32_t G, int32_t me,
                                                     int64_t cap, uint8_t* const* __restrict__ peers,
                                                     int64_t off_ids, int64_t off_cnt,
                                                     int32_t* __restrict__ slot_of,
                                                     unsigned long long* __restrict__ sent) {
  __shared__ int32_t warp_tot[32];
  __shared__ int32_t base_s;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int32_t o = 0; o < G; ++o) {
    int32_t* ids_o = reinterpret_cast<int32_t*>(peers[o] + off_ids) + (int64_t)me * cap;
    const int64_t rows = (N - o + G - 1) / G;  // ids o, o+G, ... < N
    if (tid == 0) base_s = 0;
    __syncthreads();
    for (int64_t t0 = 0; t0 < rows; t0 += 1024) {
      const int64_t t = t0 + tid;
      const int64_t v = o + t * G;
      const int32_t f = (t < rows && needed[v]) ? 1 : 0;
      int32_t incl = f;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += y;
      }
      if (lane == 31) warp_tot[wid] = incl;
      __syncthreads();
      if (wid == 0) {
        const int32_t w = warp_tot[lane];
        int32_t wi = w;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int32_t y = __shfl_up_sync(0xffffffffu, wi, d);
          if (lane >= d) wi += y;
        }
        warp_tot[lane] = wi - w;
      }
      __syncthreads();
      if (f) {
        const int32_t slot = base_s + warp_tot[wid] + incl - 1;
        ids_o[slot] = (int32_t)v;  // remote store into the owner's window
        slot_of[v] = slot;
        needed[v] = 0;
      }
      __syncthreads();
      if (tid == 1023) base_s += warp_tot[31] + incl;  // last thread: total of this round
      __syncthreads();
    }
    if (tid == 0) {
      reinterpret_cast<int32_t*>(peers[o] + off_cnt)[kCntFetch * G + me] = base_s;
      atomicAdd(sent + 0, (unsigned long long)(4 * base_s + 4));
    }
    __syncthreads();
  }
  __threadfence_system();  // the owner reads after the barrier
}

// ---- fetch serve / finish ----------------------------------------------
// reply record per requested id: [mem row (Qm float4)] [ts, pad] (+ [mail row (Qa)] [mail_ts, pad]),
// stored into the requester's window at slot (me, j)
__global__ void k_shard_serve(const int32_t* __restrict__ req_ids, const int32_t* __restrict__ req_cnt, int64_t cap,
                              int32_t G, int32_t me, const float4* __restrict__ mem,
                              const double* __restrict__ mem_ts, int32_t Qm, const float4* __restrict__ mail,
                              const double* __restrict__ mail_ts, int32_t Qa, uint8_t* const* __restrict__ peers,
                              int64_t off_rep, unsigned long long* __restrict__ sent) {
  const int lane = threadIdx.x & 31;
  const int32_t Qr = Qm + 1 + (Qa > 0 ? Qa + 1 : 0);
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long bytes = 0;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < (int64_t)G * cap; r += nwarps) {
    const int32_t s = (int32_t)(r / cap);
    const int64_t j = r - (int64_t)s * cap;
    if (j >= __ldg(req_cnt + kCntFetch * G + s)) continue;
    const int32_t v = __ldg(req_ids + r);
    const int64_t loc = v / G;
    float4* rec = reinterpret_cast<float4*>(peers[s] + off_rep) + ((int64_t)me * cap + j) * Qr;
    for (int32_t c = lane; c < Qm; c += 32) rec[c] = __ldg(mem + loc * Qm + c);
    if (lane == 0) {
      double2 t;
      t.x = __ldg(mem_ts + loc);
      t.y = 0.0;
      reinterpret_cast<double2*>(rec)[Qm] = t;
    }
    if (Qa > 0) {
      for (int32_t c = lane; c < Qa; c += 32) rec[Qm + 1 + c] = __ldg(mail + loc * Qa + c);
      if (lane == 0) {
        double2 t;
        t.x = __ldg(mail_ts + loc);
        t.y = 0.0;
        reinterpret_cast<double2*>(rec)[Qm + 1 + Qa] = t;
      }
    }
    bytes += 16ull * Qr;
  }
  if (lane == 0 && bytes) atomicAdd(sent + 1, bytes);
  __threadfence_system();
}

__global__ void k_shard_finish(const int32_t* __restrict__ ids, int64_t n, int64_t N, int32_t G, int64_t cap,
                               const int32_t* __restrict__ slot_of, const float4* __restrict__ rep,
                               int32_t Qm, int32_t Qa, float4* __restrict__ out_mem, double* __restrict__ out_mem_ts,
                               float4* __restrict__ out_mail, double* __restrict__ out_mail_ts) {
  const int lane = threadIdx.x & 31;
  const int32_t Qr = Qm + 1 + (Qa > 0 ? Qa + 1 : 0);
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < n; p += nwarps) {
    const int32_t v = __ldg(ids + p);
    const bool ok = v >= 0 && v < N;
    const float4* rec = ok ? rep + ((int64_t)(v % G) * cap + __ldg(slot_of + v)) * Qr : nullptr;
    for (int32_t c = lane; c < Qm; c += 32) out_mem[p * Qm + c] = ok ? __ldcg(rec + c) : z;
    if (lane == 0) out_mem_ts[p] = ok ? __ldcg(reinterpret_cast<const double2*>(rec) + Qm).x : 0.0;
    if (Qa > 0) {
      for (int32_t c = lane; c < Qa; c += 32) out_mail[p * Qa + c] = ok ? __ldcg(rec + Qm + 1 + c) : z;
      if (lane == 0) out_mail_ts[p] = ok ? __ldcg(reinterpret_cast<const double2*>(rec) + Qm + 1 + Qa).x : 0.0;
    }
  }
}

// ---- commit pack / merge ------------------------------------------------
// record: [key i64, node i64] [ts f64, pad] [h' (M/4 float4)] [mail (stride/4 float4)]
// one CTA assigns each local winner a slot in its owner's window (per-owner
// counters; the slot order is irrelevant to the merge result) and stores the
// per-owner counts into the owners' windows
__global__ void __launch_bounds__(1024) k_shard_pack_plan(const int32_t* __restrict__ nodes,
                                                          const int32_t* __restrict__ num, int64_t max_n,
                                                          int32_t G, int32_t me, int64_t capw,
                                                          int32_t* __restrict__ dest,
                                                          uint8_t* const* __restrict__ peers, int64_t off_cnt,
                                                          int64_t rec_bytes, unsigned long long* __restrict__ sent) {
  __shared__ int32_t cnt[64];
  if (threadIdx.x < 64) cnt[threadIdx.x] = 0;
  __syncthreads();
  const int64_t U = min64((int64_t)__ldg(num), max_n);
  for (int64_t u = threadIdx.x; u < U; u += blockDim.x) {
    const int32_t node = __ldg(nodes + u);
    const int32_t o = node % G;
    const int32_t s = atomicAdd(&cnt[o], 1);
    if (s >= capw) {
      raise_dev(MSPIPE_DEVERR_CAPACITY);
      dest[u] = -1;
    } else {
      dest[u] = (int32_t)(o * capw + s);
    }
  }
  __syncthreads();
  if ((int)threadIdx.x < G) {
    const int32_t c = cnt[threadIdx.x] < capw ? cnt[threadIdx.x] : (int32_t)capw;
    reinterpret_cast<int32_t*>(peers[threadIdx.x] + off_cnt)[kCntCommit * G + me] = c;
    atomicAdd(sent + 2, (unsigned long long)(c * rec_bytes + 4));
  }
  __threadfence_system();
}

__global__ void k_shard_pack(const int32_t* __restrict__ nodes, const int32_t* __restrict__ winner,
                             const int32_t* __restrict__ num, int64_t max_n, const int32_t* __restrict__ dest,
                             int64_t key_base, const float4* __restrict__ new_mem, const double* __restrict__ new_ts,
                             const float4* __restrict__ new_mail, int32_t Qm, int32_t Qa, int32_t me, int64_t capw,
                             uint8_t* const* __restrict__ peers, int64_t off_com) {
  const int lane = threadIdx.x & 31;
  const int32_t Qr = 2 + Qm + Qa;
  const int64_t U = min64((int64_t)__ldg(num), max_n);
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < U; u += nwarps) {
    const int32_t d = __ldg(dest + u);
    if (d < 0) continue;
    const int32_t o = (int32_t)(d / capw);
    const int64_t s = d - (int64_t)o * capw;
    float4* r = reinterpret_cast<float4*>(peers[o] + off_com) + ((int64_t)me * capw + s) * Qr;
    if (lane == 0) {
      reinterpret_cast<longlong2*>(r)[0] = make_longlong2(key_base + __ldg(winner + u), (long long)__ldg(nodes + u));
      double2 t;
      t.x = __ldg(new_ts + u);
      t.y = 0.0;
      reinterpret_cast<double2*>(r)[1] = t;
    }
    for (int32_t c = lane; c < Qm; c += 32) r[2 + c] = __ldg(new_mem + u * Qm + c);
    for (int32_t c = lane; c < Qa; c += 32) r[2 + Qm + c] = __ldg(new_mail + u * Qa + c);
  }
  __threadfence_system();
}

// records of sender s occupy slots [s·capw, s·capw + count_s) of the window
__global__ void k_shard_merge_key(const float4* __restrict__ rec, const int32_t* __restrict__ cnt, int32_t G,
                                  int64_t capw, int32_t Qr, int64_t rows, unsigned long long* __restrict__ keytab) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < (int64_t)G * capw;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s = (int32_t)(r / capw);
    if (r - (int64_t)s * capw >= __ldcg(cnt + kCntCommit * G + s)) continue;
    const longlong2 h = __ldcg(reinterpret_cast<const longlong2*>(rec + r * Qr));
    const int64_t loc = h.y / G;
    if (h.x < 0 || loc < 0 || loc >= rows) {
      raise_dev(MSPIPE_DEVERR_RANGE);
      continue;
    }
    atomicMax(keytab + loc, (unsigned long long)h.x);
  }
}

__global__ void k_shard_merge_apply(const float4* __restrict__ rec, const int32_t* __restrict__ cnt, int32_t G,
                                    int64_t capw, int32_t Qr, int64_t rows,
                                    const unsigned long long* __restrict__ keytab, int32_t Qm, int32_t Qa,
                                    float4* __restrict__ mem, double* __restrict__ mem_ts, float4* __restrict__ mail,
                                    double* __restrict__ mail_ts) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < (int64_t)G * capw; r += nwarps) {
    const int32_t s = (int32_t)(r / capw);
    if (r - (int64_t)s * capw >= __ldcg(cnt + kCntCommit * G + s)) continue;
    const float4* p = rec + r * Qr;
    const longlong2 h = __ldcg(reinterpret_cast<const longlong2*>(p));
    const int64_t loc = h.y / G;
    if (h.x < 0 || loc < 0 || loc >= rows || __ldcg(keytab + loc) != (unsigned long long)h.x) continue;  // not the LWW winner
    for (int32_t c = lane; c < Qm; c += 32) mem[loc * Qm + c] = __ldcg(p + 2 + c);
    for (int32_t c = lane; c < Qa; c += 32) mail[loc * Qa + c] = __ldcg(p + 2 + Qm + c);
    if (lane == 0) {
      const double t = __ldcg(reinterpret_cast<const double2*>(p) + 1).x;
      mem_ts[loc] = t;
      mail_ts[loc] = t;
    }
  }
}

// ---- MSPipe-S with sharded memory (A4) ----------------------
// The mitigation of target w reads S.mem_ts[w], S.mem_ts of its 2-hop
// candidates and S.mem of the chosen Ω, all owned by other ranks.  After the
// subgraph fetch (which delivered w's own row and mem_ts as the root row),
// one warp per target decides eligibility and lists the candidates exactly
// as k_mitigate enumerates them (the T-CSR is replicated): out_ids[t] =
// [w, candidates of sample(x, t*) for x in sample(w, t*)] (pads -1; the
// candidates only for eligible targets, w for every target: k_mitigate reads
// S.mem_ts[w] and, ineligible, S.mem[w]).  A second fetch of that list fills a node-indexed table
// from which k_mitigate then runs unchanged.
__global__ void k_shard_mit_candidates(Tcsr g, const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                                       const double* __restrict__ ts, int64_t B, const double* __restrict__ root_ts,
                                       int64_t root_step, double gamma, int32_t F, int32_t* __restrict__ out_ids) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int32_t L = 1 + F * F;
  for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < 2 * B; t += nwarps) {
    const int64_t a = t < B ? t : t - B;
    const int32_t w = t < B ? __ldg(src + a) : __ldg(dst + a);
    const double tstar = __ldg(ts + a);
    int32_t* row = out_ids + t * L;
    const bool wok = w >= 0 && w < g.num_nodes;
    const bool elig = wok && (tstar - __ldcg(root_ts + t * root_step)) > gamma;  // G11
    for (int32_t q = lane; q < L; q += 32) row[q] = (q == 0 && wok) ? w : -1;  // k_mitigate reads every w
    __syncwarp();
    if (!elig) continue;
    int64_t begw;
    const int64_t endw = lower_bound_ts(g, w, tstar, &begw);
    const int32_t cntw = (int32_t)min64(endw - begw, (int64_t)F);
    int32_t x = (lane < cntw) ? __ldg(g.nbr + (endw - 1 - lane)) : -1;
    if (x == w) x = -1;
    if (lane < F && x >= 0) {
      int64_t begx;
      const int64_t endx = lower_bound_ts(g, x, tstar, &begx);
      const int32_t cx = (int32_t)min64(endx - begx, (int64_t)F);
      for (int32_t i = 0; i < cx; ++i) {
        const int32_t u = __ldg(g.nbr + (endx - 1 - i));
        row[1 + lane * F + i] = u == w ? -1 : u;
      }
    }
    __syncwarp();
  }
}

// rows of a finished fetch written into a node-indexed table (pads skipped;
// repeated ids write identical rows)
__global__ void k_shard_finish_table(const int32_t* __restrict__ ids, int64_t n, int64_t N, int32_t G, int64_t cap,
                                     const int32_t* __restrict__ slot_of, const float4* __restrict__ rep, int32_t Qm,
                                     int32_t Qa, float4* __restrict__ tab_mem, double* __restrict__ tab_ts) {
  const int lane = threadIdx.x & 31;
  const int32_t Qr = Qm + 1 + (Qa > 0 ? Qa + 1 : 0);
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < n; p += nwarps) {
    const int32_t v = __ldg(ids + p);
    if (v < 0 || v >= N) continue;
    const float4* rec = rep + ((int64_t)(v % G) * cap + __ldg(slot_of + v)) * Qr;
    for (int32_t c = lane; c < Qm; c += 32) tab_mem[(int64_t)v * Qm + c] = __ldcg(rec + c);
    if (lane == 0) tab_ts[v] = __ldcg(reinterpret_cast<const double2*>(rec) + Qm).x;
  }
}

void shard_mit_candidates(const Tcsr& g, const int32_t* src, const int32_t* dst, const double* ts, int64_t B,
                          const double* root_ts, int64_t root_step, double gamma, int32_t F, int32_t* out_ids,
                          cudaStream_t s) {
  k_shard_mit_candidates<<<blocks_for(2 * B * 32, 8), 256, 0, s>>>(g, src, dst, ts, B, root_ts, root_step, gamma,
                                                                   F, out_ids);
}

void shard_fetch_finish_table(mspipe_memory* st, const int32_t* ids, int64_t n, float* tab_mem, double* tab_ts,
                              cudaStream_t s) {
  const int p = (int)(st->sh_fetch_iter & 1);
  const int32_t Qm = st->mem_dim / 4, Qa = st->sh_with_mail ? (int32_t)(st->mail_stride / 4) : 0;
  k_shard_finish_table<<<blocks_for(n * 32, 8), 256, 0, s>>>(
      ids, n, st->num_nodes, st->world, st->sh_cap, st->sh_slot_of,
      reinterpret_cast<const float4*>(st->sh_window + st->sh_off_rep[p]), Qm, Qa, (float4*)tab_mem, tab_ts);
}

// ---- window layout --------------------------------------------------------
int64_t shard_fetch_rec_bytes(const mspipe_memory* st, bool with_mail) {
  return 16LL * (st->mem_dim / 4 + 1 + (with_mail ? st->mail_stride / 4 + 1 : 0));
}

int64_t shard_commit_rec_bytes(const mspipe_memory* st) { return 16LL * (2 + st->mem_dim / 4 + st->mail_stride / 4); }

// per parity: ids [world][cap] i32 | counts [3][world] i32 | replies [world][cap] rec | commits [world][capw] rec,
// every region 256-byte aligned
void shard_layout(mspipe_memory* st) {
  auto al = [](int64_t x) { return (x + 255) / 256 * 256; };
  const int64_t G = st->world;
  int64_t off = 0;
  for (int p = 0; p < 2; ++p) {
    st->sh_off_ids[p] = off;
    off += al(4 * G * st->sh_cap);
    st->sh_off_cnt[p] = off;
    off += al(4 * 3 * G);
    st->sh_off_rep[p] = off;
    off += al(shard_fetch_rec_bytes(st, true) * G * st->sh_cap);
    st->sh_off_com[p] = off;
    off += al(shard_commit_rec_bytes(st) * G * st->sh_capw);
  }
  st->sh_win_bytes = off;
}

// ---- host launchers -----------------------------------------------------
void shard_fetch_plan(mspipe_memory* st, const int32_t* ids, int64_t n, cudaStream_t s) {
  const int p = (int)(st->sh_fetch_iter & 1);
  k_shard_mark<<<blocks_for(n, 8), 256, 0, s>>>(ids, n, st->num_nodes, st->sh_needed);
  k_shard_plan<<<1, 1024, 0, s>>>(st->sh_needed, st->num_nodes, st->world, st->rank, st->sh_cap, st->sh_peers,
                                  st->sh_off_ids[p], st->sh_off_cnt[p], st->sh_slot_of, st->sh_sent);
}

void shard_fetch_serve(mspipe_memory* st, bool with_mail, cudaStream_t s) {
  const int p = (int)(st->sh_fetch_iter & 1);
  const int32_t Qm = st->mem_dim / 4, Qa = with_mail ? (int32_t)(st->mail_stride / 4) : 0;
  const int64_t total = (int64_t)st->world * st->sh_cap;
  k_shard_serve<<<blocks_for(total * 32, 8), 256, 0, s>>>(
      reinterpret_cast<const int32_t*>(st->sh_window + st->sh_off_ids[p]),
      reinterpret_cast<const int32_t*>(st->sh_window + st->sh_off_cnt[p]), st->sh_cap, st->world, st->rank,
      (const float4*)st->mem, st->mem_ts, Qm, (const float4*)st->mail, st->mail_ts, Qa, st->sh_peers,
      st->sh_off_rep[p], st->sh_sent);
}

void shard_fetch_finish(mspipe_memory* st, const int32_t* ids, int64_t n, float* out_mem, double* out_mem_ts,
                        float* out_mail, double* out_mail_ts, cudaStream_t s) {
  const int p = (int)(st->sh_fetch_iter & 1);
  const int32_t Qm = st->mem_dim / 4, Qa = out_mail ? (int32_t)(st->mail_stride / 4) : 0;
  k_shard_finish<<<blocks_for(n * 32, 8), 256, 0, s>>>(
      ids, n, st->num_nodes, st->world, st->sh_cap, st->sh_slot_of,
      reinterpret_cast<const float4*>(st->sh_window + st->sh_off_rep[p]), Qm, Qa, (float4*)out_mem, out_mem_ts,
      (float4*)out_mail, out_mail_ts);
}

void shard_commit_pack(mspipe_memory* st, int64_t commit_version, const int32_t* nodes, const int32_t* winner,
                       const int32_t* num, int64_t max_n, int64_t key_base, const float* new_mem,
                       const double* new_ts, const float* new_mail, cudaStream_t s) {
  const int p = (int)(commit_version & 1);
  const int32_t Qm = st->mem_dim / 4, Qa = (int32_t)(st->mail_stride / 4);
  k_shard_pack_plan<<<1, 1024, 0, s>>>(nodes, num, max_n, st->world, st->rank, st->sh_capw, st->sh_dest,
                                       st->sh_peers, st->sh_off_cnt[p], shard_commit_rec_bytes(st), st->sh_sent);
  k_shard_pack<<<blocks_for(max_n * 32, 8), 256, 0, s>>>(nodes, winner, num, max_n, st->sh_dest, key_base,
                                                         (const float4*)new_mem, new_ts, (const float4*)new_mail, Qm,
                                                         Qa, st->rank, st->sh_capw, st->sh_peers, st->sh_off_com[p]);
}

void shard_commit_merge(mspipe_memory* st, int64_t commit_version, cudaStream_t s) {
  const int p = (int)(commit_version & 1);
  const int32_t Qm = st->mem_dim / 4, Qa = (int32_t)(st->mail_stride / 4);
  const int32_t Qr = 2 + Qm + Qa;
  const int64_t total = (int64_t)st->world * st->sh_capw;
  const float4* rec = reinterpret_cast<const float4*>(st->sh_window + st->sh_off_com[p]);
  const int32_t* cnt = reinterpret_cast<const int32_t*>(st->sh_window + st->sh_off_cnt[p]);
  k_shard_merge_key<<<blocks_for(total, 8), 256, 0, s>>>(rec, cnt, st->world, st->sh_capw, Qr, st->local_rows,
                                                         st->sh_keytab);
  k_shard_merge_apply<<<blocks_for(total * 32, 8), 256, 0, s>>>(rec, cnt, st->world, st->sh_capw, Qr,
                                                                st->local_rows, st->sh_keytab, Qm, Qa,
                                                                (float4*)st->mem, st->mem_ts, (float4*)st->mail,
                                                                st->mail_ts);
}

}  // namespace mspipe
