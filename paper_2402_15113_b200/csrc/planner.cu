// planner.cu — row F1: the minimal-staleness planner of MSPipe §3.2, host code.
//
// Five stages per iteration i (j = 1..5: sample, fetch feature, fetch memory,
// train, update memory) with profiled durations tau^(j).  Start times follow
// Eq. 3: stage 1 runs back to back; stage 2 shares the copy
// engine with stage 3 of the previous iteration; stages 3-5 wait for their own
// previous instance and the previous stage of the iteration.  A plan k_i adds
// the gate of Alg. 1 L8-L11 to stage 3: the fetch of iteration i
// starts after the update of iteration i - k_i ends (C1, reading F2).
// mspipe_plan_min_staleness picks, iteration by iteration, the least k_i in
// [1, min(i, k_max)) whose gated fetch still ends before the training stage
// would start (C2, reading F3); C3's k_max is an input (see
// mspipe_stale_histogram).  O(E * k_max) time, O(k_max) memory beyond the
// outputs: a ring of the last k_max update end times.
#include <vector>

#include "internal.cuh"

namespace {

struct Ends {  // e_{i-1}^(j) of the previous iteration and the update ring
  double e[6] = {0, 0, 0, 0, 0, 0};
};

// stage start/end times of iteration i given the previous iteration's ends;
// gate_end < 0: no gate
inline void stage_times(const double* tau, const Ends& prev, double gate_end, double* b, double* e) {
  for (int j = 1; j <= 5; ++j) {
    double s;
    if (j == 1) s = prev.e[1];
    else if (j == 2) s = e[1] > prev.e[3] ? e[1] : prev.e[3];
    else s = e[j - 1] > prev.e[j] ? e[j - 1] : prev.e[j];
    if (j == 3 && gate_end > s) s = gate_end;
    b[j] = s;
    e[j] = s + tau[j - 1];
  }
}

bool tau_ok(const double* tau) {
  if (!tau) return false;
  for (int j = 0; j < 5; ++j)
    if (!(tau[j] >= 0.0)) return false;
  return true;
}

}  // namespace

using namespace mspipe;

extern "C" {

mspipe_status mspipe_plan_timeline(const double* tau, int64_t num_iters, const int32_t* k, double* out_b,
                                   double* out_e) {
  if (!tau_ok(tau) || num_iters < 0 || (num_iters > 0 && (!out_b || !out_e)))
    return fail(MSPIPE_EINVAL, "plan_timeline: tau must be 5 values >= 0, num_iters >= 0, outputs non-NULL");
  Ends prev;
  for (int64_t i = 1; i <= num_iters; ++i) {
    double gate = -1.0;
    if (k) {
      const int64_t ki = k[i - 1];
      if (ki < 1) return fail(MSPIPE_EINVAL, "plan_timeline: k_%lld = %lld < 1", (long long)i, (long long)ki);
      if (i - ki >= 1) gate = out_e[(i - ki - 1) * 5 + 4];  // e_{i-k_i}^(5)
    }
    double b[6], e[6];
    stage_times(tau, prev, gate, b, e);
    for (int j = 1; j <= 5; ++j) {
      out_b[(i - 1) * 5 + j - 1] = b[j];
      out_e[(i - 1) * 5 + j - 1] = e[j];
      prev.e[j] = e[j];
    }
  }
  return MSPIPE_OK;
}

mspipe_status mspipe_plan_min_staleness(const double* tau, int64_t num_iters, int32_t k_max, int32_t* out_k,
                                        int64_t* out_infeasible_iter) {
  if (!tau_ok(tau) || num_iters < 0 || k_max < 1 || (num_iters > 0 && !out_k))
    return fail(MSPIPE_EINVAL, "plan_min_staleness: tau must be 5 values >= 0, num_iters >= 0, k_max >= 1");
  if (out_infeasible_iter) *out_infeasible_iter = 0;
  // ring of update end times e_{i'}^(5) for i' in (i - k_max, i)
  std::vector<double> upd_end((size_t)k_max + 1, 0.0);
  auto e5 = [&](int64_t it) { return it < 1 ? 0.0 : upd_end[(size_t)(it % (k_max + 1))]; };
  Ends prev;
  for (int64_t i = 1; i <= num_iters; ++i) {
    double b[6], e[6];
    stage_times(tau, prev, -1.0, b, e);  // the schedule with this iteration's gate relaxed
    const double latest_fetch_start = b[4] - tau[2];
    const int64_t hi = i < k_max ? i : k_max;  // k_i < min(i, k_max)
    int64_t ki = 0;
    for (int64_t c = 1; c < hi; ++c)
      if (e5(i - c) <= latest_fetch_start) {
        ki = c;
        break;
      }
    if (ki == 0) {
      if (i <= k_max || hi <= 1) {
        ki = i;  // warm-up: no gate ("will not wait")
      } else {
        ki = hi - 1;  // infeasible: the stalest allowed bound; C2 binds
        if (out_infeasible_iter && *out_infeasible_iter == 0) *out_infeasible_iter = i;
      }
    }
    out_k[i - 1] = (int32_t)ki;
    stage_times(tau, prev, i - ki >= 1 ? e5(i - ki) : -1.0, b, e);
    for (int j = 1; j <= 5; ++j) prev.e[j] = e[j];
    upd_end[(size_t)(i % (k_max + 1))] = e[5];
  }
  return MSPIPE_OK;
}

mspipe_status mspipe_plan_stale_fractions(const int64_t* hist, int32_t nbins, const int32_t* k_values,
                                          int32_t nk, double* out) {
  if (!hist || !k_values || !out || nbins < 2 || nk < 0)
    return mspipe::fail(MSPIPE_EINVAL, "plan_stale_fractions: NULL or nbins=%d nk=%d", nbins, nk);
  int64_t tot = 0;
  for (int32_t d = 0; d < nbins; ++d) tot += hist[d];
  for (int32_t q = 0; q < nk; ++q) {
    const int32_t k = k_values[q];
    if (k < 1) return mspipe::fail(MSPIPE_EINVAL, "plan_stale_fractions: k=%d < 1", k);
    int64_t stale = 0;  // bins d = 1 .. k-1 (the last bin holds d > max_d)
    for (int32_t d = 1; d <= k - 1 && d < nbins; ++d) stale += hist[d];
    out[q] = tot ? (double)stale / (double)tot : 0.0;
  }
  return MSPIPE_OK;
}

}  // extern "C"
