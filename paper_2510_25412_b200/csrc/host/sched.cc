// Inference scheduler batch formation (§4.4): Poisson-rate-sized batches of queued
// pred requests in FIFO order.  Rules in include/kvfs.h ("inference scheduler") and DESIGN.md reading S1.
#include <algorithm>
#include <cmath>
#include <deque>
#include <mutex>
#include <new>
#include <unordered_set>
#include <vector>

#include "../../../include/kvfs.h"

struct kvfs_sched {
  kvfs_sched_config cfg{};
  std::mutex mu;
  bool has_rate = false;
  double lam = 0.0, t_prev = 0.0;
  struct Req {
    int fd;
    std::vector<int32_t> pos;
    double t;
  };
  std::deque<Req> pool;

  int target() const {
    const double l = has_rate ? lam : 1.0 / cfg.dt_default;
    const double b = std::nearbyint(l * cfg.w_max);  // round half to even (default rounding mode)
    if (!(b >= 1.0)) return 1;
    if (b >= static_cast<double>(cfg.b_max)) return cfg.b_max;
    return static_cast<int>(b);
  }
};

extern "C" {

int kvfs_sched_create(const kvfs_sched_config *cfg, kvfs_sched **out) {
  if (!cfg || !out || !(cfg->w_max > 0) || cfg->b_max < 1 || !(cfg->alpha > 0) || cfg->alpha > 1 ||
      !(cfg->dt_default > 0))
    return KVFS_EINVAL;
  auto *s = new (std::nothrow) kvfs_sched();
  if (!s) return KVFS_ENOMEM;
  s->cfg = *cfg;
  *out = s;
  return KVFS_OK;
}

int kvfs_sched_destroy(kvfs_sched *s) {
  if (!s) return KVFS_EINVAL;
  delete s;
  return KVFS_OK;
}

// No exception crosses the C ABI (include/kvfs.h conventions): the allocating steps run first, inside a
// function-try-block, and the queue is changed only after they succeeded (strong guarantee).
int kvfs_sched_enqueue(kvfs_sched *s, int fd, int n_q, const int32_t *pos, double now) try {
  if (!s || n_q < 0 || (n_q > 0 && !pos)) return KVFS_EINVAL;
  kvfs_sched::Req req{fd, std::vector<int32_t>(pos, pos + n_q), now};
  std::lock_guard<std::mutex> lk(s->mu);
  s->pool.push_back(std::move(req));  // may throw (strong guarantee): before the rate changes
  if (!s->has_rate) {
    s->lam = 1.0 / s->cfg.dt_default;
    s->has_rate = true;
  } else {
    const double dt = std::max(now - s->t_prev, 1e-9);
    s->lam = (1.0 - s->cfg.alpha) * s->lam + s->cfg.alpha / dt;
  }
  s->t_prev = now;
  return KVFS_OK;
} catch (...) {  // std::bad_alloc building or queueing the request: nothing changed
  return KVFS_ENOMEM;
}

int kvfs_sched_state(kvfs_sched *s, double *lambda, int *target, int *n_waiting) {
  if (!s) return KVFS_EINVAL;
  std::lock_guard<std::mutex> lk(s->mu);
  if (lambda) *lambda = s->has_rate ? s->lam : 1.0 / s->cfg.dt_default;
  if (target) *target = s->target();
  if (n_waiting) *n_waiting = static_cast<int>(s->pool.size());
  return KVFS_OK;
}

int kvfs_sched_form(kvfs_sched *s, double now, pred_desc *descs, int desc_cap, int32_t *pos, int64_t pos_cap,
                    int *n_desc, int64_t *n_rows) try {
  if (!s || !n_desc || !n_rows) return KVFS_EINVAL;
  std::lock_guard<std::mutex> lk(s->mu);
  if (s->pool.empty()) return 0;
  if (static_cast<int>(s->pool.size()) < s->target() && now - s->pool.front().t < s->cfg.w_max) return 0;
  // choose: FIFO, at most b_max, one request per fd
  std::vector<size_t> take;
  std::unordered_set<int> seen;
  int64_t rows = 0;
  for (size_t i = 0; i < s->pool.size() && static_cast<int>(take.size()) < s->cfg.b_max; ++i) {
    if (seen.count(s->pool[i].fd)) continue;
    seen.insert(s->pool[i].fd);
    take.push_back(i);
    rows += static_cast<int64_t>(s->pool[i].pos.size());
  }
  if (static_cast<int>(take.size()) > desc_cap || rows > pos_cap || (!take.empty() && !descs) ||
      (rows > 0 && !pos))
    return KVFS_ENOMEM;
  int64_t r = 0;
  for (size_t j = 0; j < take.size(); ++j) {
    const auto &q = s->pool[take[j]];
    descs[j] = {q.fd, static_cast<int32_t>(q.pos.size())};
    std::copy(q.pos.begin(), q.pos.end(), pos + r);
    r += static_cast<int64_t>(q.pos.size());
  }
  std::deque<kvfs_sched::Req> rest;
  size_t k = 0;
  for (size_t i = 0; i < s->pool.size(); ++i) {
    if (k < take.size() && take[k] == i) {
      ++k;
      continue;
    }
    rest.push_back(s->pool[i]);  // a copy: if it throws, the queue is intact
  }
  s->pool.swap(rest);
  *n_desc = static_cast<int>(take.size());
  *n_rows = rows;
  return 1;
} catch (...) {
  return KVFS_ENOMEM;
}

}  // extern "C"
