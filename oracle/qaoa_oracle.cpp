/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the B200 backend.
 *
 * A plain C++ restatement of the reference's accelerated (numba) kernel set and
 * the orchestration around it, used by tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py as the checker / CPU baseline.  Never part of the
 * product path.  Compiled with -ffp-contract=off and glibc libm so the
 * arithmetic is the numba set's (no FMA contraction, same cos/sin), which makes
 * its outputs bit-identical to the reference; tests/test_oracle_golden.py pins
 * it against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py).  Parallel loops run on a persistent std::thread
 * pool (static chunks); reductions keep the reference's neighbour-pair association, so the
 * thread count never changes a result.
 *
 * Each function cites the reference source it restates
 * (/root/reference/pkg/src/qaoasim/...).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <condition_variable>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

namespace {

struct c128 {
  double re, im;
};

int g_threads = 0;  // 0: all hardware threads

int threads_now() {
  if (g_threads > 0) return g_threads;
  unsigned h = std::thread::hardware_concurrency();
  return h ? (int)h : 1;
}

// Persistent worker pool (like numba's workqueue layer, numba_impl.py:24, the
// reference's threads live across kernel calls): spawning threads per call would
// add tens of microseconds to each of the reference's ~10^3 whole-array passes.
class Pool {
 public:
  explicit Pool(int workers) {
    for (int t = 1; t <= workers; ++t) th_.emplace_back([this, t] { loop(t); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int size() const { return (int)th_.size() + 1; }
  // job(t) for t in [0, size()): the caller runs t = 0
  void run(const std::function<void(int)>& job) {
    {
      std::lock_guard<std::mutex> g(m_);
      job_ = &job;
      pending_ = (int)th_.size();
      ++gen_;
    }
    cv_.notify_all();
    job(0);
    std::unique_lock<std::mutex> g(m_);
    done_.wait(g, [this] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  void loop(int t) {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int)>* job;
      {
        std::unique_lock<std::mutex> g(m_);
        cv_.wait(g, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
        job = job_;
      }
      (*job)(t);
      std::lock_guard<std::mutex> g(m_);
      if (--pending_ == 0) done_.notify_one();
    }
  }
  std::vector<std::thread> th_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* job_ = nullptr;
  uint64_t gen_ = 0;
  int pending_ = 0;
  bool stop_ = false;
};

Pool& pool() {
  static std::unique_ptr<Pool> p;
  static int size = 0;
  const int T = threads_now();
  if (!p || size != T) {
    p.reset();
    p.reset(new Pool(T - 1));
    size = T;
  }
  return *p;
}

// static-schedule parallel loop: f(i) for i in [0, n); `grain` = iterations below
// which the loop runs on the calling thread (elementwise loops: 16384 elements; the
// blocked reductions: a few 2048-element blocks -- numba's prange splits those too)
template <class F>
void parallel_for(int64_t n, F f, int64_t grain = 16384) {
  const int T = threads_now();
  if (T <= 1 || n < grain) {
    for (int64_t i = 0; i < n; ++i) f(i);
    return;
  }
  const int64_t chunk = (n + T - 1) / T;
  pool().run([&](int t) {
    const int64_t lo = t * chunk, hi = std::min<int64_t>(n, lo + chunk);
    for (int64_t i = lo; i < hi; ++i) f(i);
  });
}

constexpr uint64_t BLOCK = 2048;  // numba_impl.py:26 (any power of two gives the same tree)

// numba_impl.py:89-97: in-place neighbour-pair fold of a full power-of-two block
double block_tree(double* buf, uint64_t m) {
  for (uint64_t w = m >> 1; w >= 1; w >>= 1)
    for (uint64_t i = 0; i < w; ++i) buf[i] = buf[2 * i] + buf[2 * i + 1];
  return buf[0];
}

// numba_impl.py:100-111: pairwise fold of partials with an implicit 0.0 pad
double fold(std::vector<double> cur) {
  uint64_t m = cur.size();
  while (m > 1) {
    const uint64_t half = (m + 1) >> 1;
    for (uint64_t i = 0; i < half; ++i) cur[i] = cur[2 * i] + (2 * i + 1 < m ? cur[2 * i + 1] : 0.0);
    m = half;
  }
  return cur[0];
}

// blocked tree over a 2-component element generator g(i, &re, &im)
template <class G>
void tree2(G g, uint64_t len, double* out_re, double* out_im) {
  const uint64_t nb = (len + BLOCK - 1) / BLOCK;
  std::vector<double> pre(nb), pim(nb);
  parallel_for(
      (int64_t)nb,
      [&](int64_t b) {
        double br[BLOCK], bi[BLOCK];
        memset(br, 0, sizeof(br));
        memset(bi, 0, sizeof(bi));
        const uint64_t s = (uint64_t)b * BLOCK, e = std::min(s + BLOCK, len);
        for (uint64_t i = s; i < e; ++i) g(i, &br[i - s], &bi[i - s]);
        pre[b] = block_tree(br, BLOCK);
        pim[b] = block_tree(bi, BLOCK);
      },
      8);
  *out_re = fold(pre);
  *out_im = fold(pim);
}

uint64_t mix64(uint64_t z) {  // rng.py:22-27
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

double uniform_at(uint64_t seed, uint64_t t) {  // rng.py:30-37
  return (double)(mix64(seed + (t + 1) * 0x9E3779B97F4A7C15ull) >> 11) * (1.0 / 9007199254740992.0);
}

}  // namespace

extern "C" {

void or_set_num_threads(int k) { g_threads = k; }
int or_num_threads(void) { return threads_now(); }

// numba_impl.py:40-44
void or_fill_plus(c128* a, uint64_t len) {
  const double v = 1.0 / sqrt((double)len);
  parallel_for((int64_t)len, [&](int64_t i) { a[i] = {v, 0.0}; });
}

// numba_impl.py:47-51: ang = -gamma * t; a *= complex(cos(ang), sin(ang))
void or_phase_by_table(c128* a, const double* t, uint64_t len, double gamma) {
  const double ng = -gamma;
  parallel_for((int64_t)len, [&](int64_t i) {
    const double ang = ng * t[i];
    const double c = cos(ang), s = sin(ang);
    const c128 x = a[i];
    a[i] = {x.re * c - x.im * s, x.re * s + x.im * c};
  });
}

// numba_impl.py:54-57
void or_diag_scale(c128* a, const double* t, uint64_t len) {
  parallel_for((int64_t)len, [&](int64_t i) { a[i] = {a[i].re * t[i], a[i].im * t[i]}; });
}

// numba_impl.py:60-72: pair (i0, i0 | 2^j); c*t + (-is)*u, (-is)*t + c*u
void or_rx_qubit(c128* a, uint64_t len, int j, double c, double s) {
  const uint64_t low = (1ull << j) - 1ull, bit = 1ull << j;
  parallel_for((int64_t)(len >> 1), [&](int64_t k) {
    const uint64_t i0 = (((uint64_t)k & ~low) << 1) | ((uint64_t)k & low), i1 = i0 | bit;
    const c128 t = a[i0], u = a[i1];
    a[i0] = {c * t.re + s * u.im, c * t.im - s * u.re};
    a[i1] = {s * t.im + c * u.re, c * u.im - s * t.re};
  });
}

// numba_impl.py:75-86
void or_weighted_probs(const c128* a, const double* t, double* out, uint64_t len) {
  parallel_for((int64_t)len, [&](int64_t i) { out[i] = t[i] * (a[i].re * a[i].re + a[i].im * a[i].im); });
}

void or_probs(const c128* a, double* out, uint64_t len) {
  parallel_for((int64_t)len, [&](int64_t i) { out[i] = a[i].re * a[i].re + a[i].im * a[i].im; });
}

// numba_impl.py:114-126
double or_tree_sum(const double* v, uint64_t len) {
  double re, im;
  tree2([&](uint64_t i, double* r, double* m) { *r = v[i]; *m = 0.0; }, len, &re, &im);
  return re;
}

// numba_impl.py:129-144 (serial scans)
double or_reduce_min(const double* v, uint64_t len) {
  double m = v[0];
  for (uint64_t i = 1; i < len; ++i)
    if (v[i] < m) m = v[i];
  return m;
}

double or_reduce_max(const double* v, uint64_t len) {
  double m = v[0];
  for (uint64_t i = 1; i < len; ++i)
    if (v[i] > m) m = v[i];
  return m;
}

// numba_impl.py:147-170: sum conj(a) b in real arithmetic
void or_inner(const c128* a, const c128* b, uint64_t len, double* out2) {
  tree2(
      [&](uint64_t i, double* r, double* m) {
        const c128 p = a[i], q = b[i];
        *r = p.re * q.re + p.im * q.im;
        *m = p.re * q.im - p.im * q.re;
      },
      len, &out2[0], &out2[1]);
}

// numba_impl.py:173-197
void or_diag_inner(const c128* a, const double* t, const c128* b, uint64_t len, double* out2) {
  tree2(
      [&](uint64_t i, double* r, double* m) {
        const c128 p = a[i], q = b[i];
        *r = (p.re * q.re + p.im * q.im) * t[i];
        *m = (p.re * q.im - p.im * q.re) * t[i];
      },
      len, &out2[0], &out2[1]);
}

// numba_impl.py:200-226: per qubit a full tree, then total += in ascending j
void or_xsum(const c128* a, const c128* b, uint64_t len, int nq, double* out2) {
  double re = 0.0, im = 0.0;
  for (int j = 0; j < nq; ++j) {
    const uint64_t bit = 1ull << j;
    double r, m;
    tree2(
        [&](uint64_t i, double* rr, double* mm) {
          const c128 p = a[i], q = b[i ^ bit];
          *rr = p.re * q.re + p.im * q.im;
          *mm = p.re * q.im - p.im * q.re;
        },
        len, &r, &m);
    re += r;
    im += m;
  }
  out2[0] = re;
  out2[1] = im;
}

// numba_impl.py:229-238: term-ordered sum from 0.0
void or_precompute_table(const double* w, const int64_t* m, uint64_t nterms, double* out, uint64_t len) {
  parallel_for((int64_t)len, [&](int64_t x) {
    double acc = 0.0;
    for (uint64_t k = 0; k < nterms; ++k)
      if (((uint64_t)x & (uint64_t)m[k]) == (uint64_t)m[k]) acc += w[k];
    out[x] = acc;
  });
}

// numba_impl.py:241-244
void or_pairwise_level(const double* src, double* dst, uint64_t dst_len) {
  parallel_for((int64_t)dst_len, [&](int64_t i) { dst[i] = src[2 * i] + src[2 * i + 1]; });
}

// backend.py:200-207: c, s on the host, qubits ascending
static void rx_layer(c128* a, int n, double theta) {
  const double c = cos(theta / 2.0), s = sin(theta / 2.0);
  for (int j = 0; j < n; ++j) or_rx_qubit(a, 1ull << n, j, c, s);
}

// circuit.py:98-103
void or_simulate(const double* table, c128* a, int n, int p, const double* gammas, const double* betas) {
  const uint64_t len = 1ull << n;
  or_fill_plus(a, len);
  for (int i = 0; i < p; ++i) {
    or_phase_by_table(a, table, len, gammas[i]);
    rx_layer(a, n, -2.0 * betas[i]);
  }
}

// circuit.py:106-113, without the clamp
double or_expectation(const double* table, const c128* a, int n) {
  const uint64_t len = 1ull << n;
  std::vector<double> w(len);
  or_weighted_probs(a, table, w.data(), len);
  return or_tree_sum(w.data(), len);
}

// adjoint.py:37-77; ket holds the forward state on entry, bra is scratch
void or_gradient(const double* table, c128* ket, c128* bra, int n, int p, const double* gammas, const double* betas,
                 double* dg, double* db) {
  const uint64_t len = 1ull << n;
  memcpy(bra, ket, len * sizeof(c128));
  or_diag_scale(bra, table, len);
  for (int i = p - 1; i >= 0; --i) {
    double xs[2], di[2];
    or_xsum(bra, ket, len, n, xs);
    db[i] = -2.0 * xs[1];
    rx_layer(bra, n, 2.0 * betas[i]);
    rx_layer(ket, n, 2.0 * betas[i]);
    or_diag_inner(bra, table, ket, len, di);
    dg[i] = 2.0 * di[1];
    or_phase_by_table(bra, table, len, -gammas[i]);
    or_phase_by_table(ket, table, len, -gammas[i]);
  }
}

// rng.py:40-47
void or_uniform(uint64_t seed, uint64_t start, uint64_t count, double* out) {
  for (uint64_t t = 0; t < count; ++t) out[t] = uniform_at(seed, start + t);
}

// backend.py:261-299 + sampling.py:23-30: every pairwise level, one descent per
// shot.  Returns 0, or 1 when |root - 1| > 1e-9 (*total is set either way).
int or_sample(const c128* a, const double* table, int n, uint64_t shots, uint64_t seed, int64_t* idx, double* cost,
              double* total) {
  const uint64_t len = 1ull << n;
  std::vector<std::vector<double>> lv(n + 1);
  lv[0].resize(len);
  or_probs(a, lv[0].data(), len);
  for (int l = 1; l <= n; ++l) {
    lv[l].resize(len >> l);
    or_pairwise_level(lv[l - 1].data(), lv[l].data(), len >> l);
  }
  const double root = lv[n][0];
  *total = root;
  if (fabs(root - 1.0) > 1e-9) return 1;
  parallel_for((int64_t)shots, [&](int64_t s) {
    double u = uniform_at(seed, (uint64_t)s) * root;
    uint64_t k = 0;
    for (int l = n - 1; l >= 0; --l) {
      const double left = lv[l][2 * k];
      const bool right = u >= left;
      if (right) u = u - left;
      k = 2 * k + (right ? 1 : 0);
    }
    idx[s] = (int64_t)k;
    if (cost) cost[s] = table[k];
  });
  return 0;
}

}  // extern "C"
