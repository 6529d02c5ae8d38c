// lg_ic0.cu -- IC(0) factorization (host, bit-exact) and the device apply.
//
// Factorization: ic0.py:48-116.  The reference builds each row i of L as a
// dict, subtracting sum_p l_ip l_kp over the common pattern for every lower
// entry k of the row (ic0.py:56-71).  Whichever dict it iterates, the
// subtraction runs in ascending p, so a sorted-merge restatement with the
// same operation order (s -= l_ip * l_kp; l_ik = s / l_kk; d = diag*(1+alpha);
// d -= l_ip^2; l_ii = sqrt(d)) reproduces the factor bit for bit when built
// without FMA contraction (-ffp-contract=off, see build.py).
//
// Apply: ic0.py:40-45 solves L y = r then L^T z = y (SuperLU, natural
// ordering).  On the GPU each triangular sweep is a dependency DAG: 227
// levels on C4, 476 on C3, 72 on C2; its time is depth x dependency hop, not
// bytes.  What this file does about it, in order of appearance:
//   * host: the sweep's system is rewritten into a level-merged form
//     (merge_levels: auxiliary partial sums + the level below substituted in;
//     ~0.6x the depth for ~1.5x the entries, exact in real arithmetic), hub
//     rows get their deepest inputs first, and the rows are permuted into
//     processing order and packed into warp tasks -- 32/L rows of one length
//     class (L = 1 ... 32 lanes per row, chosen per level width), or a
//     256-entry chunk of a hub row whose partials chunk 0 sums in chunk order;
//   * device, default: the dataflow sweep (sweep_flow_kernel) -- no barriers,
//     the solution vector is its own dependency flag, one cooperative
//     persistent launch per triangle;
//   * device, kept for comparison / tracing (LG_SWEEP_MODE=0, lg_ic0_trace):
//     the level-barrier sweep (sweep_kernel: grid barriers after wide levels,
//     runs of narrow levels on one cluster);
//   * device, opt-in (LG_SWEEP_CTA=1): the resident sweep (sweep_cta_kernel:
//     both triangles in one CTA).
// All three run the same schedule with the same per-row summation order
// (lane-strided, butterfly), so they agree bit for bit and z is reproducible.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <omp.h>

#include "lg_common.cuh"

namespace lg {

constexpr int kSweepThreads = 512;          // 16 warps per CTA
constexpr int kSweepWarps = kSweepThreads / 32;
constexpr int kHubChunk = 256;              // nonzeros per hub-row chunk task
constexpr int kSegSmem = 1024;              // level segments kept in shared memory

struct SweepTask {
  int32_t p;  // pack: first permuted row          | chunk: permuted hub row
  int32_t b;  // pack: lanes << 8 | count          | chunk: 0
  int32_t c;  // chunk: chunk index
  int32_t d;  // chunk: hub-row id
};

struct SweepSeg {
  int32_t t0, t1;   // task range
  int32_t narrow;   // 1: run by the first cluster alone
  int32_t barrier;  // 1: grid barrier follows, 2: cluster barrier follows
  int32_t run_t1;   // end task of the maximal run of same-mode segments
  int32_t pad;
};

struct RowInfo {   // per permuted row position (dataflow sweep)
  double dg;       // diagonal
  int32_t xrow;    // row of x written (factor numbering)
  int32_t bidx;    // index of b read
};

// Device data of one sweep direction.  Rows are stored PERMUTED into
// processing order (level, length class), so a level's nonzeros are one
// contiguous stream and a task needs one row-pointer load.
struct SweepDev {
  int64_t* prp = nullptr;    // permuted strictly-triangular row pointers
  int32_t* pcol = nullptr;   // columns (original numbering)
  double* pval = nullptr;
  int32_t* perm = nullptr;   // permuted position -> original row
  double* pdiag = nullptr;   // diagonal in permuted order
  SweepTask* tasks = nullptr;
  int64_t* tbase = nullptr;
  uint16_t* lanetab = nullptr;
  SweepSeg* segs = nullptr;
  int32_t* hub_first = nullptr;   // first partial slot of each hub row
  int32_t* hub_nchunk = nullptr;
  unsigned* hub_ticket = nullptr;
  double* hub_part = nullptr;
  unsigned long long* bar = nullptr;
  int32_t* tlevel = nullptr;      // level of every task
  int32_t* lexpect = nullptr;     // [levels * 32] tasks per (level, shard)
  unsigned* lcount = nullptr;     // [levels * 32] completion counters
  unsigned long long* ttrace = nullptr;   // debug: dataflow per-task timestamps
  RowInfo* rinfo = nullptr;       // dataflow row records, permuted order
  int32_t* oidx = nullptr;        // permuted row -> second-output index (or NULL)
  void* cdesc = nullptr;          // [ntasks] CtaDesc records (resident sweep)
  int32_t* lhub0 = nullptr;       // [levels + 1] first hub-row id of each level (resident sweep)
  int32_t* hub_prow = nullptr;    // [hub rows] permuted row of each hub row
  int32_t* ubidx = nullptr;       // unknown -> b index (-1: auxiliary unknown)
  int32_t* uoidx = nullptr;       // unknown -> output index (-1: none)
  int32_t n = 0;             // rows of the factor
  int32_t N = 0;             // unknowns of the sweep (entries with col >= N read the right-hand side)
  int64_t nent = 0;          // entries the sweep streams (after level merging)
  int32_t ntasks = 0;
  int32_t nparts = 0;        // hub partial slots
  int32_t nsegs = 0;
  int32_t nbar = 0;          // grid barriers per sweep
  int levels = 0;            // depth of the sweep's DAG as scheduled (after level merging)
  int flevels = 0;           // depth of the factor's own DAG
};

}  // namespace lg

struct lg_ic0 {
  int64_t n = 0, nnz_l = 0;  // nnz_l counts the diagonal
  unsigned long long* trace = nullptr;  // debug timestamps (fwd segs, bwd segs)
  lg::SweepDev fwd, bwd;
  double* diag = nullptr;
  double* tmp = nullptr;     // forward sweep's unknowns [fwd.N]: its first n are L^{-1} r
  double* xb = nullptr;      // backward sweep's unknowns [bwd.N]; z is written through oidx
  int grid = 0;
  // dataflow sweeps hand their scratch state to each other: the forward
  // sweep re-arms the backward one (x sentinels, counters, hub slots) and
  // vice versa, so an apply is exactly two launches; false after a
  // level-barrier apply (the state then needs one explicit re-arm)
  mutable bool flow_armed = false;
  // 1: both sweeps run as one resident CTA (opt-in), 0: dataflow sweeps
  int cta_mode = 0;
  int cta_threads = 0;
};

namespace lg {

// ------------------------------------------------------------ host side --
// One no-fill factorization pass (ic0.py:48-78).  Returns true on success.
// lrp/lcol describe the lower pattern of A plus the diagonal (last per row);
// lval receives the factor.
#pragma GCC push_options
#pragma GCC optimize("fp-contract=off")
// Row i of the factor, given rows < i (ic0.py:56-78): for each lower entry
// k of row i (ascending), s = a_ik - sum_p l_ip l_kp over the common pattern
// in ascending p, l_ik = s / l_kk; then l_ii = sqrt(diag (1 + alpha) -
// sum_k l_ik^2).  The common p are enumerated in ascending order whichever
// row is walked (the shorter one; p looked up in the other by binary search
// or a linear advance), so the arithmetic -- hence every bit -- is the
// reference's.  Returns false on a pivot below the floor.
static inline bool ic0_row(int64_t i, const std::vector<double>& diag,
                           const std::vector<int64_t>& lrp, const std::vector<int64_t>& lcol,
                           const std::vector<double>& aval, double alpha,
                           std::vector<double>& lval, int64_t* stamp, int64_t* pos) {
  const double floor_ = 1e-14;  // _PIVOT_FLOOR, ic0.py:17
  const int64_t lo = lrp[i], hi = lrp[i + 1] - 1;  // hi: diagonal slot
  const int64_t* C = lcol.data();
  for (int64_t t = lo; t < hi; ++t) {
    stamp[C[t]] = i;
    pos[C[t]] = t;
  }
  for (int64_t t = lo; t < hi; ++t) {
    const int64_t k = C[t];
    double s = aval[t];
    const int64_t klo = lrp[k], khi = lrp[k + 1] - 1;  // row k strictly lower
    const int64_t nli = t - lo, nk = khi - klo;
    if (nli <= nk) {
      // walk the computed prefix of row i (ascending p), find p in row k
      int64_t q = klo;
      for (int64_t u = lo; u < t; ++u) {
        const int64_t p = C[u];
        if (nk > 32) q = std::lower_bound(C + q, C + khi, p) - C;
        else
          while (q < khi && C[q] < p) ++q;
        if (q < khi && C[q] == p) s -= lval[u] * lval[q];
      }
    } else {
      // walk row k (ascending p), look p up in row i's computed prefix
      // (stamp / pos: this thread's map of row i's columns)
      for (int64_t q = klo; q < khi; ++q) {
        const int64_t p = C[q];
        if (stamp[p] == i && pos[p] < t) s -= lval[pos[p]] * lval[q];
      }
    }
    lval[t] = s / lval[khi];
  }
  const double scaled = diag[i] * (1.0 + alpha);
  double d = scaled;
  for (int64_t t = lo; t < hi; ++t) d -= lval[t] * lval[t];
  if (d <= floor_ * std::fabs(scaled) || d <= 0.0) return false;
  lval[hi] = std::sqrt(d);
  return true;
}

// One no-fill factorization pass (ic0.py:48-78).  Returns true on success.
// lrp/lcol describe the lower pattern of A plus the diagonal (last per row);
// lval receives the factor.  Rows of one dependency level (rows whose lower
// neighbours all sit in earlier levels) are independent, so a level's rows
// are factored in parallel (OpenMP) -- every row still reads exactly the
// finished rows it reads in the sequential order, so the factor is the same
// bit for bit.  order / lstart: rows grouped by level.
static bool ic0_attempt(int64_t n, const std::vector<double>& diag,
                        const std::vector<int64_t>& lrp,
                        const std::vector<int64_t>& lcol,
                        const std::vector<double>& aval, double alpha,
                        std::vector<double>& lval, const std::vector<int64_t>& order,
                        const std::vector<int64_t>& lstart,
                        std::vector<std::vector<int64_t>>& maps) {
  const int64_t nlev = (int64_t)lstart.size() - 1;
  for (auto& m : maps) std::fill(m.begin(), m.end(), (int64_t)-1);
  for (int64_t L = 0; L < nlev; ++L) {
    const int64_t a = lstart[(size_t)L], b = lstart[(size_t)L + 1];
    int ok = 1;
    if (b - a >= 64 && maps.size() > 1) {
#pragma omp parallel num_threads((int)maps.size()) reduction(min : ok)
      {
        int64_t* st = maps[(size_t)omp_get_thread_num()].data();
#pragma omp for schedule(dynamic, 16)
        for (int64_t q = a; q < b; ++q)
          if (!ic0_row(order[(size_t)q], diag, lrp, lcol, aval, alpha, lval, st, st + n)) ok = 0;
      }
    } else {
      int64_t* st = maps[0].data();
      for (int64_t q = a; q < b && ok; ++q)
        if (!ic0_row(order[(size_t)q], diag, lrp, lcol, aval, alpha, lval, st, st + n)) ok = 0;
    }
    if (!ok) return false;
  }
  return true;
}
#pragma GCC pop_options

// A triangular sweep as the device runs it: N unknowns -- the factor's n rows
// first, auxiliary partial sums after them -- each computed as
//     y_u = (b[bidx_u] - sum_k val_k * src_k) / dg_u
// where an entry's source is an unknown (col < N) or the right-hand side (a
// "b entry", col = N + index into b; during the transformation -1 - index).
// `order` is a topological order of the unknowns.  For an auxiliary unknown
// bidx = -1 (no right-hand side), dg = -1 (y = the plain sum) and oidx = -1.
struct SweepSys {
  int64_t n = 0, N = 0;
  std::vector<int64_t> rp;
  std::vector<int32_t> col;
  std::vector<double> val;
  std::vector<double> dg;
  std::vector<int32_t> bidx, oidx, order;
};

static int dag_levels(const SweepSys& s, std::vector<int32_t>& level) {
  level.assign((size_t)s.N, 0);
  int maxl = 0;
  for (int64_t q = 0; q < s.N; ++q) {
    const int32_t i = s.order[(size_t)q];
    int l = 0;
    for (int64_t k = s.rp[(size_t)i]; k < s.rp[(size_t)i + 1]; ++k) {
      const int32_t c = s.col[(size_t)k];   // b entries: negative, or >= N once encoded
      if (c >= 0 && c < s.N) l = std::max(l, level[(size_t)c] + 1);
    }
    level[(size_t)i] = l;
    maxl = std::max(maxl, l);
  }
  return s.N ? maxl + 1 : 0;
}

// Level merging (one pass takes ~30 % off the depth of a sweep's dependency
// DAG for ~20 % more entries).  A sweep's time is its DAG depth times the
// dependency hop (~1.6 us), not its bytes, and on power-law graphs the long
// chains run through hub rows.  Two rewrites, both exact in real arithmetic:
//  * split: an odd-level unknown j with at least kSplitMin (12: measured best
//    of 2 ... 32; fewer auxiliary rows than at 4, C4 539 -> 515 us) inputs below
//    the level just under it gets an auxiliary unknown p_j = sum of those early
//    terms (ready a level sooner); row j keeps p_j and its late inputs.
//  * substitute: in a row i of an even level every input j on the level just
//    below is replaced by j's own equation, a_ij y_j = c b_j - c p_j -
//    sum_late c a_jk y_k with c = a_ij / d_j (short rows j without a p_j are
//    substituted whole; long ones stay and keep their hop).  Row i then reads
//    the right-hand side at j -- a b entry, which never waits -- and inputs two
//    levels down: even rows chain to even rows.
// The rewritten system has the same form, so passes compose (at most
// LG_IC0_MERGE passes, default 3: two wherever the DAG is latency-bound, a
// third on narrow DAGs; 0 keeps the factor's own sweep).  Results equal the plain
// sweep's to roundoff (coefficient products are rounded once on the host), not
// bitwise.
static int64_t env_i64(const char* name, int64_t dflt) {
  const char* e = getenv(name);
  return e ? (int64_t)atoll(e) : dflt;
}
// rows up to kMergeLen entries are substituted whole; kSplitMin early inputs
// earn an auxiliary unknown (LG_IC0_MERGELEN / LG_IC0_SPLITMIN override)
static int64_t merge_len() { return env_i64("LG_IC0_MERGELEN", 16); }
static int64_t split_min() { return env_i64("LG_IC0_SPLITMIN", 12); }

constexpr int64_t kMergeWide = 16384;   // mean rows per level beyond which a sweep is not latency-bound
constexpr int64_t kMergeNarrow = 2048;  // ... up to which a third pass still pays

static bool merge_levels(SweepSys& s, int64_t max_rows_per_level) {
  std::vector<int32_t> level;
  const int depth = dag_levels(s, level);
  const int64_t N = s.N;
  const int64_t kMergeLen = merge_len(), kSplitMin = split_min();
  // a shallow, wide DAG (the multicolour factor: 26 levels of ~38 k rows on C4)
  // is bound by its entries, not its depth: merging only adds work there
  // (measured: C4 multicolour DACG iteration 424 -> 620 us)
  if (N > max_rows_per_level * (int64_t)depth) return false;
  auto early = [&](int64_t j, int64_t k) {   // entry k of row j is not on the level just below
    const int32_t c = s.col[(size_t)k];
    return c < 0 || level[(size_t)c] < level[(size_t)j] - 1;
  };
  std::vector<int32_t> aux((size_t)N, -1);
  int64_t na = 0;
  for (int64_t q = 0; q < N; ++q) {
    const int32_t j = s.order[(size_t)q];
    if (!(level[(size_t)j] & 1)) continue;
    int64_t ne = 0;
    for (int64_t k = s.rp[(size_t)j]; k < s.rp[(size_t)j + 1]; ++k) ne += early(j, k);
    if (ne >= kSplitMin) aux[(size_t)j] = (int32_t)(N + na++);
  }
  const int64_t NN = N + na;
  // how an entry (i, k) of an even-level row is rewritten
  auto subst = [&](int64_t i, int64_t k) {
    const int32_t j = s.col[(size_t)k];
    if (j < 0 || (level[(size_t)i] & 1) || level[(size_t)j] != level[(size_t)i] - 1) return 0;
    if (aux[(size_t)j] >= 0) return 2;                                   // through p_j
    return s.rp[(size_t)j + 1] - s.rp[(size_t)j] <= kMergeLen ? 1 : 0;   // whole row
  };
  std::vector<int64_t> nrp((size_t)NN + 1, 0);
  for (int64_t i = 0; i < N; ++i) {
    int64_t len = 0;
    if (aux[(size_t)i] >= 0) {
      int64_t ne = 0;
      for (int64_t k = s.rp[(size_t)i]; k < s.rp[(size_t)i + 1]; ++k) ne += early(i, k);
      len = 1 + (s.rp[(size_t)i + 1] - s.rp[(size_t)i] - ne);
      nrp[(size_t)aux[(size_t)i] + 1] = ne;
    } else {
      for (int64_t k = s.rp[(size_t)i]; k < s.rp[(size_t)i + 1]; ++k) {
        const int how = subst(i, k);
        if (!how) {
          ++len;
          continue;
        }
        const int32_t j = s.col[(size_t)k];
        len += s.bidx[(size_t)j] >= 0;
        if (how == 1) {
          len += s.rp[(size_t)j + 1] - s.rp[(size_t)j];
        } else {
          ++len;
          for (int64_t q = s.rp[(size_t)j]; q < s.rp[(size_t)j + 1]; ++q) len += !early(j, q);
        }
      }
    }
    nrp[(size_t)i + 1] = len;
  }
  for (int64_t i = 0; i < NN; ++i) nrp[(size_t)i + 1] += nrp[(size_t)i];
  std::vector<int32_t> ncol((size_t)nrp[(size_t)NN]);
  std::vector<double> nval((size_t)nrp[(size_t)NN]);
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t i = 0; i < N; ++i) {
    int64_t w = nrp[(size_t)i];
    auto put = [&](int32_t c, double v) {
      ncol[(size_t)w] = c;
      nval[(size_t)w++] = v;
    };
    if (aux[(size_t)i] >= 0) {
      int64_t wa = nrp[(size_t)aux[(size_t)i]];
      put(aux[(size_t)i], 1.0);
      for (int64_t k = s.rp[(size_t)i]; k < s.rp[(size_t)i + 1]; ++k) {
        if (early(i, k)) {
          ncol[(size_t)wa] = s.col[(size_t)k];
          nval[(size_t)wa++] = s.val[(size_t)k];
        } else {
          put(s.col[(size_t)k], s.val[(size_t)k]);
        }
      }
      continue;
    }
    for (int64_t k = s.rp[(size_t)i]; k < s.rp[(size_t)i + 1]; ++k) {
      const int how = subst(i, k);
      const int32_t j = s.col[(size_t)k];
      if (!how) {
        put(j, s.val[(size_t)k]);
        continue;
      }
      const double c = s.val[(size_t)k] / s.dg[(size_t)j];
      if (s.bidx[(size_t)j] >= 0) put(-1 - s.bidx[(size_t)j], c);
      if (how == 2) put(aux[(size_t)j], -c);
      for (int64_t q = s.rp[(size_t)j]; q < s.rp[(size_t)j + 1]; ++q)
        if (how == 1 || !early(j, q)) put(s.col[(size_t)q], -(c * s.val[(size_t)q]));
    }
  }
  std::vector<int32_t> norder;
  norder.reserve((size_t)NN);
  for (int64_t q = 0; q < N; ++q) {
    const int32_t u = s.order[(size_t)q];
    if (aux[(size_t)u] >= 0) norder.push_back(aux[(size_t)u]);
    norder.push_back(u);
  }
  s.dg.resize((size_t)NN, -1.0);
  s.bidx.resize((size_t)NN, -1);
  s.oidx.resize((size_t)NN, -1);
  s.N = NN;
  s.rp.swap(nrp);
  s.col.swap(ncol);
  s.val.swap(nval);
  s.order.swap(norder);
  return true;
}

static int merge_passes() {   // read at every factor creation
  const char* e = getenv("LG_IC0_MERGE");
  return e ? std::max(0, std::min(4, atoi(e))) : 3;
}

// Lanes per row.  On wide levels (many more rows than warps) tasks are
// packed densely, one lane per row up to kLaneMax entries, to minimise the
// number of tasks a warp walks; on the others rows are spread over more lanes
// so each lane's share of the chain is short -- the more so on narrow levels
// (<= LG_FINE_ROWS = 4096 rows: idle warps abound and only the hop counts; measured
// on the merged schedules: C1 39.4 -> 34.5 us, C2 148 -> 132 us, C3 918 -> 849
// us, while C4's ~7.5 k-row levels lose 7 % with it and keep the middle
// classes).
static int lanes_for(int64_t len, int width) {
  if (width == 2) {          // wide level: dense packing
    if (len <= 8) return 1;
    if (len <= 16) return 2;
    if (len <= 32) return 4;
    if (len <= 64) return 8;
    return 32;
  }
  if (width == -1) {         // very narrow level: at most two entries per lane
    if (len <= 4) return 4;
    if (len <= 16) return 8;
    return 32;
  }
  if (width == 0) {          // narrow level: short chains per lane
    if (len <= 2) return 2;
    if (len <= 8) return 4;
    if (len <= 32) return 8;
    return 32;
  }
  if (len <= 4) return 2;
  if (len <= 16) return 4;
  if (len <= 64) return 8;
  return 32;  // <= kHubChunk: at most 8 entries per lane in every class
}

struct SweepHost {
  std::vector<int32_t> perm;
  std::vector<int64_t> prp;
  std::vector<int32_t> pcol;
  std::vector<double> pval, pdiag;
  std::vector<SweepTask> tasks;
  std::vector<int64_t> tbase;     // first entry of each task
  std::vector<uint16_t> lanetab;  // per task x lane: rel_start << 5 | count
  std::vector<SweepSeg> segs;
  std::vector<int32_t> hub_first, hub_nchunk;
  std::vector<int32_t> tlevel, lexpect;
  std::vector<int32_t> lhub0, hub_prow;   // resident sweep: hub rows per level
  int32_t nparts = 0;
  int32_t nbar = 0;
  int levels = 0;
};

// Level schedule of one sweep: rows grouped by DAG level and length class,
// permuted into that order, packed into warp tasks; every task carries a
// 32-lane table of (start, count) so staging a task is one level of
// independent loads.  Levels with at most `narrow_tasks` tasks run on the
// first cluster only.
static void build_sweep(const SweepSys& sys, int narrow_tasks, SweepHost& h) {
  const int64_t n = sys.N;   // unknowns of the scheduled system
  const std::vector<int64_t>& rp = sys.rp;
  const std::vector<int32_t>& col = sys.col;
  const std::vector<double>& val = sys.val;
  const std::vector<double>& diag = sys.dg;
  std::vector<int32_t> level;
  h.levels = dag_levels(sys, level);
  const int nl = h.levels;
  std::vector<int64_t> lcount((size_t)nl + 1, 0);
  for (int64_t i = 0; i < n; ++i) lcount[(size_t)level[(size_t)i] + 1]++;
  for (int l = 0; l < nl; ++l) lcount[(size_t)l + 1] += lcount[(size_t)l];
  static const int64_t wide_rows = [] {
    const char* e = getenv("LG_WIDE_ROWS");
    return e ? (int64_t)atoll(e) : (int64_t)16384;
  }();
  static const int64_t fine_rows = [] {
    const char* e = getenv("LG_FINE_ROWS");
    return e ? (int64_t)atoll(e) : (int64_t)4096;
  }();
  static const int64_t ultra_rows = [] {
    const char* e = getenv("LG_ULTRA_ROWS");
    return e ? (int64_t)atoll(e) : (int64_t)1024;
  }();
  static const int64_t task_target = [] {
    const char* e = getenv("LG_TASK_TARGET");
    return e ? (int64_t)atoll(e) : (int64_t)128;
  }();
  std::vector<signed char> lwide((size_t)nl);   // -1 very narrow, 0 narrow, 1 middle, 2 wide
  for (int l = 0; l < nl; ++l) {
    const int64_t rows = lcount[(size_t)l + 1] - lcount[(size_t)l];
    lwide[(size_t)l] = rows > wide_rows ? 2 : (rows > fine_rows ? 1 : (rows > ultra_rows ? 0 : -1));
  }
  auto cls = [&](int32_t r) {
    const int64_t len = rp[(size_t)r + 1] - rp[(size_t)r];
    return len > kHubChunk ? 64 : lanes_for(len, lwide[(size_t)level[(size_t)r]]);
  };
  h.perm.resize((size_t)n);
  {
    std::vector<int64_t> fill(lcount.begin(), lcount.end() - 1);
    for (int64_t k = 0; k < n; ++k) {
      const int64_t i = sys.order[(size_t)k];
      h.perm[(size_t)fill[(size_t)level[(size_t)i]]++] = (int32_t)i;
    }
  }
  for (int l = 0; l < nl; ++l)
    std::stable_sort(h.perm.begin() + lcount[(size_t)l], h.perm.begin() + lcount[(size_t)l + 1],
                     [&](int32_t a, int32_t b) { return cls(a) < cls(b); });
  h.prp.assign((size_t)n + 1, 0);
  h.pdiag.resize((size_t)n);
  for (int64_t p = 0; p < n; ++p) {
    const int32_t r = h.perm[(size_t)p];
    h.prp[(size_t)p + 1] = h.prp[(size_t)p] + (rp[(size_t)r + 1] - rp[(size_t)r]);
    h.pdiag[(size_t)p] = diag[(size_t)r];
  }
  h.pcol.resize(col.size());
  h.pval.resize(val.size());
  for (int64_t p = 0; p < n; ++p) {
    const int32_t r = h.perm[(size_t)p];
    std::copy(col.begin() + rp[(size_t)r], col.begin() + rp[(size_t)r + 1],
              h.pcol.begin() + h.prp[(size_t)p]);
    std::copy(val.begin() + rp[(size_t)r], val.begin() + rp[(size_t)r + 1],
              h.pval.begin() + h.prp[(size_t)p]);
  }
  auto push_task = [&](SweepTask tk, int64_t base, const uint16_t* lanes) {
    h.tasks.push_back(tk);
    h.tbase.push_back(base);
    h.lanetab.insert(h.lanetab.end(), lanes, lanes + 32);
  };
  for (int l = 0; l < nl; ++l) {
    const int32_t t0 = (int32_t)h.tasks.size();
    h.lhub0.push_back((int32_t)h.hub_first.size());
    int64_t t = lcount[(size_t)l];
    const int64_t te = lcount[(size_t)l + 1];
    while (t < te) {
      const int L = cls(h.perm[(size_t)t]);
      uint16_t lanes[32];
      if (L == 64) {  // hub row: chunk tasks of kHubChunk entries
        const int64_t len = h.prp[(size_t)t + 1] - h.prp[(size_t)t];
        const int32_t nch = (int32_t)((len + kHubChunk - 1) / kHubChunk);
        const int32_t hid = (int32_t)h.hub_first.size();
        h.hub_first.push_back(h.nparts);
        h.hub_nchunk.push_back(nch);
        h.hub_prow.push_back((int32_t)t);
        h.nparts += nch;
        for (int32_t c = 0; c < nch; ++c) {
          const int64_t lo = h.prp[(size_t)t] + (int64_t)c * kHubChunk;
          const int64_t hi = std::min<int64_t>(h.prp[(size_t)t + 1], lo + kHubChunk);
          for (int ln = 0; ln < 32; ++ln) {
            const int64_t cntl = hi - (lo + ln) > 0 ? (hi - (lo + ln) + 31) / 32 : 0;
            lanes[ln] = (uint16_t)((ln << 5) | (int)cntl);
          }
          push_task({(int32_t)t, 0, c, hid}, lo, lanes);
        }
        ++t;
        continue;
      }
      // rows per task: a full warp, or -- on a level with few rows -- as few as
      // leave the level ~task_target tasks (fewer inputs to wait for per task)
      const int64_t lrows = lcount[(size_t)l + 1] - lcount[(size_t)l];
      const int cap = task_target > 0 && lrows <= fine_rows
                          ? (int)std::max<int64_t>(1, std::min<int64_t>(32 / L, lrows / task_target))
                          : 32 / L;
      int cnt = 1;
      while (cnt < cap && t + cnt < te && cls(h.perm[(size_t)(t + cnt)]) == L) ++cnt;
      const int64_t base = h.prp[(size_t)t];
      for (int ln = 0; ln < 32; ++ln) {
        const int g = ln / L, li = ln % L;
        int cntl = 0, rel = 0;
        if (g < cnt) {
          const int64_t lo = h.prp[(size_t)(t + g)] + li, hi = h.prp[(size_t)(t + g) + 1];
          cntl = lo < hi ? (int)((hi - lo + L - 1) / L) : 0;
          rel = (int)(lo - base);
        }
        lanes[ln] = (uint16_t)((rel << 5) | cntl);
      }
      push_task({(int32_t)t, (L << 8) | cnt, 0, 0}, base, lanes);
      t += cnt;
    }
    const int32_t t1 = (int32_t)h.tasks.size();
    h.segs.push_back({t0, t1, (t1 - t0) <= narrow_tasks ? 1 : 0, 0, 0, 0});
    for (int32_t t = t0; t < t1; ++t) h.tlevel.push_back(l);
  }
  h.lhub0.push_back((int32_t)h.hub_first.size());
  // re-lay the entries task by task, every task starting on a multiple of 4
  // entries (16-byte aligned columns, 32-byte aligned values); lane tables
  // are relative to the task base
  {
    const size_t nt = h.tasks.size();
    std::vector<int32_t> qcol;
    std::vector<double> qval;
    qcol.reserve(h.pcol.size() + 4 * nt);
    qval.reserve(h.pval.size() + 4 * nt);
    for (size_t t = 0; t < nt; ++t) {
      const SweepTask& tk = h.tasks[t];
      const int64_t lo = h.tbase[t];
      const int64_t hi = tk.b != 0 ? h.prp[(size_t)tk.p + (size_t)(tk.b & 0xff)]
                                   : std::min<int64_t>(h.prp[(size_t)tk.p + 1], lo + kHubChunk);
      const int64_t nb = (int64_t)qcol.size();
      qcol.insert(qcol.end(), h.pcol.begin() + lo, h.pcol.begin() + hi);
      qval.insert(qval.end(), h.pval.begin() + lo, h.pval.begin() + hi);
      while (qcol.size() & 3) {
        qcol.push_back(0);
        qval.push_back(0.0);
      }
      h.tbase[t] = nb;
    }
    h.pcol.swap(qcol);
    h.pval.swap(qval);
  }
  h.lexpect.assign((size_t)nl * 32, 0);
  for (size_t t = 0; t < h.tlevel.size(); ++t) h.lexpect[(size_t)h.tlevel[t] * 32 + (t & 31)]++;
  for (size_t sg = h.segs.size(); sg-- > 0;) {
    const bool same = sg + 1 < h.segs.size() && h.segs[sg + 1].narrow == h.segs[sg].narrow;
    h.segs[sg].run_t1 = same ? h.segs[sg + 1].run_t1 : h.segs[sg].t1;
  }
  // barrier flags: 2 = cluster barrier (narrow -> narrow), 1 = grid barrier
  // (after a wide level, or a narrow run followed by a wide level); none
  // after the final segment
  h.nbar = 0;
  for (size_t sg = 0; sg + 1 < h.segs.size(); ++sg) {
    if (h.segs[sg].narrow && h.segs[sg + 1].narrow) {
      h.segs[sg].barrier = 2;
    } else {
      h.segs[sg].barrier = 1;
      ++h.nbar;
    }
  }
}

// ----------------------------------------------------------- device side --
// Source of entry `col` of a sweep: the solution vector, or -- a b entry of a
// level-merged row (col >= n) -- the right-hand side.
__device__ __forceinline__ const double* entry_src(const double* x, const double* b, int32_t n,
                                                   int32_t col) {
  return (col >= n ? b - n : x) + col;
}

struct SweepArgs {
  const int64_t* prp;
  const int32_t* pcol;
  const double* pval;
  const int32_t* perm;
  const double* pdiag;
  const SweepTask* tasks;
  const int64_t* tbase;
  const uint16_t* lanetab;
  const SweepSeg* segs;
  int32_t nsegs;
  int32_t nbar;
  int32_t csize;           // CTAs per cluster (1: no clusters)
  const int32_t* hub_first;
  const int32_t* hub_nchunk;
  unsigned* hub_ticket;
  double* hub_part;
  unsigned long long* bar;
  const double* b;
  double* x;
  const int32_t* bmap;   // unknown -> b index (-1: none)
  double* out2;          // the sweep's output vector (or NULL)
  const int32_t* omap;   // unknown -> index in out2 (-1: none)
  const int* skip;
  unsigned long long* trace;  // optional: globaltimer after every segment (CTA 0)
  int dbg;                    // timing experiments only (LG_SWEEP_DBG)
  int32_t n;
};

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

constexpr int kLaneMax = 8;   // entries per lane per task (any class)

// Everything a lane needs for one task that does not depend on the solve;
// loaded between barrier arrive and wait of the previous level.
struct Staged {
  int32_t col[kLaneMax];
  double val[kLaneMax];
  int32_t row;    // original row of this lane's group (pack) / permuted hub row
  int32_t ne;     // entries held by this lane
  int32_t info;   // task.b (0: hub chunk)
  int32_t c, d;   // hub chunk index / id
  double bv, dg;
};

// Staging is split in two phases so that neither blocks the warp: phase 1
// loads the task descriptor and this lane's (start, count) word; phase 2
// (at least one barrier later, when those have arrived) loads the lane's
// entries and its row's diagonal / right-hand side.
struct Stage1 {
  SweepTask tk;
  int64_t base;
  uint32_t lt;
};

__device__ __forceinline__ void stage1(const SweepArgs& a, int64_t t, int lane, Stage1& s1) {
  s1.tk = a.tasks[t];
  s1.base = a.tbase[t];
  s1.lt = a.lanetab[t * 32 + lane];
}

__device__ __forceinline__ void stage2(const SweepArgs& a, const Stage1& s1, int lane,
                                       Staged& st) {
  const SweepTask tk = s1.tk;
  st.info = tk.b;
  st.ne = s1.lt & 31;
  const int64_t lo = s1.base + (s1.lt >> 5);
  int step;
  if (tk.b != 0) {
    const int L = tk.b >> 8, cnt = tk.b & 0xff;
    const int g = lane / L;
    step = L;
    if (g < cnt) {
      const int64_t p = tk.p + g;
      st.row = a.perm[p];
      st.dg = a.pdiag[p];
      const int32_t bi = a.bmap[st.row];
      st.bv = bi >= 0 ? a.b[bi] : 0.0;   // auxiliary unknowns have no right-hand side
    }
  } else {
    st.row = tk.p;
    st.c = tk.c;
    st.d = tk.d;
    step = 32;
  }
#pragma unroll
  for (int e = 0; e < kLaneMax; ++e) {
    if (e < st.ne) {
      const int64_t k = lo + (int64_t)e * step;
      st.col[e] = a.pcol[k];
      st.val[e] = a.pval[k];
    }
  }
}

__device__ __forceinline__ void stage(const SweepArgs& a, int64_t t, int lane, Staged& st) {
  Stage1 s1;
  stage1(a, t, lane, s1);
  stage2(a, s1, lane, st);
}

__device__ __forceinline__ void finish(const SweepArgs& a, const Staged& st, int lane) {
  double s = 0.0;
  if (a.dbg & 4) {
#pragma unroll
    for (int e = 0; e < kLaneMax; ++e)
      if (e < st.ne) s += st.val[e];
  } else {
#pragma unroll
    for (int e = 0; e < kLaneMax; ++e)
      if (e < st.ne) s += st.val[e] * __ldcg(entry_src(a.x, a.b, a.n, st.col[e]));
  }
  if (st.info != 0) {
    const int L = st.info >> 8, cnt = st.info & 0xff;
    for (int o = L >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((lane / L) < cnt && (lane % L) == 0 && !(a.dbg & 8)) {
      const double v = (st.bv - s) / st.dg;
      a.x[st.row] = v;
      if (a.out2) {
        const int32_t oi = a.omap[st.row];
        if (oi >= 0) a.out2[oi] = v;
      }
    }
    return;
  }
  // chunk of a hub row: publish the partial; the last chunk sums all of
  // them lane-strided + butterfly (fixed order whoever arrives last)
  s = warp_sum(s);
  const int32_t first = a.hub_first[st.d], nch = a.hub_nchunk[st.d];
  unsigned arrived = 0;
  if (lane == 0) {
    a.hub_part[first + st.c] = s;
    __threadfence();
    arrived = atomicAdd(a.hub_ticket + st.d, 1u);
  }
  arrived = __shfl_sync(0xffffffffu, arrived, 0);
  if (arrived == (unsigned)nch - 1u) {
    __threadfence();
    double t = 0.0;
    for (int32_t c = lane; c < nch; c += 32) t += __ldcg(a.hub_part + first + c);
    t = warp_sum(t);
    if (lane == 0) {
      a.hub_ticket[st.d] = 0u;
      const int32_t row = a.perm[st.row];
      const int32_t bi = a.bmap[row];
      const double v = ((bi >= 0 ? a.b[bi] : 0.0) - t) / a.pdiag[st.row];
      a.x[row] = v;
      if (a.out2) {
        const int32_t oi = a.omap[row];
        if (oi >= 0) a.out2[oi] = v;
      }
    }
  }
}

__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __launch_bounds__(kSweepThreads, 1) sweep_kernel(SweepArgs a) {
  if (a.skip && *a.skip) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t G = gridDim.x;
  const int64_t gw = (int64_t)blockIdx.x * kSweepWarps + warp;
  const int64_t W = G * kSweepWarps;
  const int csize = a.csize;
  const bool first_cluster = blockIdx.x < (unsigned)csize;
  const int64_t cw = (int64_t)blockIdx.x * kSweepWarps + warp;   // valid in cluster 0
  const int64_t CW = (int64_t)csize * kSweepWarps;
  // every launch adds exactly nbar * G arrivals; barrier 0 cannot complete
  // before this CTA arrives, so rounding down recovers this launch's base
  __shared__ unsigned long long base_sm;
  __shared__ SweepSeg seg_sm[kSegSmem];
  if (threadIdx.x == 0) {
    const unsigned long long per = (unsigned long long)a.nbar * (unsigned long long)G;
    const unsigned long long v = ld_relaxed_u64(a.bar);
    base_sm = per ? (v / per) * per : 0ull;
  }
  const bool segs_in_smem = a.nsegs <= kSegSmem;
  if (segs_in_smem)
    for (int i = threadIdx.x; i < a.nsegs; i += blockDim.x) seg_sm[i] = a.segs[i];
  __syncthreads();
  const SweepSeg* segs = segs_in_smem ? seg_sm : a.segs;
  const unsigned long long base = base_sm;
  int nb = 0;
  Staged st;
  // Task t of a segment belongs to the warp with index t mod stride (grid
  // warps for wide segments, first-cluster warps for narrow ones).  Tasks
  // are numbered consecutively across levels, so consecutive small levels
  // land on different warps and a warp can stage its next task many levels
  // before that level opens: after a barrier only the x gathers remain.
  // my_t: my next task in the current run of same-mode segments (tasks
  // t == id mod stride); only a mode switch needs a modulo (32-bit).
  const int icw = (int)cw, iCW = (int)CW, igw = (int)gw, iW = (int)W;
  auto mine_from = [&](int t, bool narrow) -> int {
    const int id = narrow ? icw : igw, st_ = narrow ? iCW : iW;
    int r = (id - t) % st_;
    if (r < 0) r += st_;
    return t + r;
  };
  // staging state of my next task: 0 none, 1 phase 1 issued, 2 staged
  int sstate = 0;
  int sttask = -1;
  Stage1 s1;
  int my_t = -1;
  if (a.nsegs > 0) {
    const SweepSeg s0 = segs[0];
    if (!s0.narrow || first_cluster) {
      my_t = mine_from(s0.t0, s0.narrow);
      if (my_t < s0.run_t1) {
        stage(a, my_t, lane, st);
        sttask = my_t;
        sstate = 2;
      }
    } else {
      my_t = 0x7fffffff;
    }
  }
  for (int s = 0; s < a.nsegs; ++s) {
    const SweepSeg sg = segs[s];
    const bool part = !sg.narrow || first_cluster;
    if (part) {
      const int stride = sg.narrow ? iCW : iW;
      if (my_t < sg.t1) {
        // make sure my first task of this segment is fully staged
        if (sttask != my_t || sstate != 2) {
          if (sttask == my_t && sstate == 1) {
            if (!(a.dbg & 2)) stage2(a, s1, lane, st);
          } else if (!(a.dbg & 2)) {
            stage(a, my_t, lane, st);
          }
          if (a.trace && lane == 0) atomicAdd(a.trace + a.nsegs, 1ull);
        }
        // three-stage software pipeline over my tasks of this level:
        // descriptor loads two tasks ahead, entry loads one task ahead,
        // finish the current one -- no dependent stall on the way
        Stage1 s1n;
        if (my_t + stride < sg.t1) stage1(a, my_t + stride, lane, s1n);
        for (; my_t < sg.t1; my_t += stride) {
          const int t1n = my_t + stride, t2n = my_t + 2 * stride;
          Staged stn;
          Stage1 s1nn;
          if (t2n < sg.t1) stage1(a, t2n, lane, s1nn);
          if (t1n < sg.t1) stage2(a, s1n, lane, stn);
          if (!(a.dbg & 1)) finish(a, st, lane);
          st = stn;
          s1n = s1nn;
        }
        sstate = 0;
        sttask = -1;
      }
    }
    // entering a new run (mode change): my first task there
    if (s + 1 < a.nsegs && sg.run_t1 == sg.t1) {
      const SweepSeg sn = segs[s + 1];
      sstate = 0;
      sttask = -1;
      my_t = (!sn.narrow || first_cluster) ? mine_from(sn.t0, sn.narrow) : 0x7fffffff;
    }
    const int run_end = (s + 1 < a.nsegs) ? segs[s + 1].run_t1 : 0;
    // advance the staging pipeline of my next task by one phase; neither
    // phase stalls the warp (phase 2 uses data loaded a barrier earlier)
    auto advance = [&]() {
      if (my_t >= run_end || (a.dbg & 2)) return;
      if (sstate == 0) {
        stage1(a, my_t, lane, s1);
        sttask = my_t;
        sstate = 1;
      } else if (sstate == 1 && sttask == my_t) {
        stage2(a, s1, lane, st);
        sstate = 2;
      }
    };
    if (sg.barrier == 1) {
      // split-phase grid barrier: arrive, advance staging, wait
      ++nb;
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(a.bar, 1ull);
      }
      advance();
      if (threadIdx.x == 0) {
        const unsigned long long target = base + (unsigned long long)nb * (unsigned long long)G;
        while (ld_relaxed_u64(a.bar) < target) {
        }
        __threadfence();
      }
      __syncthreads();
    } else if (sg.barrier == 2) {
      if (first_cluster) {
        if (csize > 1) cluster_arrive();
        advance();
        if (csize > 1) cluster_wait();
        else __syncthreads();
      }
    } else {
      advance();
    }
    if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.trace[s] = t;
    }
  }
}

// ---- dataflow sweep (default) ------------------------------------------------
// The solution vector is its own dependency flag: before a sweep x is filled
// with an all-ones NaN sentinel, every row is stored once with a relaxed
// 8-byte store (never the sentinel: a computed all-ones NaN is canonicalised)
// and a consumer re-polls exactly the entries it still sees as the sentinel.
// A dependency hop then costs one L2 store + one L2 load (~0.33 us measured,
// scripts/micro/chain.cu) instead of a fence + flag + acquire (~0.9 us), and
// no warp ever waits for a whole level -- only for the rows it reads.
//
// Warp w (of W workers) walks tasks t = w, w+W, ... in level order, staging
// task t+W while it completes task t.  Everything a task needs is at most
// three dependent loads away: the task descriptor / lane table, then the
// lane's columns + values + the row record {diag, x row, b index}, then the
// x gathers and b.  To keep polling traffic off L2, a task of level L only
// starts once levels <= L - gate are fully counted: one poller warp per CTA
// watches relaxed per-(level, shard) completion counters and publishes the
// highest complete level in shared memory (the counts only throttle;
// correctness rests on the sentinels).  Deadlock freedom: every task depends
// only on tasks of lower levels, which precede it in their own warps' lists,
// and the cooperative launch keeps all warps resident.
constexpr unsigned long long kSentinel = ~0ull;
// CTA size of the dataflow sweep, one CTA per SM: 1 poller + 11 worker warps
// (139 registers), or + 15 (128 registers) for schedules with many tasks per
// level, where resident warps rather than the hop bound the sweep (level-
// merged C4: 577 -> 551 us; C1-C3 lose 2-4 % with it)
constexpr int kFlowThreads = 384;
constexpr int kFlowThreadsWide = 512;
constexpr int kFlowThreadsSm = 768;   // entries staged through shared memory: 23 worker warps
constexpr int kFlowWideTasks = 512;   // mean tasks per level from which the wide CTA is used

struct FlowArgs {
  const int32_t* pcol;
  const double* pval;
  const RowInfo* rinfo;
  const int32_t* oidx;   // permuted row -> out2 index (NULL: no second output)
  const SweepTask* tasks;
  const int64_t* tbase;
  const uint16_t* lanetab;
  const int32_t* tlevel;
  const int32_t* lexpect;
  unsigned* lcount;
  const int32_t* hub_first;
  const int32_t* hub_nchunk;
  double* hub_part;
  const double* b;
  double* x;
  double* out2;
  const int* skip;
  unsigned long long* ttrace;   // debug: per task {start, inputs ready, done}
  double* next_x;               // x of the other sweep: row re-armed after its b is read
  unsigned* next_cnt;           // the other sweep's counters / hub slots, re-armed here
  double* next_part;
  int32_t next_ncnt, next_npart;
  int32_t ntasks;
  int32_t levels;
  int32_t gate;
  uint32_t backoff;   // max poll back-off (ns)
  int32_t n;          // unknowns of this sweep (entries with col >= n read b)
  int32_t nreal;      // rows of the factor (unknowns beyond are auxiliary)
  int32_t next_n;     // unknowns of the other sweep (length of next_x)
  // next_x is this sweep's own right-hand side (the backward sweep re-arming
  // the forward scratch): level-merged rows read b at other rows too, so the
  // rows are re-armed once the whole sweep is complete, not one by one
  int32_t defer_rearm;
};

__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double ld_relaxed_f64(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_f64(double* p, double v) {
  if (__double_as_longlong(v) == (long long)kSentinel) v = __longlong_as_double(0x7ff8000000000000ll);
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void red_relaxed_add(unsigned* p, unsigned v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ bool is_sentinel(double v) {
  return __double_as_longlong(v) == (long long)kSentinel;
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void flow_init_kernel(double* x, int64_t n, unsigned* cnt, int ncnt, double* part,
                                 int npart, const int* skip) {
  if (skip && *skip) return;
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = i0; i < ncnt; i += st) cnt[i] = 0u;
  for (int64_t i = i0; i < npart; i += st) part[i] = __longlong_as_double((long long)kSentinel);
  for (int64_t i = i0; i < n; i += st) x[i] = __longlong_as_double((long long)kSentinel);
}

// Task staging in two non-blocking phases (phase 2 one task later).
struct FStage1 {
  SweepTask tk;
  int64_t base;
  uint32_t lt;
  int32_t lev;
};
struct FStaged {
  int32_t info;   // task.b (0: hub chunk)
  int32_t p;      // pack: permuted row of the lane's group (-1: idle) | chunk: permuted hub row
  int32_t c, hid; // chunk: chunk index, hub id
  int32_t ne, sh, lev;
  int32_t oi;     // output index of the owner lane's row (-1: none), staged with the row record
  int32_t col[kLaneMax];
  double val[kLaneMax];
  RowInfo ri;
};

template <class A>
__device__ __forceinline__ void fstage1(const A& a, int64_t t, int lane, FStage1& s) {
  s.tk = a.tasks[t];
  s.base = a.tbase[t];
  s.lt = a.lanetab[t * 32 + lane];
  s.lev = a.tlevel[t];
}

// Entries staged through shared memory (SM = true, opt-in LG_FLOW_WIDE=2):
// the lane's columns and values go from global into its own slots with
// cp.async -- no registers and no scoreboard wait -- so the kernel fits 23
// worker warps per SM instead of 15 (80 registers); slot of entry e of stage
// g: [(g * kLaneMax + e) * 32 + lane].  Same bits; not faster (launch_flow).
__device__ __forceinline__ void cp_async4(void* dst_smem, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst_smem)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst_smem, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst_smem)),
               "l"(src)
               : "memory");
}

__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <bool SM = false, class A>
__device__ __forceinline__ void fstage2(const A& a, const FStage1& s, int lane, FStaged& st,
                                        int32_t* sc = nullptr, double* sv = nullptr) {
  const SweepTask tk = s.tk;
  st.info = tk.b;
  st.lev = s.lev;
  st.ne = s.lt & 31;
  const int64_t lo = s.base + (s.lt >> 5);
  if (tk.b != 0) {
    const int L = tk.b >> 8, cnt = tk.b & 0xff;
    st.sh = __ffs(L) - 1;
    st.p = -1;
    st.oi = -1;
    if ((lane >> st.sh) < cnt) {
      st.p = tk.p + (lane >> st.sh);
      st.ri = a.rinfo[st.p];
      if (a.out2) st.oi = a.oidx[st.p];
    }
  } else {
    st.p = tk.p;
    st.c = tk.c;
    st.hid = tk.d;
    st.sh = 5;
    st.oi = -1;
    if (tk.c == 0) {
      st.ri = a.rinfo[tk.p];
      if (a.out2) st.oi = a.oidx[tk.p];
    }
  }
#pragma unroll
  for (int e = 0; e < kLaneMax; ++e) {
    if (e < st.ne) {
      const int64_t k = lo + ((int64_t)e << st.sh);
      if constexpr (SM) {
        cp_async4(sc + e * 32, a.pcol + k);
        cp_async8(sv + e * 32, a.pval + k);
      } else {
        st.col[e] = a.pcol[k];
        st.val[e] = a.pval[k];
      }
    }
  }
}

__device__ __forceinline__ void publish(const FlowArgs& a, int32_t oi, const RowInfo& ri, double v) {
  st_relaxed_f64(a.x + ri.xrow, v);
  if (oi >= 0) a.out2[oi] = v;
  // this row's b has been consumed: re-arm the row in the other sweep's x
  // (unless that buffer is this sweep's b, which merged rows still read)
  // (the other sweep's auxiliary unknowns are re-armed in this kernel's prologue)
  if (!a.defer_rearm && ri.xrow < a.nreal)
    a.next_x[ri.xrow] = __longlong_as_double((long long)kSentinel);
}

template <bool SM = false>
__device__ __forceinline__ void flow_complete(const FlowArgs& a, const FStaged& st, int lane,
                                              unsigned long long* tr, const int32_t* sc = nullptr,
                                              const double* sv = nullptr) {
  // entry e's column / value: the staged registers, or the lane's shared-memory slots
  auto COL = [&](int e) -> int32_t {
    if constexpr (SM) return sc[e * 32];
    else return st.col[e];
  };
  auto VAL = [&](int e) -> double {
    if constexpr (SM) return sv[e * 32];
    else return st.val[e];
  };
  const bool owner = st.info != 0 ? (st.p >= 0 && (lane & ((1 << st.sh) - 1)) == 0)
                                  : (st.c == 0 && lane == 0);
  double bv = 0.0;
  if (owner && st.ri.bidx >= 0) bv = a.b[st.ri.bidx];
  double xv[kLaneMax];
  unsigned miss = 0;
#pragma unroll
  for (int e = 0; e < kLaneMax; ++e) {
    if (e < st.ne) {
      xv[e] = ld_relaxed_f64(entry_src(a.x, a.b, a.n, COL(e)));
      if (COL(e) < a.n && is_sentinel(xv[e])) miss |= 1u << e;   // b entries never wait
    }
  }
  unsigned spins = 0, nap = 16;
#if !defined(LG_FLOW_SPINALL) && !defined(LG_FLOW_POLL2)
  // probe one missing entry per lane per round trip (less polling traffic on
  // L2: C4 apply 757 -> 733 us, C3 1401 -> 1349 us); once it lands, sweep
  // every still-missing entry of the lane again
  bool sweep = false;
  while (__any_sync(0xffffffffu, miss != 0)) {
    if (++spins > (1u << 24)) __trap();
    const int fe = miss ? __ffs(miss) - 1 : -1;
    const unsigned probe = sweep ? miss : (miss & (0u - miss));
    bool got = false;
#pragma unroll
    for (int e = 0; e < kLaneMax; ++e) {
      if (probe & (1u << e)) {
        xv[e] = ld_relaxed_f64(a.x + COL(e));
        if (!is_sentinel(xv[e])) {
          miss &= ~(1u << e);
          if (e == fe) got = true;
        }
      }
    }
    sweep = got;
  }
#elif defined(LG_FLOW_POLL2)
  // two generations of polls in flight, half a round trip apart: a value
  // that lands is seen about a quarter round trip sooner on average
  if (__any_sync(0xffffffffu, miss != 0)) {
    double xb[kLaneMax];
    __nanosleep(LG_FLOW_POLL2);
#pragma unroll
    for (int e = 0; e < kLaneMax; ++e)
      if (miss & (1u << e)) xb[e] = ld_relaxed_f64(a.x + COL(e));
    while (true) {
#pragma unroll
      for (int e = 0; e < kLaneMax; ++e)
        if (miss & (1u << e)) {
          if (!is_sentinel(xv[e])) miss &= ~(1u << e);
          else xv[e] = ld_relaxed_f64(a.x + COL(e));
        }
      if (!__any_sync(0xffffffffu, miss != 0)) break;
#pragma unroll
      for (int e = 0; e < kLaneMax; ++e)
        if (miss & (1u << e)) {
          if (!is_sentinel(xb[e])) {
            xv[e] = xb[e];
            miss &= ~(1u << e);
          } else {
            xb[e] = ld_relaxed_f64(a.x + COL(e));
          }
        }
      if (!__any_sync(0xffffffffu, miss != 0)) break;
      if (++spins > (1u << 24)) __trap();
    }
  }
#else
  while (__any_sync(0xffffffffu, miss != 0)) {
    if (nap > 16) __nanosleep(nap);   // default: spin (measured 1-2 % faster than a 16 ns nap)
    nap = min(nap * 2, a.backoff);
    if (++spins > (1u << 24)) __trap();   // a row never produced: abort, do not hang
#pragma unroll
    for (int e = 0; e < kLaneMax; ++e) {
      if (miss & (1u << e)) {
        xv[e] = ld_relaxed_f64(a.x + COL(e));
        if (!is_sentinel(xv[e])) miss &= ~(1u << e);
      }
    }
  }
#endif
  if (tr && lane == 0) tr[1] = gtimer();
  double s = 0.0;
#pragma unroll
  for (int e = 0; e < kLaneMax; ++e)
    if (e < st.ne) s += VAL(e) * xv[e];
  if (st.info != 0) {
    for (int o = (1 << st.sh) >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
#ifdef LG_FLOW_RCP
    if (owner) publish(a, st.oi, st.ri, (bv - s) * (1.0 / st.ri.dg));
#else
    if (owner) publish(a, st.oi, st.ri, (bv - s) / st.ri.dg);
#endif
    return;
  }
  // chunk of a hub row: every chunk but the first publishes its partial
  // with a relaxed store (sentinel-initialised slots); chunk 0 sums them
  // lane-strided + butterfly, a fixed order whoever finishes last
  s = warp_sum(s);
  const int32_t first = a.hub_first[st.hid], nch = a.hub_nchunk[st.hid];
  if (st.c != 0) {
    if (lane == 0) st_relaxed_f64(a.hub_part + first + st.c, s);
    return;
  }
  double t = 0.0;
  for (int32_t c = lane; c < nch; c += 32) {
    double v = s;
    if (c != 0) {
      v = ld_relaxed_f64(a.hub_part + first + c);
      for (unsigned k = 0; is_sentinel(v); ++k) {
        if (k > (1u << 24)) __trap();
        __nanosleep(20);
        v = ld_relaxed_f64(a.hub_part + first + c);
      }
    }
    t += v;
  }
  t = warp_sum(t);
  if (lane == 0) publish(a, st.oi, st.ri, (bv - t) / st.ri.dg);
}

template <int kFlowThreads, bool SM = false>
__global__ void __launch_bounds__(kFlowThreads, 1) sweep_flow_kernel(FlowArgs a) {
  if (a.skip && *a.skip) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int kWorkers = kFlowThreads / 32 - 1;
  // SM: per worker warp two stages of lane-private entry slots (columns, values)
  extern __shared__ __align__(16) unsigned char flow_smem[];
  int32_t* sc_base = nullptr;
  double* sv_base = nullptr;
  if constexpr (SM) {
    sv_base = reinterpret_cast<double*>(flow_smem) + (size_t)(warp - 1) * 2 * kLaneMax * 32 + lane;
    sc_base = reinterpret_cast<int32_t*>(flow_smem + (size_t)kWorkers * 2 * kLaneMax * 32 * 8) +
              (size_t)(warp - 1) * 2 * kLaneMax * 32 + lane;
  }
  __shared__ volatile int s_done;
  __shared__ volatile int s_active;
  if (threadIdx.x == 0) {
    s_done = -1;
    s_active = kWorkers;
  }
  __syncthreads();
  const int gate = a.gate;
  if (warp == 0) {   // level watcher
    // (a deferred re-arm waits for the whole sweep: watch through the last level)
    const int lend = a.defer_rearm ? a.levels : a.levels - gate;
    for (int L = 0; L < lend; ++L) {
      const int idx = L * 32 + lane;
      const unsigned want = (unsigned)a.lexpect[idx];
      while (true) {
        const unsigned v = ld_relaxed_u32(a.lcount + idx);
        if (__all_sync(0xffffffffu, v >= want)) break;
        if (s_active == 0 && !a.defer_rearm) return;
        __nanosleep(32);
      }
      s_done = L;
    }
    return;
  }
  const int64_t W = (int64_t)gridDim.x * kWorkers;
  const int64_t nt = a.ntasks;
  {
    const int64_t i0 = (int64_t)blockIdx.x * (kFlowThreads - 32) + threadIdx.x - 32;
    const int64_t stride = (int64_t)gridDim.x * (kFlowThreads - 32);
    for (int64_t i = i0; i < a.next_ncnt; i += stride) a.next_cnt[i] = 0u;
    for (int64_t i = i0; i < a.next_npart; i += stride)
      a.next_part[i] = __longlong_as_double((long long)kSentinel);
    if (!a.defer_rearm)
      for (int64_t i = a.nreal + i0; i < a.next_n; i += stride)
        a.next_x[i] = __longlong_as_double((long long)kSentinel);
  }
  int64_t t = (int64_t)blockIdx.x * kWorkers + warp - 1;
  if (t < nt) {
    FStaged st, stn;
    FStage1 s1n;
    int g = 0;   // SM: stage holding the current task's entries
    {
      FStage1 s1;
      fstage1(a, t, lane, s1);
      fstage2<SM>(a, s1, lane, st, sc_base, sv_base);
      if constexpr (SM) cp_async_commit();
    }
    if (t + W < nt) fstage1(a, t + W, lane, s1n);
    for (; t < nt; t += W) {
      FStage1 s1nn;
      if (t + 2 * W < nt) fstage1(a, t + 2 * W, lane, s1nn);
      if (t + W < nt)
        fstage2<SM>(a, s1n, lane, stn, sc_base + (g ^ 1) * kLaneMax * 32,
                    sv_base + (g ^ 1) * kLaneMax * 32);
      if constexpr (SM) cp_async_commit();   // one group per step, empty or not
      for (unsigned spins = 0; s_done < st.lev - gate; ++spins) {
        __nanosleep(32);
        if (spins > (1u << 24)) __trap();
      }
      unsigned long long* tr = a.ttrace ? a.ttrace + 3 * t : nullptr;
      if (tr && lane == 0) tr[0] = gtimer();
      if constexpr (SM) cp_async_wait<1>();   // the current task's entries have landed
      flow_complete<SM>(a, st, lane, tr, sc_base + g * kLaneMax * 32, sv_base + g * kLaneMax * 32);
      if (tr && lane == 0) tr[2] = gtimer();
      if (lane == 0) red_relaxed_add(a.lcount + st.lev * 32 + (t & 31), 1u);
      st = stn;
      s1n = s1nn;
      g ^= 1;
    }
  }
  __syncwarp();
  if (a.defer_rearm) {
    // every task of the sweep is complete (its b is no longer read): re-arm
    // this CTA's share of the other sweep's x
    for (unsigned spins = 0; s_done < a.levels - 1; ++spins) {
      __nanosleep(64);
      if (spins > (1u << 26)) __trap();
    }
    const int64_t i0 = (int64_t)blockIdx.x * (kFlowThreads - 32) + threadIdx.x - 32;
    const int64_t stride = (int64_t)gridDim.x * (kFlowThreads - 32);
    for (int64_t i = i0; i < a.next_n; i += stride)
      a.next_x[i] = __longlong_as_double((long long)kSentinel);
  }
  if (lane == 0) atomicSub((int*)&s_active, 1);
}

// ---- resident sweep (narrow DAGs: one CTA runs the whole apply) -------------
// On a factor whose levels are narrow (C1: ~90 rows a level, C2: ~200, C3:
// ~300) the dataflow sweep is bound by its dependency hop through L2 (store +
// poll: 1.0-1.4 us a level).  One CTA alone has no such hop: its warps see each
// other's stores after a __syncthreads (~50 ns) and both sweeps run in ONE
// launch.  Measured (scripts/micro/sweepchain.cu): 0.22-0.29 us per level for
// one CTA against 0.83 us for a level across a cluster with x in L2.  The
// tasks, lane tables and summation order are the dataflow sweep's, so the
// result is bitwise the same: warp w takes tasks w, w + W, ... (consecutive
// tasks of a level land on distinct warps) and passes one barrier per level; a
// level holding hub rows adds a second barrier -- every chunk publishes its
// partial, then a warp per hub row sums them in chunk order.
//
// With only W warps on the SM nothing may wait on a dependent load chain, so a
// warp's future tasks are staged into shared memory with cp.async, two levels
// deep: the 96-byte descriptor (task, entry base and count, level, lane table)
// of the task 2 D ahead, and -- from the descriptor that has landed by then --
// the entries (columns, values) and row records of the task D ahead.  One
// commit group per step; cp.async.wait_group<D - 1> covers both.  At its turn
// a task reads everything but x and b from shared memory.  One SM's
// throughput bounds the sweep; measured, it only ties the dataflow sweeps on
// the smallest factor (C1) and loses elsewhere, so it is opt-in
// (pick_cta_mode below).
struct CtaDesc {        // 96 bytes, 16-byte aligned
  SweepTask tk;
  int64_t base;         // first entry (multiple of 4)
  int32_t lev;
  int32_t nent4;        // entries of the task, rounded up to a multiple of 4
  uint16_t lanetab[32];
};
static_assert(sizeof(CtaDesc) == 96, "CtaDesc layout");

constexpr int kCtaEntMax = 256;   // entries per task (pack: 32 lanes x 8; chunk: kHubChunk)

struct CtaDir {
  const int32_t* pcol;
  const double* pval;
  const RowInfo* rinfo;
  const int32_t* oidx;
  const CtaDesc* desc;
  const int32_t* lhub0;
  const int32_t* hub_prow;
  const int32_t* hub_first;
  const int32_t* hub_nchunk;
  double* hub_part;
  const double* b;
  double* x;
  double* out2;
  unsigned long long* ttrace;   // debug: per task {start, inputs ready, done}
  int32_t ntasks;
  int32_t levels;
  int32_t n;
};

struct CtaArgs {
  CtaDir dir[2];
  const int* skip;
};

template <int B>
struct CtaSlots {       // one warp's staging area
  CtaDesc desc[2 * (B - 1) + 1];
  int32_t col[B][kCtaEntMax];
  double val[B][kCtaEntMax];
  RowInfo ri[B][32];
};

__device__ __forceinline__ void cp_async16(void* dst_smem, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst_smem)),
               "l"(src)
               : "memory");
}

__device__ __forceinline__ unsigned long long gtimer_after(double dep) {
  unsigned long long t;
  asm volatile("{ .reg .f64 d; mov.f64 d, %1; mov.u64 %0, %%globaltimer; }" : "=l"(t) : "d"(dep));
  return t;
}

__device__ __forceinline__ void cta_publish(const CtaDir& a, int32_t p, const RowInfo& ri,
                                            double v) {
  if (__double_as_longlong(v) == (long long)kSentinel) v = __longlong_as_double(0x7ff8000000000000ll);
  a.x[ri.xrow] = v;
  if (a.out2) {
    const int32_t oi = a.oidx[p];
    if (oi >= 0) a.out2[oi] = v;
  }
}

// One staged task: same entry order per lane, same butterfly, same division as
// flow_complete.
__device__ __forceinline__ void cta_complete(const CtaDir& a, const CtaDesc& d, const int32_t* col,
                                             const double* val, const RowInfo* ris, int lane,
                                             unsigned long long* tr) {
  const uint32_t lt = d.lanetab[lane];
  const int ne = lt & 31, rel = lt >> 5;
  const int32_t info = d.tk.b;
  int sh = 5;
  bool owner = false;
  RowInfo ri;
  double bv = 0.0;
  if (info != 0) {
    const int L = info >> 8, cnt = info & 0xff;
    sh = __ffs(L) - 1;
    owner = (lane >> sh) < cnt && (lane & (L - 1)) == 0;
    if (owner) {
      ri = ris[lane >> sh];
      if (ri.bidx >= 0) bv = a.b[ri.bidx];
    }
  }
  double xv[kLaneMax], vv[kLaneMax];
#pragma unroll
  for (int e = 0; e < kLaneMax; ++e) {
    if (e < ne) {
      const int k = rel + (e << sh);
      xv[e] = *entry_src(a.x, a.b, a.n, col[k]);
      vv[e] = val[k];
    }
  }
  double s = 0.0;
#pragma unroll
  for (int e = 0; e < kLaneMax; ++e)
    if (e < ne) s += vv[e] * xv[e];
  if (tr && lane == 0) tr[1] = gtimer_after(s);
  if (info != 0) {
    for (int o = (1 << sh) >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (owner) cta_publish(a, d.tk.p + (lane >> sh), ri, (bv - s) / ri.dg);
    return;
  }
  // chunk of a hub row: every chunk (the first too) publishes its partial;
  // the row is finished behind the level's barrier (cta_level_end)
  s = warp_sum(s);
  if (lane == 0) a.hub_part[a.hub_first[d.tk.d] + d.tk.c] = s;
}

// Split CTA barrier on an mbarrier (one arrival per warp): a warp arrives as
// soon as its last task of the level is stored and only waits when it next
// needs the level -- the staging work in between is off the critical path.
__device__ __forceinline__ void lvl_arrive(uint64_t* bar, int lane) {
  __syncwarp();   // the warp's stores are ordered before the elected lane's release
  if (lane == 0)
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(bar))
                 : "memory");
}
__device__ __forceinline__ void lvl_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n LVLW_%=:\n"
      " mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra LVLW_%=;\n}\n" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
      "r"(parity)
      : "memory");
}

constexpr int kCtaHubLevels = 4096;   // level hub flags kept in shared memory

struct CtaShared {
  uint64_t bar;
  unsigned char hub[kCtaHubLevels];
};

// per-warp barrier bookkeeping: the phase the warp will wait on next, and
// whether it has already arrived there
struct CtaSync {
  unsigned phase;
  bool arrived;
};

// Pass level l: (arrive,) wait; hub rows of the level are then summed in chunk
// order (lane-strided, butterfly: the dataflow sweep's order) behind a second
// phase.  Every warp of the CTA passes every level once.
__device__ __forceinline__ void cta_level_end(const CtaDir& a, CtaShared& sh, CtaSync& sy, int l,
                                              int warp, int lane, int W) {
  // (the flag is read before the wait: once the sweep's last level is passed
  // the next sweep's flags may overwrite it)
  const bool hub = l < kCtaHubLevels ? sh.hub[l] != 0 : a.lhub0[l + 1] > a.lhub0[l];
  if (!sy.arrived) lvl_arrive(&sh.bar, lane);
  lvl_wait(&sh.bar, sy.phase & 1u);
  ++sy.phase;
  sy.arrived = false;
  if (hub) {
    const int32_t h0 = a.lhub0[l], h1 = a.lhub0[l + 1];
    for (int32_t hid = h0 + warp; hid < h1; hid += W) {
      const int32_t p = a.hub_prow[hid];
      const RowInfo ri = a.rinfo[p];
      const int32_t first = a.hub_first[hid], nch = a.hub_nchunk[hid];
      double t = 0.0;
      for (int32_t c = lane; c < nch; c += 32) t += a.hub_part[first + c];
      t = warp_sum(t);
      if (lane == 0) cta_publish(a, p, ri, ((ri.bidx >= 0 ? a.b[ri.bidx] : 0.0) - t) / ri.dg);
    }
    lvl_arrive(&sh.bar, lane);
    lvl_wait(&sh.bar, sy.phase & 1u);
    ++sy.phase;
  }
}

template <int B>
__device__ __forceinline__ void cta_run_dir(const CtaDir& a, CtaSlots<B>& sm, CtaShared& sh,
                                            CtaSync& sy, int warp, int lane, int W) {
  constexpr int D = B - 1;          // entries are staged D tasks ahead
  constexpr int ND = 2 * D + 1;     // descriptors 2 D ahead
  const int nt = a.ntasks;
  // hub flags of this direction's levels (the previous direction is done with them)
  for (int l = threadIdx.x; l < a.levels && l < kCtaHubLevels; l += blockDim.x)
    sh.hub[l] = a.lhub0[l + 1] > a.lhub0[l];
  lvl_arrive(&sh.bar, lane);
  lvl_wait(&sh.bar, sy.phase & 1u);
  ++sy.phase;
  int cur = 0;
  // ring positions of step i (descriptor), i + D (descriptor, entries), i + 2 D
  // (each ring slot of step j is j mod its ring size)
  int dq0 = 1, dq1 = (D + 1) % ND, dq2 = 0, eq0 = 0, eq1 = 0;
  // step i handles task warp + i W; the first 2 D steps only stage
  int t = warp - 2 * D * W;
  for (int i = -2 * D;; ++i, t += W) {
    if (i >= 0 && t >= nt) break;
    {   // descriptor of the task 2 D steps ahead
      const int td = t + 2 * D * W;
      if (td < nt && lane < 6)
        cp_async16(reinterpret_cast<char*>(&sm.desc[dq2]) + 16 * lane,
                   reinterpret_cast<const char*>(a.desc + td) + 16 * lane);
    }
    cp_async_wait<D - 1 < 0 ? 0 : D - 1>();
    __syncwarp();
    {   // entries and row records of the task D steps ahead
      const int te = t + D * W;
      if (te >= 0 && te < nt) {
        const CtaDesc& d = sm.desc[dq1];
        const int n4 = d.nent4 >> 2;
        const int32_t* gc = a.pcol + d.base;
        const double* gv = a.pval + d.base;
        for (int q = lane; q < n4; q += 32) cp_async16(&sm.col[eq1][4 * q], gc + 4 * q);
        for (int q = lane; q < 2 * n4; q += 32) cp_async16(&sm.val[eq1][2 * q], gv + 2 * q);
        if (d.tk.b != 0 && lane < (d.tk.b & 0xff))
          cp_async16(&sm.ri[eq1][lane], a.rinfo + d.tk.p + lane);
      }
    }
    cp_async_commit();
    if (i >= 0) {
      const CtaDesc& d = sm.desc[dq0];
      const int lev = d.lev;
      while (cur < lev) cta_level_end(a, sh, sy, cur++, warp, lane, W);
      unsigned long long* tr = a.ttrace ? a.ttrace + 3 * (int64_t)t : nullptr;
      if (tr && lane == 0) tr[0] = gtimer();
      cta_complete(a, d, sm.col[eq0], sm.val[eq0], sm.ri[eq0], lane, tr);
      if (tr && lane == 0) tr[2] = gtimer();
      // the warp's last task of this level: arrive now, stage under the wait
      const int tn = t + W;
      const int nlev = tn < nt ? sm.desc[dq0 + 1 == ND ? 0 : dq0 + 1].lev : 0x7fffffff;
      if (nlev > lev) {
        lvl_arrive(&sh.bar, lane);
        sy.arrived = true;
      } else {
        __syncwarp();   // the slot and the descriptor are reused D / 2 D steps on
      }
    }
    dq0 = dq0 + 1 == ND ? 0 : dq0 + 1;
    dq1 = dq1 + 1 == ND ? 0 : dq1 + 1;
    dq2 = dq2 + 1 == ND ? 0 : dq2 + 1;
    if (i >= 0) eq0 = eq0 + 1 == B ? 0 : eq0 + 1;
    if (i + D >= 0) eq1 = eq1 + 1 == B ? 0 : eq1 + 1;
  }
  cp_async_wait<0>();
  // remaining levels (every warp passes every level)
  while (cur < a.levels) cta_level_end(a, sh, sy, cur++, warp, lane, W);
}

template <int W, int B>
__global__ void __launch_bounds__(32 * W, 1) sweep_cta_kernel(CtaArgs args) {
  if (args.skip && *args.skip) return;
  extern __shared__ __align__(16) unsigned char cta_smem[];
  __shared__ CtaShared sh;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&sh.bar)),
                 "r"(W)
                 : "memory");
  __syncthreads();
  CtaSlots<B>& sm = reinterpret_cast<CtaSlots<B>*>(cta_smem)[warp];
  CtaSync sy{0u, false};
  cta_run_dir<B>(args.dir[0], sm, sh, sy, warp, lane, W);
  cta_run_dir<B>(args.dir[1], sm, sh, sy, warp, lane, W);
}

template <typename T>
static bool upload(T** dst, const std::vector<T>& v) {
  if (v.empty()) return true;
  if (cudaMalloc((void**)dst, sizeof(T) * v.size()) != cudaSuccess) return false;
  return cudaMemcpy(*dst, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice) == cudaSuccess;
}

// Launch configuration: clusters of kCluster CTAs (one CTA per SM) when the
// device allows a cooperative clustered launch, else plain cooperative.
struct SweepLaunch {
  int grid = 0;
  int csize = 1;
  bool probed = false;
};

static SweepLaunch& sweep_launch() {
  static SweepLaunch L;
  if (L.probed) return L;
  L.probed = true;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sweep_kernel, kSweepThreads, 0) !=
          cudaSuccess ||
      occ < 1)
    occ = 1;
  occ = std::min(occ, 1);
  L.grid = occ * dev_info().sm_count;
  L.csize = 1;
  const char* env = getenv("LG_SWEEP_CLUSTER");
  int want = env ? atoi(env) : 16;
  for (int cs : {want, 8}) {
    if (cs <= 1) break;
    if (cs > 8 && cudaFuncSetAttribute(sweep_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed,
                                       1) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(kSweepThreads);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, sweep_kernel, &cfg) == cudaSuccess &&
        nclusters >= 1) {
      L.csize = cs;
      L.grid = nclusters * cs;
      break;
    }
    cudaGetLastError();
  }
  if (getenv("LG_DEBUG"))
    fprintf(stderr, "[lapb200] sweep launch: grid %d, cluster %d\n", L.grid, L.csize);
  return L;
}

// omap (permuted factor, else NULL): factor row -> original row; the forward
// sweep reads b there and the backward sweep writes its second output there.
// omap (permuted factor, else NULL): factor row -> original row; the forward
// sweep reads b there and the backward sweep writes z there.  The backward
// sweep's right-hand side is the forward sweep's solution (factor numbering).
// Host half of make_sweep: the sweep's system in its level-merged form, b
// entries encoded as N + index.  flevels: depth of the factor's own DAG.
static bool build_system(int64_t n, std::vector<int64_t>& rp, std::vector<int32_t>& col,
                         std::vector<double>& val, const std::vector<double>& diag, bool forward,
                         const int32_t* omap, int passes, SweepSys& sys, int* flevels) {
  sys.n = sys.N = n;
  sys.rp.swap(rp);
  sys.col.swap(col);
  sys.val.swap(val);
  sys.dg = diag;
  sys.bidx.resize((size_t)n);
  sys.oidx.resize((size_t)n);
  sys.order.resize((size_t)n);
  for (int64_t r = 0; r < n; ++r) {
    sys.bidx[(size_t)r] = (int32_t)((forward && omap) ? omap[r] : r);
    sys.oidx[(size_t)r] = forward ? -1 : (int32_t)(omap ? omap[r] : r);
    sys.order[(size_t)r] = (int32_t)(forward ? r : n - 1 - r);
  }
  {
    std::vector<int32_t> lv;
    const int fl = dag_levels(sys, lv);
    if (flevels) *flevels = fl;
  }
  // two passes wherever the sweep is latency-bound; a third only on narrow
  // DAGs, where the extra entries are free (C3 809 -> 762 us, C2 121 -> 111 us;
  // C4's ~8 k-row levels lose with it)
  for (int p = 0; p < passes && 3 * sys.N < ((int64_t)1 << 31); ++p)
    if (!merge_levels(sys, p < 2 ? kMergeWide : kMergeNarrow)) break;
  if (!getenv("LG_IC0_NOHUBSORT")) {
    // A hub row (> kHubChunk entries) is cut into chunk tasks whose partials
    // chunk 0 sums -- a second hop after the last chunk.  Put the entries whose
    // sources sit deepest first: the late inputs then belong to chunk 0 itself,
    // the other chunks (early inputs only) are done long before, and the row
    // finishes one hop after its last input.  (Summation order changes within
    // the row: roundoff only, still fixed.)
    std::vector<int32_t> lv;
    dag_levels(sys, lv);
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t u = 0; u < sys.N; ++u) {
      const int64_t lo = sys.rp[(size_t)u], hi = sys.rp[(size_t)u + 1];
      if (hi - lo <= kHubChunk) continue;
      std::vector<std::pair<int32_t, int64_t>> key((size_t)(hi - lo));
      for (int64_t k = lo; k < hi; ++k) {
        const int32_t c = sys.col[(size_t)k];
        key[(size_t)(k - lo)] = {c < 0 ? -1 : lv[(size_t)c], k};
      }
      std::stable_sort(key.begin(), key.end(),
                       [](const std::pair<int32_t, int64_t>& a, const std::pair<int32_t, int64_t>& b) {
                         return a.first > b.first;
                       });
      std::vector<int32_t> c2((size_t)(hi - lo));
      std::vector<double> v2((size_t)(hi - lo));
      for (size_t q = 0; q < key.size(); ++q) {
        c2[q] = sys.col[(size_t)key[q].second];
        v2[q] = sys.val[(size_t)key[q].second];
      }
      std::copy(c2.begin(), c2.end(), sys.col.begin() + lo);
      std::copy(v2.begin(), v2.end(), sys.val.begin() + lo);
    }
  }
  // b entries: -1 - index  ->  N + index (entry_src on the device)
  for (int32_t& c : sys.col)
    if (c < 0) c = (int32_t)(sys.N + (-1 - (int64_t)c));
  // every entry reads an unknown of this sweep or one of the n right-hand-side
  // values, and every unknown has a nonzero pivot (the device trusts this)
  bool valid = true;
  for (const int32_t c : sys.col) valid = valid && c >= 0 && (int64_t)c < sys.N + n;
  for (int64_t u = 0; u < sys.N; ++u)
    valid = valid && sys.dg[(size_t)u] != 0.0 && sys.bidx[(size_t)u] < n && sys.oidx[(size_t)u] < n;
  if (!valid) {
    fprintf(stderr, "[lapb200] internal error: level-merged sweep system failed validation\n");
    return false;
  }
  return true;
}

static bool make_sweep(int64_t n, std::vector<int64_t>& rp, std::vector<int32_t>& col,
                       std::vector<double>& val, const std::vector<double>& diag, bool forward,
                       const int32_t* omap, SweepDev& d) {
  SweepSys sys;
  if (!build_system(n, rp, col, val, diag, forward, omap, merge_passes(), sys, &d.flevels))
    return false;
  SweepHost h;
  d.n = (int32_t)n;
  d.N = (int32_t)sys.N;
  d.nent = (int64_t)sys.col.size();
  const SweepLaunch& L = sweep_launch();
  const char* nm = getenv("LG_NARROW_MULT");
  const int mult = nm ? atoi(nm) : 1;
  build_sweep(sys, L.csize * kSweepWarps * mult, h);
  d.nsegs = (int32_t)h.segs.size();
  d.nbar = h.nbar;
  d.levels = h.levels;
  bool ok = upload(&d.pcol, h.pcol) && upload(&d.pval, h.pval) &&
            upload(&d.perm, h.perm) && upload(&d.pdiag, h.pdiag) && upload(&d.tasks, h.tasks) &&
            upload(&d.tbase, h.tbase) && upload(&d.lanetab, h.lanetab) &&
            upload(&d.segs, h.segs) && upload(&d.hub_first, h.hub_first) &&
            upload(&d.hub_nchunk, h.hub_nchunk) && upload(&d.tlevel, h.tlevel) &&
            upload(&d.lexpect, h.lexpect) && upload(&d.lhub0, h.lhub0) &&
            upload(&d.hub_prow, h.hub_prow);
  d.ntasks = (int32_t)h.tasks.size();
  {
    std::vector<CtaDesc> cd(h.tasks.size());
    for (size_t t = 0; t < h.tasks.size(); ++t) {
      CtaDesc& c = cd[t];
      c.tk = h.tasks[t];
      c.base = h.tbase[t];
      c.lev = h.tlevel[t];
      const int64_t end = t + 1 < h.tasks.size() ? h.tbase[t + 1] : (int64_t)h.pcol.size();
      c.nent4 = (int32_t)(end - h.tbase[t]);
      for (int ln = 0; ln < 32; ++ln) c.lanetab[ln] = h.lanetab[t * 32 + (size_t)ln];
    }
    CtaDesc* dp = nullptr;
    ok = ok && upload(&dp, cd);
    d.cdesc = dp;
  }
  d.nparts = h.nparts;
  {
    std::vector<RowInfo> ri((size_t)sys.N);
    std::vector<int32_t> oi((size_t)sys.N);
    for (int64_t p = 0; p < sys.N; ++p) {
      const int32_t r = h.perm[(size_t)p];
      ri[(size_t)p] = {h.pdiag[(size_t)p], r, sys.bidx[(size_t)r]};
      oi[(size_t)p] = sys.oidx[(size_t)r];
    }
    // (the level-barrier kernel indexes b and the output by unknown)
    ok = ok && upload(&d.rinfo, ri) && upload(&d.oidx, oi) && upload(&d.ubidx, sys.bidx) &&
         upload(&d.uoidx, sys.oidx);
  }
  if (ok && !h.lexpect.empty())
    ok = cudaMalloc(&d.lcount, 4 * h.lexpect.size()) == cudaSuccess &&
         cudaMemset(d.lcount, 0, 4 * h.lexpect.size()) == cudaSuccess;
  if (!ok) return false;
  if (!h.hub_first.empty()) {
    if (cudaMalloc(&d.hub_ticket, sizeof(unsigned) * h.hub_first.size()) != cudaSuccess ||
        cudaMemset(d.hub_ticket, 0, sizeof(unsigned) * h.hub_first.size()) != cudaSuccess ||
        cudaMalloc(&d.hub_part, sizeof(double) * (size_t)h.nparts) != cudaSuccess)
      return false;
  }
  if (cudaMalloc(&d.bar, sizeof(unsigned long long)) != cudaSuccess ||
      cudaMemset(d.bar, 0, sizeof(unsigned long long)) != cudaSuccess)
    return false;
  return true;
}

static void free_sweep(SweepDev& d) {
  cudaFree(d.prp);
  cudaFree(d.pcol);
  cudaFree(d.pval);
  cudaFree(d.perm);
  cudaFree(d.pdiag);
  cudaFree(d.tasks);
  cudaFree(d.tbase);
  cudaFree(d.lanetab);
  cudaFree(d.segs);
  cudaFree(d.hub_first);
  cudaFree(d.hub_nchunk);
  cudaFree(d.hub_ticket);
  cudaFree(d.hub_part);
  cudaFree(d.bar);
  cudaFree(d.tlevel);
  cudaFree(d.lexpect);
  cudaFree(d.lcount);
  cudaFree(d.ttrace);
  cudaFree(d.rinfo);
  cudaFree(d.oidx);
  cudaFree(d.lhub0);
  cudaFree(d.hub_prow);
  cudaFree(d.cdesc);
  cudaFree(d.ubidx);
  cudaFree(d.uoidx);
  d = SweepDev();
}

static SweepArgs sweep_args(const SweepDev& d, const double* b, double* x, const int* skip) {
  SweepArgs a;
  a.prp = d.prp;
  a.pcol = d.pcol;
  a.pval = d.pval;
  a.perm = d.perm;
  a.pdiag = d.pdiag;
  a.tasks = d.tasks;
  a.tbase = d.tbase;
  a.lanetab = d.lanetab;
  a.segs = d.segs;
  a.nsegs = d.nsegs;
  a.nbar = d.nbar;
  a.csize = sweep_launch().csize;
  a.hub_first = d.hub_first;
  a.hub_nchunk = d.hub_nchunk;
  a.hub_ticket = d.hub_ticket;
  a.hub_part = d.hub_part;
  a.bar = d.bar;
  a.b = b;
  a.x = x;
  a.bmap = d.ubidx;
  a.out2 = nullptr;
  a.omap = d.uoidx;
  a.skip = skip;
  a.trace = nullptr;
  const char* dbg = getenv("LG_SWEEP_DBG");
  a.dbg = dbg ? atoi(dbg) : 0;
  a.n = d.N;
  return a;
}

// LG_SWEEP_MODE=0 selects the level-barrier sweep (kept for comparison and
// for the per-level trace); the default is the dataflow sweep.
static int sweep_mode() {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("LG_SWEEP_MODE");
    mode = e ? atoi(e) : 1;
  }
  return mode;
}

static int sweep_gate() {
  static int g = -1;
  if (g < 0) {
    const char* e = getenv("LG_SWEEP_GATE");
    g = e ? std::max(1, atoi(e)) : 4;   // re-measured on the merged schedules: 2 / 3 / 4 / 5 -> C3 868 / 743 / 725 / 732 us
  }
  return g;
}

template <int THREADS, bool SM>
static size_t flow_smem() {
  return SM ? (size_t)(THREADS / 32 - 1) * 2 * kLaneMax * 32 * 12 : 0;
}

template <int THREADS, bool SM>
static int flow_grid() {
  static int grid = 0;
  if (!grid) {
    if (SM)
      cudaFuncSetAttribute(sweep_flow_kernel<THREADS, SM>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)flow_smem<THREADS, SM>());
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sweep_flow_kernel<THREADS, SM>,
                                                      THREADS, flow_smem<THREADS, SM>()) !=
            cudaSuccess ||
        occ < 1)
      occ = 1;
    grid = std::min(occ, 1) * dev_info().sm_count;
  }
  return grid;
}

template <int THREADS, bool SM>
static int launch_flow_t(const FlowArgs& a, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(flow_grid<THREADS, SM>());
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = flow_smem<THREADS, SM>();
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;   // all warps co-resident
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  LG_CUDA(cudaLaunchKernelEx(&cfg, sweep_flow_kernel<THREADS, SM>, a));
  return LG_OK;
}

static int launch_flow(const SweepDev& dv, const SweepDev& other, const double* b, double* x,
                       double* out2, double* next_x, const int* skip, cudaStream_t s) {
  const bool wide = (int64_t)dv.ntasks > (int64_t)kFlowWideTasks * std::max(1, dv.levels);
  FlowArgs a;
  a.pcol = dv.pcol;
  a.pval = dv.pval;
  a.rinfo = dv.rinfo;
  a.oidx = dv.oidx;
  a.tasks = dv.tasks;
  a.tbase = dv.tbase;
  a.lanetab = dv.lanetab;
  a.tlevel = dv.tlevel;
  a.lexpect = dv.lexpect;
  a.lcount = dv.lcount;
  a.hub_first = dv.hub_first;
  a.hub_nchunk = dv.hub_nchunk;
  a.hub_part = dv.hub_part;
  a.b = b;
  a.x = x;
  a.out2 = out2;
  a.skip = skip;
  a.ttrace = dv.ttrace;
  a.next_x = next_x;
  a.next_cnt = other.lcount;
  a.next_ncnt = other.levels * 32;
  a.next_part = other.hub_part;
  a.next_npart = other.nparts;
  a.ntasks = dv.ntasks;
  a.levels = dv.levels;
  a.n = dv.N;
  a.nreal = dv.n;
  a.next_n = other.N;
  a.defer_rearm = next_x == b;
  a.gate = sweep_gate();
  {
    const char* e = getenv("LG_SWEEP_BACKOFF");
    a.backoff = e ? (uint32_t)std::max(16, atoi(e)) : 16u;
  }
  // LG_FLOW_WIDE: 0 narrow CTA everywhere, 1 (default) the register-staged wide
  // CTA, 2 the shared-memory-staged one (23 worker warps) -- measured on the
  // merged C4 schedule: 560 / 534 / 552 us: beyond 15 warps the extra resident
  // tasks only add pollers
  static const int wide_kind = [] {
    const char* e = getenv("LG_FLOW_WIDE");
    return e ? atoi(e) : 1;
  }();
  if (wide && wide_kind == 2) return launch_flow_t<kFlowThreadsSm, true>(a, s);
  if (wide && wide_kind == 1) return launch_flow_t<kFlowThreadsWide, false>(a, s);
  return launch_flow_t<kFlowThreads, false>(a, s);
}

static CtaDir cta_dir(const SweepDev& dv, const double* b, double* x, double* out2) {
  CtaDir a;
  a.pcol = dv.pcol;
  a.pval = dv.pval;
  a.rinfo = dv.rinfo;
  a.oidx = dv.oidx;
  a.desc = static_cast<const CtaDesc*>(dv.cdesc);
  a.lhub0 = dv.lhub0;
  a.hub_prow = dv.hub_prow;
  a.hub_first = dv.hub_first;
  a.hub_nchunk = dv.hub_nchunk;
  a.hub_part = dv.hub_part;
  a.b = b;
  a.x = x;
  a.out2 = out2;
  a.ttrace = dv.ttrace;
  a.ntasks = dv.ntasks;
  a.levels = dv.levels;
  a.n = dv.N;
  return a;
}

template <int W, int B>
static int launch_cta_t(const CtaArgs& ca, cudaStream_t s) {
  constexpr size_t smem = sizeof(CtaSlots<B>) * W;
  static bool once = false;
  if (!once) {
    LG_CUDA(cudaFuncSetAttribute(sweep_cta_kernel<W, B>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    once = true;
  }
  sweep_cta_kernel<W, B><<<1, 32 * W, smem, s>>>(ca);
  LG_CUDA(cudaGetLastError());
  return LG_OK;
}

static int launch_cta(const CtaArgs& ca, int threads, cudaStream_t s) {
  switch (threads) {
    case 768: return launch_cta_t<24, 2>(ca, s);
    case 256: return launch_cta_t<8, 3>(ca, s);
    case 128: return launch_cta_t<4, 3>(ca, s);
    default: return launch_cta_t<16, 3>(ca, s);
  }
}

// Resident-sweep choice.  Measured on B200 (scripts/ic0_modes.py, r02aj):
// C1 53.6 us against 54.8 us for the dataflow sweeps, C2 287 against 175, C3
// 5,191 against 1,351 -- one SM completes a level step in ~0.9 us (0.19 us L2
// gather of x + 0.2 us reduce / divide / store + barrier and staging), no
// faster than the dataflow hop, and has 1/148 of the task throughput.  So it
// is opt-in only: LG_SWEEP_CTA=1, or lg_ic0_set_mode(f, 1).
static int pick_cta_mode(const lg_ic0*) {
  const char* e = getenv("LG_SWEEP_CTA");
  return e ? atoi(e) != 0 : 0;
}

static int launch_sweep(SweepArgs& args, cudaStream_t s) {
  const SweepLaunch& L = sweep_launch();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(L.grid);
  cfg.blockDim = dim3(kSweepThreads);
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int na = 0;
  at[na].id = cudaLaunchAttributeCooperative;
  at[na].val.cooperative = 1;
  ++na;
  if (L.csize > 1) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = L.csize;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  LG_CUDA(cudaLaunchKernelEx(&cfg, sweep_kernel, args));
  return LG_OK;
}

}  // namespace lg

using namespace lg;

// Strictly lower part of L by rows, its transpose by rows, and the diagonal
// (validated: lower triangular, sorted, the diagonal last in every row).
static int split_factor(int64_t n, const int64_t* l_rp, const int64_t* l_col, const double* l_val,
                        std::vector<int64_t>& frp, std::vector<int32_t>& fcol,
                        std::vector<double>& fval, std::vector<int64_t>& brp,
                        std::vector<int32_t>& bcol, std::vector<double>& bval,
                        std::vector<double>& dg) {
  // validate: lower triangular with the diagonal last in every row
  for (int64_t i = 0; i < n; ++i) {
    int64_t lo = l_rp[i], hi = l_rp[i + 1];
    if (hi <= lo || l_col[hi - 1] != i)
      return fail(LG_EINVAL, "lg_ic0_create: every row needs its diagonal last");
    for (int64_t k = lo; k < hi - 1; ++k)
      if (l_col[k] < 0 || l_col[k] >= i || (k > lo && l_col[k] <= l_col[k - 1]))
        return fail(LG_EINVAL, "lg_ic0_create: factor must be strictly lower, sorted");
    if (!(l_val[hi - 1] != 0.0)) return fail(LG_EINVAL, "lg_ic0_create: zero pivot");
  }
  const int64_t nnz = n ? l_rp[n] : 0;
  const int64_t noff = nnz - n;
  frp.assign((size_t)n + 1, 0);
  brp.assign((size_t)n + 1, 0);
  fcol.assign((size_t)noff, 0);
  bcol.assign((size_t)noff, 0);
  fval.assign((size_t)noff, 0.0);
  bval.assign((size_t)noff, 0.0);
  dg.assign((size_t)n, 0.0);
  for (int64_t i = 0; i < n; ++i) {
    int64_t lo = l_rp[i], hi = l_rp[i + 1] - 1;
    frp[(size_t)i + 1] = frp[(size_t)i] + (hi - lo);
    for (int64_t k = lo; k < hi; ++k) {
      fcol[(size_t)(frp[(size_t)i] + k - lo)] = (int32_t)l_col[k];
      fval[(size_t)(frp[(size_t)i] + k - lo)] = l_val[k];
      brp[(size_t)l_col[k] + 1]++;
    }
    dg[(size_t)i] = l_val[hi];
  }
  for (int64_t i = 0; i < n; ++i) brp[(size_t)i + 1] += brp[(size_t)i];
  {
    // transpose: row j of L^T lists i > j in ascending i
    std::vector<int64_t> fill(brp.begin(), brp.end() - 1);
    for (int64_t i = 0; i < n; ++i)
      for (int64_t k = frp[(size_t)i]; k < frp[(size_t)i + 1]; ++k) {
        int64_t j = fcol[(size_t)k];
        bcol[(size_t)fill[(size_t)j]] = (int32_t)i;
        bval[(size_t)fill[(size_t)j]] = fval[(size_t)k];
        fill[(size_t)j]++;
      }
  }
  return LG_OK;
}

extern "C" {

int lg_ic0_factorize(int64_t n, const int64_t* rp, const int64_t* col,
                     const double* val, double shift0, const double* sched,
                     int nsched, int64_t* l_rp, int64_t* l_col, double* l_val,
                     double* shift, int* attempts) {
  if (n < 0 || !rp || (rp[n] > 0 && (!col || !val)) || !l_rp || !shift || !attempts ||
      nsched < 0 || (nsched > 0 && !sched))
    return fail(LG_EINVAL, "lg_ic0_factorize: bad argument");
  // split A into its strictly-lower pattern + diagonal (ic0.py:94-101)
  std::vector<double> diag((size_t)n, 0.0);
  std::vector<int64_t> lrp((size_t)n + 1, 0);
  for (int64_t i = 0; i < n; ++i) {
    int64_t c = 0;
    for (int64_t k = rp[i]; k < rp[i + 1] && col[k] < i; ++k) ++c;
    lrp[(size_t)i + 1] = lrp[(size_t)i] + c + 1;
  }
  const int64_t nl = lrp[(size_t)n];
  std::vector<int64_t> lcol((size_t)nl);
  std::vector<double> aval((size_t)nl, 0.0);
  for (int64_t i = 0; i < n; ++i) {
    int64_t o = lrp[(size_t)i];
    int64_t k = rp[i];
    for (; k < rp[i + 1] && col[k] < i; ++k) {
      lcol[(size_t)o] = col[k];
      aval[(size_t)o] = val[k];
      ++o;
    }
    if (k < rp[i + 1] && col[k] == i) diag[(size_t)i] = val[k];
    lcol[(size_t)o] = i;  // diagonal slot
  }
  double dmax = 0.0;
  for (int64_t i = 0; i < n; ++i) dmax = (i == 0) ? diag[0] : std::max(dmax, diag[(size_t)i]);
  // shift ladder (ic0.py:98-111)
  std::vector<double> shifts{shift0};
  for (int s = 0; s < nsched; ++s)
    if (sched[s] > shift0) shifts.push_back(sched[s]);
  const double last = 0.1 * dmax;
  if (dmax > 0 && (shifts.empty() || last > shifts.back())) shifts.push_back(last);
  std::vector<double> lval((size_t)nl, 0.0);
  // dependency levels of the lower pattern, rows grouped by level
  std::vector<int64_t> order((size_t)n), lstart;
  {
    std::vector<int32_t> lev((size_t)n, 0);
    int32_t maxl = -1;
    for (int64_t i = 0; i < n; ++i) {
      int32_t l = 0;
      for (int64_t t = lrp[(size_t)i]; t < lrp[(size_t)i + 1] - 1; ++t)
        l = std::max(l, lev[(size_t)lcol[(size_t)t]] + 1);
      lev[(size_t)i] = l;
      maxl = std::max(maxl, l);
    }
    lstart.assign((size_t)maxl + 2, 0);
    for (int64_t i = 0; i < n; ++i) lstart[(size_t)lev[(size_t)i] + 1]++;
    for (int32_t l = 0; l <= maxl; ++l) lstart[(size_t)l + 1] += lstart[(size_t)l];
    std::vector<int64_t> fill(lstart.begin(), lstart.end() - 1);
    for (int64_t i = 0; i < n; ++i) order[(size_t)fill[(size_t)lev[(size_t)i]]++] = i;
  }
  // per-thread column maps of the row being factored (stamp | pos, 16 B a
  // node each): 16 threads x 0.5 GB at C5 size
  const int nthr = std::max(1, std::min(omp_get_max_threads(), 64));
  std::vector<std::vector<int64_t>> maps((size_t)nthr, std::vector<int64_t>(2 * (size_t)n));
  int tries = 0;
  for (double alpha : shifts) {
    ++tries;
    if (ic0_attempt(n, diag, lrp, lcol, aval, alpha, lval, order, lstart, maps)) {
      std::memcpy(l_rp, lrp.data(), sizeof(int64_t) * (size_t)(n + 1));
      std::memcpy(l_col, lcol.data(), sizeof(int64_t) * (size_t)nl);
      std::memcpy(l_val, lval.data(), sizeof(double) * (size_t)nl);
      *shift = alpha;
      *attempts = tries;
      return LG_OK;
    }
  }
  *attempts = tries;
  return fail(LG_EBREAKDOWN, "pivot breakdown at every shift");
}

int lg_ic0_create(int64_t n, const int64_t* l_rp, const int64_t* l_col,
                  const double* l_val, lg_ic0** out) {
  return lg_ic0_create_perm(n, l_rp, l_col, l_val, nullptr, out);
}

int lg_ic0_create_perm(int64_t n, const int64_t* l_rp, const int64_t* l_col,
                       const double* l_val, const int64_t* perm_h, lg_ic0** out) {
  if (!out || n < 0 || !l_rp || (n > 0 && (!l_col || !l_val)))
    return fail(LG_EINVAL, "lg_ic0_create: bad argument");
  if (n >= ((int64_t)1 << 31)) return fail(LG_EINVAL, "lg_ic0_create: n too large");
  std::vector<int64_t> frp, brp;
  std::vector<int32_t> fcol, bcol;
  std::vector<double> fval, bval, dg;
  {
    const int rc = split_factor(n, l_rp, l_col, l_val, frp, fcol, fval, brp, bcol, bval, dg);
    if (rc) return rc;
  }
  const int64_t nnz = n ? l_rp[n] : 0;
  std::vector<int32_t> om;
  if (perm_h) {
    om.resize((size_t)n);
    std::vector<char> seen((size_t)n, 0);
    for (int64_t i = 0; i < n; ++i) {
      if (perm_h[i] < 0 || perm_h[i] >= n || seen[(size_t)perm_h[i]])
        return fail(LG_EINVAL, "lg_ic0_create_perm: perm is not a permutation");
      seen[(size_t)perm_h[i]] = 1;
      om[(size_t)i] = (int32_t)perm_h[i];
    }
  }
  const int32_t* omp = perm_h ? om.data() : nullptr;
  lg_ic0* f = new lg_ic0();
  f->n = n;
  f->nnz_l = nnz;
  bool ok = make_sweep(n, frp, fcol, fval, dg, true, omp, f->fwd) &&
            make_sweep(n, brp, bcol, bval, dg, false, omp, f->bwd) && upload(&f->diag, dg) &&
            (n == 0 || (cudaMalloc(&f->tmp, 8 * (size_t)f->fwd.N) == cudaSuccess &&
                        cudaMalloc(&f->xb, 8 * (size_t)f->bwd.N) == cudaSuccess));
  if (ok && n) {   // arm the dataflow forward sweep (all-ones = the x sentinel)
    ok = cudaMemset(f->tmp, 0xff, 8 * (size_t)f->fwd.N) == cudaSuccess &&
         cudaMemset(f->xb, 0xff, 8 * (size_t)f->bwd.N) == cudaSuccess;
    for (SweepDev* d : {&f->fwd, &f->bwd})
      if (ok && d->nparts)
        ok = cudaMemset(d->hub_part, 0xff, 8 * (size_t)d->nparts) == cudaSuccess;
    f->flow_armed = ok;
  }
  if (!ok) {
    lg_ic0_destroy(f);
    return fail(LG_ENOMEM, "lg_ic0_create: device allocation / upload failed");
  }
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) {
    lg_ic0_destroy(f);
    return fail(LG_ECUDA, std::string("lg_ic0_create: ") + cudaGetErrorString(err));
  }
  f->grid = sweep_launch().grid;
  f->cta_mode = pick_cta_mode(f);
  {
    const char* e = getenv("LG_SWEEP_CTA_THREADS");
    f->cta_threads = e ? atoi(e) : 512;
  }
  *out = f;
  return LG_OK;
}

// Sweep implementation of a factor: 0 dataflow sweeps, 1 resident CTA sweep
// (the default is chosen at creation from the level widths).  Both give the
// same bits; returns the previous mode.
int lg_ic0_set_mode(lg_ic0* f, int mode) {
  if (!f) return fail(LG_EINVAL, "lg_ic0_set_mode: NULL handle");
  const int prev = f->cta_mode;
  if (mode == 0 || mode == 1) f->cta_mode = mode;
  return prev;
}

// Debug: record a device timestamp after every level segment of both sweeps
// (CTA 0's view) into a host array of fwd.nsegs + bwd.nsegs entries.
int lg_ic0_trace(lg_ic0* f, int enable, unsigned long long* host_out, int cap) {
  if (!f) return fail(LG_EINVAL, "lg_ic0_trace: NULL handle");
  const int total = f->fwd.nsegs + f->bwd.nsegs;
  if (enable && !f->trace) {
    if (cudaMalloc(&f->trace, sizeof(unsigned long long) * (size_t)(total + 2)) != cudaSuccess)
      return fail(LG_ENOMEM, "lg_ic0_trace: alloc");
    cudaMemset(f->trace, 0, sizeof(unsigned long long) * (size_t)(total + 2));
  }
  if (host_out && f->trace) {
    LG_CUDA(cudaDeviceSynchronize());
    LG_CUDA(cudaMemcpy(host_out, f->trace,
                       sizeof(unsigned long long) * (size_t)std::min(cap, total + 2),
                       cudaMemcpyDeviceToHost));
  }
  if (!enable && f->trace) {
    cudaFree(f->trace);
    f->trace = nullptr;
  }
  return total;
}

// Debug: dataflow sweep task timestamps.  enable=1 allocates the buffers
// (the following applies record); host_out receives, per sweep direction,
// ntasks records {level, start, inputs ready, done} (ns, globaltimer).
// Returns the total number of records (fwd + bwd).
int lg_ic0_flow_trace(lg_ic0* f, int enable, unsigned long long* host_out, int cap) {
  if (!f) return fail(LG_EINVAL, "lg_ic0_flow_trace: NULL handle");
  const int total = f->fwd.ntasks + f->bwd.ntasks;
  SweepDev* dirs[2] = {&f->fwd, &f->bwd};
  if (enable) {
    for (SweepDev* d : dirs)
      if (!d->ttrace && d->ntasks &&
          cudaMalloc(&d->ttrace, 24 * (size_t)d->ntasks) != cudaSuccess)
        return fail(LG_ENOMEM, "lg_ic0_flow_trace: alloc");
  }
  if (host_out) {
    LG_CUDA(cudaDeviceSynchronize());
    int k = 0;
    for (SweepDev* d : dirs) {
      if (!d->ttrace) continue;
      std::vector<unsigned long long> tr(3 * (size_t)d->ntasks);
      std::vector<int32_t> lv((size_t)d->ntasks);
      LG_CUDA(cudaMemcpy(tr.data(), d->ttrace, 24 * (size_t)d->ntasks, cudaMemcpyDeviceToHost));
      LG_CUDA(cudaMemcpy(lv.data(), d->tlevel, 4 * (size_t)d->ntasks, cudaMemcpyDeviceToHost));
      for (int t = 0; t < d->ntasks && 4 * (k + 1) <= cap; ++t, ++k) {
        host_out[4 * k] = (unsigned long long)lv[(size_t)t];
        for (int j = 0; j < 3; ++j) host_out[4 * k + 1 + j] = tr[3 * (size_t)t + j];
      }
    }
  }
  if (!enable) {
    for (SweepDev* d : dirs) {
      cudaFree(d->ttrace);
      d->ttrace = nullptr;
    }
  }
  return total;
}

// Debug: per-segment schedule statistics {tasks, rows, entries, narrow}
int lg_ic0_schedule(const lg_ic0* f, int backward, int* host_out, int cap) {
  if (!f) return fail(LG_EINVAL, "lg_ic0_schedule: NULL handle");
  const SweepDev& d = backward ? f->bwd : f->fwd;
  std::vector<SweepSeg> segs((size_t)d.nsegs);
  if (d.nsegs)
    cudaMemcpy(segs.data(), d.segs, sizeof(SweepSeg) * (size_t)d.nsegs, cudaMemcpyDeviceToHost);
  for (int i = 0; i < d.nsegs && 4 * i + 3 < cap; ++i) {
    host_out[4 * i] = segs[(size_t)i].t1 - segs[(size_t)i].t0;
    host_out[4 * i + 1] = segs[(size_t)i].narrow;
    host_out[4 * i + 2] = segs[(size_t)i].barrier;
    host_out[4 * i + 3] = 0;
  }
  return d.nsegs;
}

// Greedy colouring in smallest-last order (Matula-Beck degeneracy order with
// a bucket queue, then first-fit in reverse removal order).  Used by the
// flagged multicolour IC(0) variant: ordering nodes by (colour, id) makes the
// factor's sweeps take #colours levels.
int lg_color_smallest_last(int64_t n, const int64_t* rp, const int64_t* col, int32_t* color,
                           int32_t* ncolors) {
  if (n < 0 || (n > 0 && (!rp || !color || !ncolors)))
    return fail(LG_EINVAL, "lg_color_smallest_last: bad argument");
  std::vector<int64_t> deg((size_t)n);
  int64_t maxd = 0;
  for (int64_t v = 0; v < n; ++v) {
    int64_t d = 0;
    for (int64_t k = rp[v]; k < rp[v + 1]; ++k) d += (col[k] != v);
    deg[(size_t)v] = d;
    maxd = std::max(maxd, d);
  }
  // bucket queue: doubly linked lists per degree
  std::vector<int64_t> head((size_t)maxd + 1, -1), nxt((size_t)n, -1), prv((size_t)n, -1);
  auto push = [&](int64_t v) {
    const int64_t d = deg[(size_t)v];
    nxt[(size_t)v] = head[(size_t)d];
    prv[(size_t)v] = -1;
    if (head[(size_t)d] >= 0) prv[(size_t)head[(size_t)d]] = v;
    head[(size_t)d] = v;
  };
  auto unlink = [&](int64_t v) {
    const int64_t d = deg[(size_t)v];
    if (prv[(size_t)v] >= 0) nxt[(size_t)prv[(size_t)v]] = nxt[(size_t)v];
    else head[(size_t)d] = nxt[(size_t)v];
    if (nxt[(size_t)v] >= 0) prv[(size_t)nxt[(size_t)v]] = prv[(size_t)v];
  };
  for (int64_t v = n - 1; v >= 0; --v) push(v);
  std::vector<char> removed((size_t)n, 0);
  std::vector<int64_t> order;
  order.reserve((size_t)n);
  int64_t cur = 0;
  for (int64_t it = 0; it < n; ++it) {
    if (cur > 0) --cur;
    while (head[(size_t)cur] < 0) ++cur;
    const int64_t v = head[(size_t)cur];
    unlink(v);
    removed[(size_t)v] = 1;
    order.push_back(v);
    for (int64_t k = rp[v]; k < rp[v + 1]; ++k) {
      const int64_t u = col[k];
      if (u == v || removed[(size_t)u]) continue;
      unlink(u);
      --deg[(size_t)u];
      push(u);
    }
  }
  std::vector<int32_t> c((size_t)n, -1);
  std::vector<int64_t> mark;
  int32_t nc = 0;
  for (int64_t it = n - 1; it >= 0; --it) {
    const int64_t v = order[(size_t)it];
    if ((int64_t)mark.size() < nc + 1) mark.resize((size_t)nc + 1, -1);
    for (int64_t k = rp[v]; k < rp[v + 1]; ++k) {
      const int64_t u = col[k];
      if (u != v && c[(size_t)u] >= 0) mark[(size_t)c[(size_t)u]] = v;
    }
    int32_t cc = 0;
    while (cc < nc && mark[(size_t)cc] == v) ++cc;
    c[(size_t)v] = cc;
    if (cc == nc) ++nc;
  }
  for (int64_t v = 0; v < n; ++v) color[v] = c[(size_t)v];
  *ncolors = nc;
  return LG_OK;
}

int lg_ic0_destroy(lg_ic0* f) {
  if (!f) return LG_OK;
  cudaFree(f->trace);
  free_sweep(f->fwd);
  free_sweep(f->bwd);
  cudaFree(f->diag);
  cudaFree(f->tmp);
  cudaFree(f->xb);
  delete f;
  return LG_OK;
}

int lg_ic0_info(const lg_ic0* f, int64_t* n, int64_t* nnz_l, int* levels) {
  if (!f) return fail(LG_EINVAL, "lg_ic0_info: NULL handle");
  if (n) *n = f->n;
  if (nnz_l) *nnz_l = f->nnz_l;
  if (levels) *levels = std::max(f->fwd.flevels, f->bwd.flevels);
  return LG_OK;
}

// Host-only (no device): one triangular solve through the level-merged system
// the device would run -- forward (L y = b) or backward (L^T y = b) -- in the
// system's topological order.  Test hook for the host transformation: y must
// equal the plain substitution to roundoff for any number of passes.
int lg_ic0_merged_solve_host(int64_t n, const int64_t* l_rp, const int64_t* l_col,
                             const double* l_val, int passes, int backward, const double* b,
                             double* y, int* depth, int64_t* entries, int64_t* unknowns) {
  if (n < 0 || !l_rp || (n > 0 && (!l_col || !l_val || !b || !y)))
    return fail(LG_EINVAL, "lg_ic0_merged_solve_host: bad argument");
  std::vector<int64_t> frp, brp;
  std::vector<int32_t> fcol, bcol;
  std::vector<double> fval, bval, dg;
  const int rc = split_factor(n, l_rp, l_col, l_val, frp, fcol, fval, brp, bcol, bval, dg);
  if (rc) return rc;
  SweepSys sys;
  const bool ok = backward ? build_system(n, brp, bcol, bval, dg, false, nullptr, passes, sys, nullptr)
                           : build_system(n, frp, fcol, fval, dg, true, nullptr, passes, sys, nullptr);
  if (!ok) return fail(LG_EINVAL, "lg_ic0_merged_solve_host: system failed validation");
  std::vector<int32_t> lv;
  const int dep = dag_levels(sys, lv);
  std::vector<double> x((size_t)sys.N, 0.0);
  for (int64_t q = 0; q < sys.N; ++q) {
    const int32_t u = sys.order[(size_t)q];
    double sum = 0.0;
    for (int64_t k = sys.rp[(size_t)u]; k < sys.rp[(size_t)u + 1]; ++k) {
      const int32_t c = sys.col[(size_t)k];
      sum += sys.val[(size_t)k] * (c >= sys.N ? b[c - sys.N] : x[(size_t)c]);
    }
    const double bv = sys.bidx[(size_t)u] >= 0 ? b[sys.bidx[(size_t)u]] : 0.0;
    x[(size_t)u] = (bv - sum) / sys.dg[(size_t)u];
  }
  for (int64_t i = 0; i < n; ++i) y[i] = x[(size_t)i];
  if (depth) *depth = dep;
  if (entries) *entries = (int64_t)sys.col.size();
  if (unknowns) *unknowns = sys.N;
  return LG_OK;
}

int lg_ic0_sweep_depth(const lg_ic0* f, int* fwd, int* bwd, int64_t* entries) {
  if (!f) return fail(LG_EINVAL, "lg_ic0_sweep_depth: NULL handle");
  if (fwd) *fwd = f->fwd.levels;
  if (bwd) *bwd = f->bwd.levels;
  if (entries) *entries = f->fwd.nent + f->bwd.nent;
  return LG_OK;
}

int lg_ic0_apply(const lg_ic0* f, const double* r, double* z, const int* skip,
                 void* stream) {
  if (!f || !r || !z) return fail(LG_EINVAL, "lg_ic0_apply: NULL argument");
  if (f->n == 0) return LG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  // forward: b = r, unknowns in tmp; backward: b = tmp, unknowns in xb, z
  // written through the sweep's output map.  r is only read by the forward
  // launch, so z may alias r.
  if (f->cta_mode && sweep_mode() != 0 && !f->trace) {
    CtaArgs ca;
    ca.dir[0] = cta_dir(f->fwd, r, f->tmp, nullptr);
    ca.dir[1] = cta_dir(f->bwd, f->tmp, f->xb, z);
    ca.skip = skip;
    f->flow_armed = false;   // tmp now holds values, not the dataflow sentinels
    return launch_cta(ca, f->cta_threads, s);
  }
  if (sweep_mode() != 0 && !f->trace) {
    if (!f->flow_armed) {   // arm the forward sweep (after a barrier / resident apply)
      flow_init_kernel<<<vec_grid(f->fwd.N), kThreads, 0, s>>>(
          f->tmp, f->fwd.N, f->fwd.lcount, f->fwd.levels * 32, f->fwd.hub_part, f->fwd.nparts,
          nullptr);
      LG_CUDA(cudaGetLastError());
      f->flow_armed = true;
    }
    int rc = launch_flow(f->fwd, f->bwd, r, f->tmp, nullptr, f->xb, skip, s);
    if (rc) return rc;
    return launch_flow(f->bwd, f->fwd, f->tmp, f->xb, z, f->tmp, skip, s);
  }
  SweepArgs fa = sweep_args(f->fwd, r, f->tmp, skip);
  SweepArgs ba = sweep_args(f->bwd, f->tmp, f->xb, skip);
  ba.out2 = z;
  if (f->trace) {
    // layout: fwd segs, fwd inline-stage counter, bwd segs, bwd counter
    fa.trace = f->trace;
    ba.trace = f->trace + f->fwd.nsegs + 1;
  }
  f->flow_armed = false;
  int rc = launch_sweep(fa, s);
  if (rc) return rc;
  return launch_sweep(ba, s);
}

}  // extern "C"
