// Host symbolic analysis -- see symbolic.h.  Steps:
//   1. validate the pose graph (self edges, indices, every variable has a cost);
//   2. minimum-degree ordering on the elimination graph, lowest index breaks ties
//      (reading A16);
//   3. elimination tree + column structures; postorder relabelling;
//   4. fundamental supernodes, then relaxed amalgamation (App. F heuristics, our pinned rule);
//   5. panel layout, level schedule, gather-form update lists, solve lists, assembly lists.
#include "symbolic.h"

#include <algorithm>
#include <functional>
#include <map>
#include <queue>
#include <sstream>
#include <utility>

namespace dnls {

namespace {

using VI = std::vector<int32_t>;

VI min_degree_order(int N, const std::vector<VI>& adj0) {
  std::vector<VI> adj = adj0;
  std::vector<char> alive(N, 1);
  VI deg(N);
  typedef std::pair<int, int> PII;
  std::priority_queue<PII, std::vector<PII>, std::greater<PII>> pq;
  for (int v = 0; v < N; ++v) {
    deg[v] = (int)adj[v].size();
    pq.push(PII(deg[v], v));
  }
  VI order;
  order.reserve(N);
  VI merged;
  while (!pq.empty()) {
    PII top = pq.top();
    pq.pop();
    int v = top.second;
    if (!alive[v] || top.first != deg[v]) continue;
    alive[v] = 0;
    order.push_back(v);
    const VI nb = adj[v];
    for (int a : nb) {
      merged.clear();
      std::set_union(adj[a].begin(), adj[a].end(), nb.begin(), nb.end(), std::back_inserter(merged));
      VI out;
      out.reserve(merged.size());
      for (int x : merged)
        if (x != a && x != v) out.push_back(x);
      adj[a].swap(out);
      deg[a] = (int)adj[a].size();
      pq.push(PII(deg[a], a));
    }
    adj[v].clear();
  }
  return order;
}

// column structures (below-diagonal block rows, permuted) and etree for a given order
void structures(int N, const std::vector<VI>& adj, const VI& perm, VI& iperm, VI& parent,
                std::vector<VI>& cs) {
  iperm.assign(N, 0);
  for (int k = 0; k < N; ++k) iperm[perm[k]] = k;
  parent.assign(N, -1);
  cs.assign(N, VI());
  std::vector<VI> children(N);
  VI tmp;
  for (int k = 0; k < N; ++k) {
    VI s;
    for (int a : adj[perm[k]]) {
      int pa = iperm[a];
      if (pa > k) s.push_back(pa);
    }
    std::sort(s.begin(), s.end());
    for (int c : children[k]) {
      tmp.clear();
      std::set_union(s.begin(), s.end(), cs[c].begin(), cs[c].end(), std::back_inserter(tmp));
      s.clear();
      for (int x : tmp)
        if (x != k) s.push_back(x);
    }
    cs[k] = s;
    if (!s.empty()) {
      parent[k] = s[0];
      children[s[0]].push_back(k);
    }
  }
}

}  // namespace

std::string analyze(int D, int N, int E, const int32_t* edges, int P, const int32_t* priors,
                    const SymbolicOptions& opt, Symbolic& S, int* code) {
  *code = 0;
  std::ostringstream err;
  if (D != 3 && D != 6) {
    *code = 1;
    err << "dnls_graph_create: group must be DNLS_SE2 (3) or DNLS_SE3 (6), got " << D;
    return err.str();
  }
  if (N < 1 || E < 0 || P < 0 || (E > 0 && !edges) || (P > 0 && !priors)) {
    *code = 1;
    err << "dnls_graph_create: invalid counts/pointers (num_vars=" << N << ", num_edges=" << E
        << ", num_priors=" << P << ")";
    return err.str();
  }
  S = Symbolic();
  S.D = D;
  S.N = N;
  S.E = E;
  S.P = P;
  S.edges.assign(edges, edges + 2 * (size_t)E);
  S.prior_vars.assign(priors, priors + P);
  std::vector<int> has_cost(N, 0);
  std::vector<VI> adj(N);
  for (int e = 0; e < E; ++e) {
    int i = edges[2 * e], j = edges[2 * e + 1];
    if (i < 0 || i >= N || j < 0 || j >= N) {
      *code = 2;
      err << "dnls_graph_create: edge " << e << " = (" << i << ", " << j << ") out of range [0, " << N << ")";
      return err.str();
    }
    if (i == j) {
      *code = 3;
      err << "dnls_graph_create: edge " << e << " is a self edge (" << i << ", " << j << ")";
      return err.str();
    }
    has_cost[i] = has_cost[j] = 1;
    adj[i].push_back(j);
    adj[j].push_back(i);
  }
  for (int k = 0; k < P; ++k) {
    int v = priors[k];
    if (v < 0 || v >= N) {
      *code = 2;
      err << "dnls_graph_create: prior " << k << " on variable " << v << " out of range [0, " << N << ")";
      return err.str();
    }
    has_cost[v] = 1;
  }
  for (int v = 0; v < N; ++v)
    if (!has_cost[v]) {
      *code = 3;
      err << "dnls_graph_create: variable " << v << " has no cost (empty diagonal block; structurally singular)";
      return err.str();
    }
  for (auto& a : adj) {
    std::sort(a.begin(), a.end());
    a.erase(std::unique(a.begin(), a.end()), a.end());
  }
  int64_t pairs = 0;
  for (int v = 0; v < N; ++v) pairs += (int64_t)adj[v].size();
  S.nnz_H_blocks = N + pairs / 2;

  // ---- 2. ordering, 3. etree + postorder
  VI order = min_degree_order(N, adj);
  VI iperm, parent;
  std::vector<VI> cs;
  structures(N, adj, order, iperm, parent, cs);
  {
    std::vector<VI> children(N);
    VI roots;
    for (int k = 0; k < N; ++k) {
      if (parent[k] < 0) roots.push_back(k);
      else children[parent[k]].push_back(k);
    }
    VI post(N);
    int cnt = 0;
    std::vector<std::pair<int, int>> stack;
    for (int r : roots) {
      stack.push_back(std::make_pair(r, 0));
      while (!stack.empty()) {
        int v = stack.back().first;
        int& ci = stack.back().second;
        if (ci < (int)children[v].size()) {
          int c = children[v][ci++];
          stack.push_back(std::make_pair(c, 0));
        } else {
          post[v] = cnt++;
          stack.pop_back();
        }
      }
    }
    VI perm2(N);
    for (int k = 0; k < N; ++k) perm2[post[k]] = order[k];
    order.swap(perm2);
  }
  structures(N, adj, order, iperm, parent, cs);
  S.perm = order;
  S.iperm = iperm;
  S.parent = parent;
  S.colstruct = cs;
  {
    VI h(N, 1);
    int hmax = 0;
    for (int k = 0; k < N; ++k) {
      if (parent[k] >= 0) h[parent[k]] = std::max(h[parent[k]], h[k] + 1);
      hmax = std::max(hmax, h[k]);
    }
    S.etree_height = hmax;
  }
  S.nnz_L_blocks = N;
  S.nnz_L = 0;
  S.factor_flops = 0;
  for (int k = 0; k < N; ++k) {
    S.nnz_L_blocks += (int64_t)cs[k].size();
    S.nnz_L += (int64_t)D * (D + 1) / 2 + (int64_t)D * D * (int64_t)cs[k].size();
    for (int a = 0; a < D; ++a) {
      double m = (double)(D - 1 - a) + (double)D * cs[k].size();
      S.factor_flops += (m + 1) * (m + 1);
    }
  }

  // ---- 4. fundamental supernodes
  VI nchild(N, 0);
  for (int k = 0; k < N; ++k)
    if (parent[k] >= 0) nchild[parent[k]]++;
  struct SN {
    int first, ncols;
    VI rows;          // below rows
    int64_t zeros;    // explicit zero blocks in the lower part of the panel
    int parent;
    bool alive;
  };
  std::vector<SN> sns;
  VI col_sn(N);
  for (int k = 0; k < N; ++k) {
    bool join = k > 0 && parent[k - 1] == k && nchild[k] == 1 && cs[k - 1].size() == cs[k].size() + 1;
    if (join) {
      sns.back().ncols++;
      sns.back().rows = cs[k];
    } else {
      SN s;
      s.first = k;
      s.ncols = 1;
      s.rows = cs[k];
      s.zeros = 0;
      s.parent = -1;
      s.alive = true;
      sns.push_back(s);
    }
    col_sn[k] = (int)sns.size() - 1;
  }
  for (size_t s = 0; s < sns.size(); ++s) {
    int last = sns[s].first + sns[s].ncols - 1;
    sns[s].parent = parent[last] >= 0 ? col_sn[parent[last]] : -1;
  }
  // relaxed amalgamation: merge the contiguous last child into its parent
  {
    std::vector<VI> kids(sns.size());
    for (size_t s = 0; s < sns.size(); ++s)
      if (sns[s].parent >= 0) kids[sns[s].parent].push_back((int)s);
    auto total_blocks = [](int ncols, size_t nrows) {
      return (int64_t)ncols * (ncols + 1) / 2 + (int64_t)ncols * (int64_t)nrows;
    };
    for (size_t p = 0; p < sns.size(); ++p) {
      while (true) {
        SN& P = sns[p];
        int cidx = -1;
        for (int c : kids[p])
          if (sns[c].alive && sns[c].first + sns[c].ncols == P.first) cidx = c;
        if (cidx < 0) break;
        SN& C = sns[cidx];
        int w = C.ncols + P.ncols;
        // zeros added in C's columns: merged rows for C cols = P cols + P rows, C had |C.rows|
        int64_t newz = (int64_t)C.ncols * ((int64_t)P.ncols + (int64_t)P.rows.size() - (int64_t)C.rows.size());
        int64_t z = C.zeros + P.zeros + newz;
        double frac = (double)z / (double)total_blocks(w, P.rows.size());
        bool ok;
        if (w > opt.relax_max_cols) ok = false;
        else if (w <= opt.relax_always_cols) ok = true;
        else if (w <= opt.relax_small_cols) ok = frac <= opt.relax_small_frac;
        else if (w <= opt.relax_mid_cols) ok = frac <= opt.relax_mid_frac;
        else ok = frac <= opt.relax_big_frac;
        if (!ok) break;
        P.first = C.first;
        P.ncols = w;
        P.zeros = z;
        C.alive = false;
        for (int g : kids[cidx]) {
          sns[g].parent = (int)p;
          kids[p].push_back(g);
        }
      }
    }
  }
  // compact
  {
    VI remap(sns.size(), -1);
    std::vector<SN> out;
    for (size_t s = 0; s < sns.size(); ++s)
      if (sns[s].alive) {
        remap[s] = (int)out.size();
        out.push_back(sns[s]);
      }
    std::sort(out.begin(), out.end(), [](const SN& a, const SN& b) { return a.first < b.first; });
    // recompute parents from columns
    for (size_t s = 0; s < out.size(); ++s)
      for (int k = out[s].first; k < out[s].first + out[s].ncols; ++k) col_sn[k] = (int)s;
    for (size_t s = 0; s < out.size(); ++s) {
      int last = out[s].first + out[s].ncols - 1;
      out[s].parent = parent[last] >= 0 ? col_sn[parent[last]] : -1;
    }
    sns.swap(out);
  }
  // split supernodes wider than relax_max_cols into consecutive pieces (always valid: piece k's
  // rows are the later pieces' columns followed by the original below rows)
  {
    std::vector<SN> out;
    for (const SN& sn : sns) {
      if (sn.ncols <= opt.relax_max_cols) {
        out.push_back(sn);
        continue;
      }
      int nf = sn.first, rem = sn.ncols;
      while (rem > 0) {
        int c = std::min(rem, opt.relax_max_cols);
        SN piece = sn;
        piece.first = nf;
        piece.ncols = c;
        piece.rows.clear();
        for (int k = nf + c; k < sn.first + sn.ncols; ++k) piece.rows.push_back(k);
        piece.rows.insert(piece.rows.end(), sn.rows.begin(), sn.rows.end());
        out.push_back(piece);
        nf += c;
        rem -= c;
      }
    }
    for (size_t s = 0; s < out.size(); ++s)
      for (int k = out[s].first; k < out[s].first + out[s].ncols; ++k) col_sn[k] = (int)s;
    for (size_t s = 0; s < out.size(); ++s) {
      int last = out[s].first + out[s].ncols - 1;
      out[s].parent = parent[last] >= 0 ? col_sn[parent[last]] : -1;
    }
    sns.swap(out);
  }
  const int NS = (int)sns.size();
  S.S = NS;
  S.col_sn = col_sn;
  S.sn_first.resize(NS);
  S.sn_ncols.resize(NS);
  S.sn_parent.resize(NS);
  S.sn_m.resize(NS);
  S.sn_ld.resize(NS);
  S.sn_w.resize(NS);
  S.sn_off.resize(NS);
  S.sn_rows.resize(NS);
  S.sn_level.assign(NS, 0);
  S.storage = 0;
  for (int s = 0; s < NS; ++s) {
    S.sn_first[s] = sns[s].first;
    S.sn_ncols[s] = sns[s].ncols;
    S.sn_parent[s] = sns[s].parent;
    S.sn_rows[s] = sns[s].rows;
    S.sn_w[s] = D * sns[s].ncols;
    S.sn_m[s] = D * (sns[s].ncols + (int)sns[s].rows.size());
    // odd leading dimension: lanes stepping along a panel row (stride ld doubles) then hit
    // distinct shared-memory banks
    S.sn_ld[s] = S.sn_m[s] | 1;
    S.storage += (int64_t)S.sn_ld[s] * S.sn_w[s];
    S.max_sn_cols_sc = std::max(S.max_sn_cols_sc, S.sn_w[s]);
    S.max_panel_rows = std::max(S.max_panel_rows, S.sn_m[s]);
  }
  if (S.storage > (int64_t)0x7fffffff) {
    *code = 8;
    err << "dnls_graph_create: factor storage " << S.storage << " doubles exceeds the int32 index range";
    return err.str();
  }
  for (int s = 0; s < NS; ++s)   // children have smaller indices (postorder)
    if (S.sn_parent[s] >= 0) S.sn_level[S.sn_parent[s]] = std::max(S.sn_level[S.sn_parent[s]], S.sn_level[s] + 1);
  S.num_levels = 0;
  for (int s = 0; s < NS; ++s) S.num_levels = std::max(S.num_levels, S.sn_level[s] + 1);
  S.level_ptr.assign(S.num_levels + 1, 0);
  for (int s = 0; s < NS; ++s) S.level_ptr[S.sn_level[s] + 1]++;
  for (int l = 0; l < S.num_levels; ++l) S.level_ptr[l + 1] += S.level_ptr[l];
  S.level_sn.assign(NS, 0);
  {
    VI fill(S.level_ptr.begin(), S.level_ptr.end() - 1);
    for (int s = 0; s < NS; ++s) S.level_sn[fill[S.sn_level[s]]++] = s;
  }
  // panel storage in LEVEL order: every level is one contiguous range [level_off[l], level_off[l+1])
  // (panels padded to 16 bytes).  Shared-memory plan: the top levels
  // [res_lo, storage) stay RESIDENT in shared memory for the whole solve; each lower level is
  // staged through a buffer of stage_cap doubles (prefix [level_off[l], level_stage_hi[l]) of
  // whole panels; panels beyond it are processed in global memory).
  {
    int64_t o = 0;
    S.level_off.assign(S.num_levels + 1, 0);
    for (int l = 0; l < S.num_levels; ++l) {
      S.level_off[l] = (int32_t)o;
      for (int i = S.level_ptr[l]; i < S.level_ptr[l + 1]; ++i) {
        int sn = S.level_sn[i];
        S.sn_off[sn] = o;
        o += ((int64_t)S.sn_ld[sn] * S.sn_w[sn] + 1) & ~int64_t(1);
      }
    }
    S.level_off[S.num_levels] = (int32_t)o;
    S.storage = o;
    const int64_t cap = opt.smem_cap_doubles;
    auto lsize = [&](int l) { return (int64_t)S.level_off[l + 1] - S.level_off[l]; };
    // most resident levels r.. such that resident + the largest lower level fits; else give the
    // resident part at most half the budget and stage partial prefixes
    int r = S.num_levels;
    for (int c = S.num_levels; c >= 0; --c) {
      int64_t res = o - (c < S.num_levels ? S.level_off[c] : o);
      int64_t lower = 0;
      for (int l = 0; l < c; ++l) lower = std::max(lower, lsize(l));
      if (res + lower <= cap) r = c;
      else break;
    }
    if (r == S.num_levels && S.num_levels > 0) {
      // lower levels cannot be staged whole: keep the largest resident suffix that leaves a
      // third of the budget for (partial) staging
      for (int c = S.num_levels - 1; c >= 0; --c) {
        if (o - S.level_off[c] <= cap - cap / 3) r = c;
        else break;
      }
    }
    S.res_lo = r < S.num_levels ? S.level_off[r] : (int32_t)o;
    S.res_n = o - S.res_lo;
    S.stage_cap = cap - S.res_n;
    S.level_stage_hi.assign(S.num_levels, 0);
    S.max_level_stage = 0;
    for (int l = 0; l < S.num_levels; ++l) {
      const int64_t lo = S.level_off[l];
      int64_t shi = lo;
      if (lo < S.res_lo) {
        for (int i = S.level_ptr[l]; i < S.level_ptr[l + 1]; ++i) {
          int sn = S.level_sn[i];
          int64_t end = S.sn_off[sn] + (((int64_t)S.sn_ld[sn] * S.sn_w[sn] + 1) & ~int64_t(1));
          if (S.sn_off[sn] == shi && end - lo <= S.stage_cap) shi = end;
          else break;
        }
      }
      S.level_stage_hi[l] = (int32_t)shi;
      S.max_level_stage = std::max<int64_t>(S.max_level_stage, shi - lo);
    }
  }

  // row position of pose p inside panel s (scalar), -1 if absent
  auto rowpos = [&](int s, int p) -> int {
    int f = S.sn_first[s], n = S.sn_ncols[s];
    if (p >= f && p < f + n) return D * (p - f);
    const VI& r = S.sn_rows[s];
    auto it = std::lower_bound(r.begin(), r.end(), p);
    if (it == r.end() || *it != p) return -1;
    return D * (n + (int)(it - r.begin()));
  };

  // ---- 5a. update tasks (gather form), grouped by target level
  {
    // key: (target sn, q, p) -> list of (src)
    std::map<std::tuple<int, int, int>, VI> tasks;
    for (int src = 0; src < NS; ++src) {
      const VI& R = S.sn_rows[src];
      size_t i0 = 0;
      while (i0 < R.size()) {
        int t = col_sn[R[i0]];
        size_t i1 = i0;
        int tend = S.sn_first[t] + S.sn_ncols[t];
        while (i1 < R.size() && R[i1] < tend) ++i1;   // K = R[i0..i1)
        for (size_t iq = i0; iq < i1; ++iq)
          for (size_t ip = iq; ip < R.size(); ++ip)
            tasks[std::make_tuple(t, R[iq], R[ip])].push_back(src);
        i0 = i1;
      }
    }
    // order tasks by (level of t, t, q, p)
    std::vector<std::tuple<int, int, int, int>> keys;
    for (auto& kv : tasks)
      keys.push_back(std::make_tuple(S.sn_level[std::get<0>(kv.first)], std::get<0>(kv.first),
                                     std::get<1>(kv.first), std::get<2>(kv.first)));
    std::sort(keys.begin(), keys.end());
    S.ut_level_ptr.assign(S.num_levels + 1, 0);
    S.ut_cptr.push_back(0);
    for (auto& k : keys) {
      int lv = std::get<0>(k), t = std::get<1>(k), q = std::get<2>(k), p = std::get<3>(k);
      S.ut_level_ptr[lv + 1]++;
      int off = (int)S.sn_off[t] + D * (q - S.sn_first[t]) * S.sn_ld[t] + rowpos(t, p);
      S.ut_off.push_back(off);
      S.ut_ld.push_back(S.sn_ld[t]);
      for (int src : tasks[std::make_tuple(t, q, p)]) {
        S.uc_a.push_back((int)S.sn_off[src] + rowpos(src, p));
        S.uc_b.push_back((int)S.sn_off[src] + rowpos(src, q));
        S.uc_ld.push_back(S.sn_ld[src]);
        S.uc_w.push_back(S.sn_w[src]);
      }
      S.ut_cptr.push_back((int)S.uc_a.size());
    }
    for (int l = 0; l < S.num_levels; ++l) S.ut_level_ptr[l + 1] += S.ut_level_ptr[l];
  }
  // ---- 5b. solve lists
  {
    std::vector<std::vector<int>> srcs(N);
    for (int src = 0; src < NS; ++src)
      for (int p : S.sn_rows[src]) srcs[p].push_back(src);
    S.fc_ptr.assign(1, 0);
    for (int p = 0; p < N; ++p) {
      for (int src : srcs[p]) {
        S.fc_off.push_back((int)S.sn_off[src] + rowpos(src, p));
        S.fc_ld.push_back(S.sn_ld[src]);
        S.fc_w.push_back(S.sn_w[src]);
        S.fc_x.push_back(D * S.sn_first[src]);
      }
      S.fc_ptr.push_back((int)S.fc_off.size());
    }
    S.snr_ptr.assign(1, 0);
    for (int s = 0; s < NS; ++s) {
      for (int p : S.sn_rows[s]) S.snr.push_back(p);
      S.snr_ptr.push_back((int)S.snr.size());
    }
    // per-supernode update-task ranges (packet construction places a panel after its tasks)
    {
      // recover the target supernode of each task from its storage offset
      std::vector<int> tsn(S.ut_off.size());
      std::vector<std::pair<int64_t, int>> starts;
      for (int sn = 0; sn < NS; ++sn) starts.push_back(std::make_pair(S.sn_off[sn], sn));
      std::sort(starts.begin(), starts.end());
      for (size_t t = 0; t < S.ut_off.size(); ++t) {
        auto it = std::upper_bound(starts.begin(), starts.end(), std::make_pair((int64_t)S.ut_off[t], NS));
        tsn[t] = (--it)->second;
      }
      std::vector<int> first(NS, -1), last(NS, -1);
      for (size_t t = 0; t < tsn.size(); ++t) {
        if (first[tsn[t]] < 0) first[tsn[t]] = (int)t;
        last[tsn[t]] = (int)t + 1;
      }
      S.ut_sn_ptr.assign(2 * NS, 0);   // [begin, end) per supernode
      for (int sn = 0; sn < NS; ++sn) {
        S.ut_sn_ptr[2 * sn] = first[sn] < 0 ? 0 : first[sn];
        S.ut_sn_ptr[2 * sn + 1] = first[sn] < 0 ? 0 : last[sn];
      }
    }
  }
  // ---- 5b'. descriptor packets (prefetched into shared memory one packet ahead).  A level is
  // emitted as one or more size-bounded packets ("chunks"); a panel is placed after all its
  // update tasks and its forward-substitution rows, so chunks of a level run in order.
  //   int4 h0 = (ntasks, ncons, nrows, nfcons), h1 = (nsn, nsnr, nul, nfl),
  //   int4 h2 = (max column blocks, level, first chunk of level, last chunk of level),
  //   task4[ntasks] = (target off, ld, c0, c1)   c0/c1 index con4 of this packet
  //   con4[ncons]   = (src row-p off, src row-q off, ld, width)
  //   row4[nrows]   = (pose row p, fc0, fc1, 0)   fc0/fc1 index fcon4 of this packet
  //   fcon4[nfcons] = (src row off, ld, width, y off)
  //   sna4[nsn] = (off, m, ld, w), snb4[nsn] = (first, snr0, snr1, 0), snr[nsnr],
  //   ulane[nul], flane[nfl] (lane maps), snm[nsn+1], snw[nsn+1] (prefix sums), pad to 4
  {
    S.pk.clear();
    S.pk_off.assign(1, 0);
    S.pk_max = 0;
    const int budget = opt.packet_ints;
    auto lane_map = [&](const std::vector<int>& work) {
      // every item gets a power-of-two group of G lanes sized to its work, packed into one round
      // of cta_threads lanes when possible (groups placed in decreasing size stay aligned);
      // entry = item << 8 | log2(G) << 5 | sub
      std::vector<int> order(work.size());
      for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
      std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return work[x] > work[y]; });
      auto gsize = [&](int k, int kc) {
        int need = (k + kc - 1) / kc, G = 1;
        while (G < need && G < 32) G *= 2;
        return G;
      };
      int kc = 1;
      for (; kc < (1 << 20); kc *= 2) {
        int64_t tot = 0;
        for (int i : order) tot += gsize(work[i], kc);
        if (tot <= opt.cta_threads) break;
      }
      std::vector<int> lanes;
      for (int i : order) {
        const int G = gsize(work[i], kc);
        int lg = 0;
        while ((1 << lg) < G) ++lg;
        for (int sub = 0; sub < G; ++sub) lanes.push_back((i << 8) | (lg << 5) | sub);
      }
      return lanes;
    };
    struct Chunk {
      std::vector<int> tasks, rows, sns;
      int ncons = 0, nfcons = 0, nsnr = 0;
    };
    auto chunk_ints = [&](const Chunk& c) {
      // header + descriptors + lane maps (upper bound: one lane per work unit, capped at 32) + prefixes
      int64_t n = 16 + 4LL * ((int64_t)c.tasks.size() + c.ncons + (int64_t)c.rows.size() + c.nfcons +
                              2LL * (int64_t)c.sns.size()) + c.nsnr;
      const int64_t ui = (int64_t)D * c.tasks.size(), fi = (int64_t)D * c.rows.size();
      const int64_t u3 = (int64_t)(D / UPD_ROWS) * c.tasks.size();
      n += std::max<int64_t>(ui, std::min<int64_t>(opt.cta_threads, 32 * ui));
      n += std::max<int64_t>(u3, std::min<int64_t>(opt.cta_threads, 32 * u3));
      n += std::max<int64_t>(fi, std::min<int64_t>(opt.cta_threads, 32 * fi));
      n += 2LL * (c.sns.size() + 1) + 4;
      return n;
    };
    auto emit = [&](const Chunk& c, int lv, bool first, bool last) {
      const int base = (int)S.pk.size();
      auto push4 = [&](int x0, int x1, int x2, int x3) {
        S.pk.push_back(x0); S.pk.push_back(x1); S.pk.push_back(x2); S.pk.push_back(x3);
      };
      // two lane maps of the update items: one row of a target block per item (the clustered kernels: more
      // items to spread over the cluster) and UPD_ROWS rows per item (the one-CTA kernel: the rows share the
      // loads of the target's column block)
      std::vector<int> uwork, uwork3, fwork;
      for (int t : c.tasks) {
        for (int a = 0; a < D; ++a) uwork.push_back(S.ut_cptr[t + 1] - S.ut_cptr[t]);
        for (int a = 0; a < D / UPD_ROWS; ++a) uwork3.push_back(S.ut_cptr[t + 1] - S.ut_cptr[t]);
      }
      for (int p : c.rows)
        for (int a = 0; a < D; ++a) fwork.push_back(S.fc_ptr[p + 1] - S.fc_ptr[p]);
      const std::vector<int> ulanes = lane_map(uwork), ulanes3 = lane_map(uwork3), flanes = lane_map(fwork);
      int maxb = 0;
      for (int sn : c.sns) maxb = std::max(maxb, S.sn_ncols[sn]);
      push4((int)c.tasks.size(), c.ncons, (int)c.rows.size(), c.nfcons);
      push4((int)c.sns.size(), c.nsnr, (int)ulanes.size(), (int)flanes.size());
      push4(maxb, lv, first ? 1 : 0, last ? 1 : 0);
      push4((int)ulanes3.size(), 0, 0, 0);
      int ccur = 0;
      for (int t : c.tasks) {
        const int n = S.ut_cptr[t + 1] - S.ut_cptr[t];
        push4(S.ut_off[t], S.ut_ld[t], ccur, ccur + n);
        ccur += n;
      }
      for (int t : c.tasks)
        for (int cc = S.ut_cptr[t]; cc < S.ut_cptr[t + 1]; ++cc) push4(S.uc_a[cc], S.uc_b[cc], S.uc_ld[cc], S.uc_w[cc]);
      int fcur = 0;
      for (int p : c.rows) {
        const int n = S.fc_ptr[p + 1] - S.fc_ptr[p];
        push4(p, fcur, fcur + n, 0);
        fcur += n;
      }
      for (int p : c.rows)
        for (int cc = S.fc_ptr[p]; cc < S.fc_ptr[p + 1]; ++cc) push4(S.fc_off[cc], S.fc_ld[cc], S.fc_w[cc], S.fc_x[cc]);
      for (int sn : c.sns) push4((int)S.sn_off[sn], S.sn_m[sn], S.sn_ld[sn], S.sn_w[sn]);
      int rcur = 0;
      for (int sn : c.sns) {
        const int n = (int)S.sn_rows[sn].size();
        push4(S.sn_first[sn], rcur, rcur + n, 0);
        rcur += n;
      }
      for (int sn : c.sns)
        for (int p : S.sn_rows[sn]) S.pk.push_back(p);
      for (int v : ulanes) S.pk.push_back(v);
      for (int v : flanes) S.pk.push_back(v);
      for (int v : ulanes3) S.pk.push_back(v);
      int pm = 0, pw = 0;
      S.pk.push_back(0);
      for (int sn : c.sns) S.pk.push_back(pm += S.sn_m[sn]);
      S.pk.push_back(0);
      for (int sn : c.sns) S.pk.push_back(pw += S.sn_w[sn]);
      while (S.pk.size() % 4) S.pk.push_back(0);
      S.pk_max = std::max(S.pk_max, (int)S.pk.size() - base);
      S.pk_off.push_back((int)S.pk.size());
      S.pk_level.push_back(lv);
    };
    for (int l = 0; l < S.num_levels; ++l) {
      std::vector<Chunk> chunks(1);
      auto fits = [&](const Chunk& c) { return chunk_ints(c) <= budget; };
      for (int i = S.level_ptr[l]; i < S.level_ptr[l + 1]; ++i) {
        const int sn = S.level_sn[i];
        for (int t = S.ut_sn_ptr[2 * sn]; t < S.ut_sn_ptr[2 * sn + 1]; ++t) {
          Chunk& c = chunks.back();
          c.tasks.push_back(t);
          c.ncons += S.ut_cptr[t + 1] - S.ut_cptr[t];
          if (!fits(c) && c.tasks.size() + c.rows.size() + c.sns.size() > 1) {
            c.tasks.pop_back();
            c.ncons -= S.ut_cptr[t + 1] - S.ut_cptr[t];
            chunks.emplace_back();
            chunks.back().tasks.push_back(t);
            chunks.back().ncons = S.ut_cptr[t + 1] - S.ut_cptr[t];
          }
        }
        for (int p = S.sn_first[sn]; p < S.sn_first[sn] + S.sn_ncols[sn]; ++p) {
          Chunk& c = chunks.back();
          c.rows.push_back(p);
          c.nfcons += S.fc_ptr[p + 1] - S.fc_ptr[p];
          if (!fits(c) && c.tasks.size() + c.rows.size() + c.sns.size() > 1) {
            c.rows.pop_back();
            c.nfcons -= S.fc_ptr[p + 1] - S.fc_ptr[p];
            chunks.emplace_back();
            chunks.back().rows.push_back(p);
            chunks.back().nfcons = S.fc_ptr[p + 1] - S.fc_ptr[p];
          }
        }
        {
          Chunk& c = chunks.back();
          c.sns.push_back(sn);
          c.nsnr += (int)S.sn_rows[sn].size();
          if (!fits(c) && c.tasks.size() + c.rows.size() + c.sns.size() > 1) {
            c.sns.pop_back();
            c.nsnr -= (int)S.sn_rows[sn].size();
            chunks.emplace_back();
            chunks.back().sns.push_back(sn);
            chunks.back().nsnr = (int)S.sn_rows[sn].size();
          }
        }
      }
      for (size_t k = 0; k < chunks.size(); ++k) emit(chunks[k], l, k == 0, k + 1 == chunks.size());
    }
    S.npk = (int)S.pk_level.size();
  }
  // ---- 5c. assembly lists
  {
    std::map<std::pair<int, int>, VI> pair_edges;   // original (min, max) -> edges
    std::vector<VI> inc(N);                          // incident edges per original var
    for (int e = 0; e < E; ++e) {
      int i = edges[2 * e], j = edges[2 * e + 1];
      pair_edges[std::make_pair(std::min(i, j), std::max(i, j))].push_back(e);
      inc[i].push_back(e);
      inc[j].push_back(e);
    }
    std::vector<VI> pri(N);
    for (int k = 0; k < P; ++k) pri[priors[k]].push_back(k);
    S.blk_cptr.assign(1, 0);
    S.dup_blk.clear();
    for (int s = 0; s < NS; ++s) {
      int f = S.sn_first[s], n = S.sn_ncols[s];
      VI rows;
      for (int k = 0; k < n; ++k) rows.push_back(f + k);
      for (int p : S.sn_rows[s]) rows.push_back(p);
      for (int ql = 0; ql < n; ++ql) {
        int q = f + ql;
        for (size_t ri = 0; ri < rows.size(); ++ri) {
          int p = rows[ri];
          S.blk_off.push_back((int)S.sn_off[s] + D * ql * S.sn_ld[s] + D * (int)ri);
          S.blk_ld.push_back(S.sn_ld[s]);
          int kind = 0;
          if (p == q) {
            kind = 1;
            int o = S.perm[p];
            for (int e : inc[o]) {
              int side = (edges[2 * e] == o) ? 0 : 1;
              S.blk_con.push_back(e * 4 + side * 2 + side);
            }
            for (int k : pri[o]) S.blk_con.push_back((E + k) * 4);
          } else if (p > q) {
            int op = S.perm[p], oq = S.perm[q];
            auto it = pair_edges.find(std::make_pair(std::min(op, oq), std::max(op, oq)));
            if (it != pair_edges.end()) {
              kind = 2;
              for (int e : it->second) {
                int rs = (edges[2 * e] == op) ? 0 : 1;
                S.blk_con.push_back(e * 4 + rs * 2 + (1 - rs));
              }
            }
          }
          S.blk_kind.push_back(kind);
          S.blk_cptr.push_back((int)S.blk_con.size());
          if (kind == 2 && S.blk_cptr.back() - S.blk_cptr[S.blk_cptr.size() - 2] > 1)
            S.dup_blk.push_back((int)S.blk_kind.size() - 1);
        }
      }
    }
    S.bc_ptr.assign(1, 0);
    for (int p = 0; p < N; ++p) {
      int o = S.perm[p];
      for (int e : inc[o]) S.bc.push_back(e * 2 + ((edges[2 * e] == o) ? 0 : 1));
      for (int k : pri[o]) S.bc.push_back((E + k) * 2);
      S.bc_ptr.push_back((int)S.bc.size());
    }
  }
  // ---- 5d. per-slot descriptors of the single-writer assembly: the storage
  // offsets / leading dims of the slot's H blocks and its permuted poses
  {
    const int slots = E + P;
    auto diag_off = [&](int p) {
      const int sn = col_sn[p];
      return (int)S.sn_off[sn] + D * (p - S.sn_first[sn]) * (S.sn_ld[sn] + 1);
    };
    std::map<std::pair<int, int>, int> pair_count;   // edges per (min, max) permuted pose pair
    for (int e = 0; e < E; ++e) {
      const int pi = S.iperm[edges[2 * e]], pj = S.iperm[edges[2 * e + 1]];
      pair_count[std::make_pair(std::min(pi, pj), std::max(pi, pj))]++;
    }
    S.slot_desc.assign(12 * (size_t)slots, 0);
    for (int sl = 0; sl < slots; ++sl) {
      int32_t* d = &S.slot_desc[12 * (size_t)sl];
      if (sl < E) {
        const int pi = S.iperm[edges[2 * sl]], pj = S.iperm[edges[2 * sl + 1]];
        const int P_ = std::max(pi, pj), Q = std::min(pi, pj);
        const int t = col_sn[Q];
        d[0] = diag_off(pi);
        d[1] = diag_off(pj);
        d[2] = (int)S.sn_off[t] + D * (Q - S.sn_first[t]) * S.sn_ld[t] + rowpos(t, P_);
        d[3] = (P_ == pj) ? 1 : 0;   // off-diagonal block = J_j^T J_i (row pose is endpoint j)
        d[4] = S.sn_ld[col_sn[pi]];
        d[5] = S.sn_ld[col_sn[pj]];
        d[6] = S.sn_ld[t];
        d[8] = pi;
        d[9] = pj;
        d[10] = pair_count[std::make_pair(Q, P_)] == 1 ? 1 : 0;   // only edge between its poses
      } else {
        const int pp = S.iperm[priors[sl - E]];
        d[0] = diag_off(pp);
        d[1] = -1;
        d[2] = -1;
        d[4] = S.sn_ld[col_sn[pp]];
        d[8] = pp;
        d[9] = -1;
      }
    }
  }
  return std::string();
}

}  // namespace dnls
