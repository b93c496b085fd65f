// oracle.cpp — the CPU ORACLE of the calling-context-tree (CCT) aggregation path.
//
// TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load or call this library. It shares no code
// with the CUDA path (paper_2411_02797_b200/csrc, include/dc.h): no headers, no helpers,
// no tables. It is deliberately plain and slow: std::map tries, one record at a time,
// literal root-ward propagation, std::sort for the views.
//
// What it computes, step by step in the paper's order (PAPER.md = /root/reference/PAPER.md):
//  * or_intern      — frame identity + unification (§4.2 "Calling Context Tree",
//                     PAPER.md:344-346): C/C++, GPU API, kernel frames are equal iff same
//                     library (module) + PC; Python frames iff same file + line; framework
//                     frames iff same operator name. The caller encodes each identity as a
//                     raw key (kind, str_id, addr); equal identity <=> equal key. Canonical
//                     frame id = rank of the key among the distinct keys in lexicographic
//                     order (reading R2).
//  * or_insert      — CCT construction by inserting call paths and collapsing frames that
//                     refer to the same location; metrics kept per node as
//                     sum / minimum / average / standard deviation via the
//                     exact integers count, sum, min, sum of squares; "once a metric has been
//                     updated at the bottom of a call path, it is propagated to the root node
//                     ... updating the metric along the entire call path":
//                     every node on the path gets the record's value in its inclusive
//                     aggregate, literally, one node at a time. The bottom node also gets it
//                     in its exclusive aggregate. GPU activities reach their call path through
//                     the correlation id: here record r *is* the joined
//                     launch record (the join is the identity).
//  * or_pc          — instruction samples extend the call path by the PC of each sampled
//                     instruction; stall reasons per instruction
//                     (PAPER.md:414-416). Launch l's call path is record l's.
//  * or_finalize    — canonical node ids: breadth-first from the root, children in
//                     ascending frame id (reading R2); PC nodes numbered after all
//                     path nodes in (context id, pc) order (reading R15).
//  * or_topk        — analysis ① hotspot identification `n.time / total_time >
//                     hotspot_threshold` with total = root; bottom-up
//                     aggregation of the same frame across call paths; stall
//                     top-k of analysis ④.
//  * or_rule_flags  — example analyses ② "Small GPU kernels" and ⑤ "CPU
//                     time abnormality" over `bfs(call_tree.nodes)`, with
//                     SPEC.md's readings (launch count of the frame's kernels, max(gpu, 1)
//                     guard, absolute floor, children of a flagged frame not re-flagged;
//                     DESIGN.md reading R22). Literal BFS over the canonical tree.
//                     ③ "Backward abnormality" per operator node, with
//                     SPEC.md's forward-time epsilon guard (reading R25).
//  * or_stall_issues — analysis ④: for n in hotspots, its children c with
//                     c.stalls > stall_threshold, topk(stall reasons) (SPEC.md analyze_stalls:
//                     the threshold is a fraction of the kernel's samples; reading R23).
//  * or_derived     — average and (population) standard deviation (reading
//                     R7): mean = sum/count, std = sqrt(count*sumsq - sum^2)/count with the
//                     radicand formed exactly in a hand-rolled 256-bit integer and rounded
//                     once to binary64.
//
// Parity pins for every function live in tests/test_oracle_*.py (brute force, SPEC/paper
// worked examples, closed forms, invariants). See DESIGN.md "Oracle and pins".
#include <stdint.h>
#include <string.h>
#include <math.h>
#include <algorithm>
#include <map>
#include <tuple>
#include <vector>

typedef unsigned __int128 u128;

struct OrKey { uint32_t kind, str_id; uint64_t addr; };
struct OrSample { uint32_t launch, pc_off; uint16_t stall, flags; uint32_t count; };
struct OrTopk { uint32_t id, pad; uint64_t value; double fraction; };

struct Agg {  // exact aggregate of a multiset of u64 values
  uint64_t sum = 0, min = UINT64_MAX;
  u128 sq = 0;
  void add(uint64_t x) {
    sum += x;
    if (x < min) min = x;
    sq += (u128)x * x;
  }
};

struct TNode {
  uint32_t parent, frame, depth;
  std::map<uint32_t, uint32_t> kids;  // frame id -> node (trie children, ascending frame id)
  uint64_t xcnt = 0, icnt = 0;
  std::vector<Agg> x, i;              // exclusive / inclusive per metric
  uint64_t xsamples = 0, isamples = 0;
  std::vector<uint64_t> xstall, istall;
};

struct OrCct {
  uint32_t M, S;
  std::vector<TNode> t;                // trie in creation order; t[0] = root
  std::vector<uint32_t> leaf;          // record -> trie node
  std::map<std::pair<uint32_t, uint32_t>, std::map<uint16_t, uint64_t>> bins;  // (trie node, pc) -> stall -> count
  uint64_t empty_paths = 0, bad_launch = 0, bad_stall = 0, zero_count = 0;
  // canonical view (after or_finalize)
  bool final_ = false;
  std::vector<uint32_t> canon;         // trie node -> canonical id
  std::vector<uint32_t> order;         // canonical id -> trie node
  std::vector<std::pair<uint32_t, uint32_t>> pcs;  // canonical pc nodes (ctx id, pc)
  std::vector<std::tuple<uint32_t, uint16_t, uint64_t>> cbins;

  uint32_t new_node(uint32_t parent, uint32_t frame, uint32_t depth) {
    TNode n;
    n.parent = parent; n.frame = frame; n.depth = depth;
    n.x.resize(M); n.i.resize(M);
    n.xstall.assign(S, 0); n.istall.assign(S, 0);
    t.push_back(std::move(n));
    return (uint32_t)(t.size() - 1);
  }
};

extern "C" {

// ---------------------------------------------------------------- interning
int or_intern(const OrKey* keys, uint64_t n, uint32_t* out_ids, OrKey* out_dict, uint64_t* out_D) {
  std::map<std::tuple<uint32_t, uint32_t, uint64_t>, uint32_t> dict;
  for (uint64_t j = 0; j < n; ++j) dict[std::make_tuple(keys[j].kind, keys[j].str_id, keys[j].addr)] = 0;
  uint32_t rank = 0;
  for (auto& kv : dict) {  // in-order traversal = lexicographic order
    if (out_dict) {
      out_dict[rank].kind = std::get<0>(kv.first);
      out_dict[rank].str_id = std::get<1>(kv.first);
      out_dict[rank].addr = std::get<2>(kv.first);
    }
    kv.second = rank++;
  }
  for (uint64_t j = 0; j < n; ++j) out_ids[j] = dict[std::make_tuple(keys[j].kind, keys[j].str_id, keys[j].addr)];
  *out_D = dict.size();
  return 0;
}

// ---------------------------------------------------------------- CCT
OrCct* or_cct_new(uint32_t M, uint32_t S) {
  OrCct* c = new OrCct();
  c->M = M; c->S = S;
  c->new_node(0xFFFFFFFFu, 0xFFFFFFFFu, 0);  // root (reading R1)
  return c;
}
void or_cct_free(OrCct* c) { delete c; }

// Insert records in trace order. X is column-major [M][ld].
int or_insert(OrCct* c, const uint64_t* offsets, const uint32_t* frames, uint64_t R, const uint64_t* X, uint64_t ld) {
  if (c->final_) return 1;
  for (uint64_t r = 0; r < R; ++r) {
    uint32_t cur = 0;
    // propagation to the root = update every node of the path
    c->t[cur].icnt += 1;
    for (uint32_t m = 0; m < c->M; ++m) c->t[cur].i[m].add(X[m * ld + r]);
    for (uint64_t j = offsets[r]; j < offsets[r + 1]; ++j) {
      uint32_t f = frames[j];
      auto it = c->t[cur].kids.find(f);
      uint32_t nxt;
      if (it == c->t[cur].kids.end()) {  // insert; equal frames collapse
        nxt = c->new_node(cur, f, c->t[cur].depth + 1);
        c->t[cur].kids[f] = nxt;
      } else {
        nxt = it->second;
      }
      cur = nxt;
      c->t[cur].icnt += 1;
      for (uint32_t m = 0; m < c->M; ++m) c->t[cur].i[m].add(X[m * ld + r]);
    }
    if (offsets[r] == offsets[r + 1]) c->empty_paths += 1;  // reading R10: root's exclusive
    c->t[cur].xcnt += 1;
    for (uint32_t m = 0; m < c->M; ++m) c->t[cur].x[m].add(X[m * ld + r]);
    c->leaf.push_back(cur);
  }
  return 0;
}

// Instruction samples: launch l -> call path of record l.
int or_pc(OrCct* c, const OrSample* s, uint64_t n, uint64_t n_launch) {
  if (c->final_ || n_launch > c->leaf.size()) return 1;
  for (uint64_t j = 0; j < n; ++j) {
    const OrSample& q = s[j];
    if (q.launch >= n_launch) { c->bad_launch++; continue; }   // reading R16
    if (q.stall >= c->S) { c->bad_stall++; continue; }
    if (q.count == 0) { c->zero_count++; continue; }
    uint32_t node = c->leaf[q.launch];
    c->bins[std::make_pair(node, q.pc_off)][q.stall] += q.count;
    c->t[node].xsamples += q.count;
    c->t[node].xstall[q.stall] += q.count;
    for (uint32_t a = node;; a = c->t[a].parent) {  // propagate to the root
      c->t[a].isamples += q.count;
      c->t[a].istall[q.stall] += q.count;
      if (a == 0) break;
    }
  }
  return 0;
}

// Canonical ids: BFS, children ascending by frame id (reading R2).
int or_finalize(OrCct* c) {
  if (c->final_) return 0;
  c->canon.assign(c->t.size(), 0);
  c->order.clear();
  c->order.push_back(0);
  for (size_t h = 0; h < c->order.size(); ++h)
    for (auto& kv : c->t[c->order[h]].kids) c->order.push_back(kv.second);
  for (size_t k = 0; k < c->order.size(); ++k) c->canon[c->order[k]] = (uint32_t)k;
  std::map<std::pair<uint32_t, uint32_t>, std::map<uint16_t, uint64_t>> cb;
  for (auto& kv : c->bins) cb[std::make_pair(c->canon[kv.first.first], kv.first.second)] = kv.second;
  uint32_t N = (uint32_t)c->order.size();
  for (auto& kv : cb) {
    uint32_t pcnode = N + (uint32_t)c->pcs.size();
    c->pcs.push_back(kv.first);
    for (auto& sv : kv.second) c->cbins.push_back(std::make_tuple(pcnode, sv.first, sv.second));
  }
  c->final_ = true;
  return 0;
}

void or_counts(const OrCct* c, uint64_t out[8]) {
  out[0] = c->t.size(); out[1] = c->pcs.size(); out[2] = c->cbins.size(); out[3] = c->leaf.size();
  uint32_t md = 0;
  for (auto& n : c->t) md = std::max(md, n.depth);
  out[4] = md; out[5] = 0; out[6] = 0; out[7] = 0;
}

void or_diag(const OrCct* c, uint64_t out[4]) {
  out[0] = c->empty_paths; out[1] = c->bad_launch; out[2] = c->bad_stall; out[3] = c->zero_count;
}

struct OrOut {
  uint32_t *parent, *frame; uint16_t* depth; uint32_t* leaf;
  uint64_t *xcnt, *icnt;
  uint64_t *xsum, *xmin, *xsq_lo, *xsq_hi, *isum, *imin, *isq_lo, *isq_hi;  // [M][N]
  uint64_t *xsamples, *isamples, *xstall, *istall;                          // [S][N]
  uint32_t *pc_ctx, *pc_off, *bin_pcnode; uint16_t* bin_stall; uint64_t* bin_count;
};

int or_get(const OrCct* c, const OrOut* o) {
  if (!c->final_) return 1;
  const uint64_t N = c->order.size();
  for (uint64_t k = 0; k < N; ++k) {
    const TNode& n = c->t[c->order[k]];
    if (o->parent) o->parent[k] = k == 0 ? 0xFFFFFFFFu : c->canon[n.parent];
    if (o->frame) o->frame[k] = n.frame;
    if (o->depth) o->depth[k] = (uint16_t)n.depth;
    if (o->xcnt) o->xcnt[k] = n.xcnt;
    if (o->icnt) o->icnt[k] = n.icnt;
    for (uint32_t m = 0; m < c->M; ++m) {
      if (o->xsum) o->xsum[m * N + k] = n.x[m].sum;
      if (o->xmin) o->xmin[m * N + k] = n.x[m].min;
      if (o->xsq_lo) o->xsq_lo[m * N + k] = (uint64_t)n.x[m].sq;
      if (o->xsq_hi) o->xsq_hi[m * N + k] = (uint64_t)(n.x[m].sq >> 64);
      if (o->isum) o->isum[m * N + k] = n.i[m].sum;
      if (o->imin) o->imin[m * N + k] = n.i[m].min;
      if (o->isq_lo) o->isq_lo[m * N + k] = (uint64_t)n.i[m].sq;
      if (o->isq_hi) o->isq_hi[m * N + k] = (uint64_t)(n.i[m].sq >> 64);
    }
    if (o->xsamples) o->xsamples[k] = n.xsamples;
    if (o->isamples) o->isamples[k] = n.isamples;
    for (uint32_t s = 0; s < c->S; ++s) {
      if (o->xstall) o->xstall[s * N + k] = n.xstall[s];
      if (o->istall) o->istall[s * N + k] = n.istall[s];
    }
  }
  if (o->leaf)
    for (size_t r = 0; r < c->leaf.size(); ++r) o->leaf[r] = c->canon[c->leaf[r]];
  for (size_t p = 0; p < c->pcs.size(); ++p) {
    if (o->pc_ctx) o->pc_ctx[p] = c->pcs[p].first;
    if (o->pc_off) o->pc_off[p] = c->pcs[p].second;
  }
  for (size_t b = 0; b < c->cbins.size(); ++b) {
    if (o->bin_pcnode) o->bin_pcnode[b] = std::get<0>(c->cbins[b]);
    if (o->bin_stall) o->bin_stall[b] = std::get<1>(c->cbins[b]);
    if (o->bin_count) o->bin_count[b] = std::get<2>(c->cbins[b]);
  }
  return 0;
}

// ---------------------------------------------------------------- views
enum { OR_VIEW_INCLUSIVE = 0, OR_VIEW_EXCLUSIVE = 1, OR_VIEW_BOTTOM_UP = 2, OR_VIEW_STALL = 3 };
static const uint32_t OR_METRIC_SAMPLES = 0xFFFFFFFFu;

static bool kind_ok(const uint8_t* fk, uint32_t nf, uint32_t frame, uint32_t mask) {
  if (!fk) return true;
  if (frame >= nf) return false;
  return fk[frame] < 32 && ((mask >> fk[frame]) & 1u);
}

int or_topk(const OrCct* c, int view, uint32_t metric, uint32_t kind_mask, const uint8_t* frame_kind,
            uint32_t n_frames, double threshold, uint32_t k, uint32_t stall_node, OrTopk* out, uint32_t* n_out) {
  *n_out = 0;
  if (!c->final_) return 1;
  if (metric != OR_METRIC_SAMPLES && metric >= c->M) return 2;
  std::vector<std::pair<uint64_t, uint32_t>> cand;  // (value, id)
  uint64_t total;
  auto val = [&](const TNode& n, bool incl) -> uint64_t {
    if (metric == OR_METRIC_SAMPLES) return incl ? n.isamples : n.xsamples;
    return incl ? n.i[metric].sum : n.x[metric].sum;
  };
  const TNode& root = c->t[0];
  if (view == OR_VIEW_INCLUSIVE || view == OR_VIEW_EXCLUSIVE) {
    total = val(root, true);
    for (size_t id = 1; id < c->order.size(); ++id) {
      const TNode& n = c->t[c->order[id]];
      if (kind_ok(frame_kind, n_frames, n.frame, kind_mask)) cand.push_back({val(n, view == OR_VIEW_INCLUSIVE), (uint32_t)id});
    }
  } else if (view == OR_VIEW_BOTTOM_UP) {
    total = val(root, true);
    std::map<uint32_t, uint64_t> by_frame;  // same frame across different call paths
    for (size_t id = 1; id < c->order.size(); ++id) {
      const TNode& n = c->t[c->order[id]];
      if (kind_ok(frame_kind, n_frames, n.frame, kind_mask)) by_frame[n.frame] += val(n, false);
    }
    for (auto& kv : by_frame) cand.push_back({kv.second, kv.first});
  } else if (view == OR_VIEW_STALL) {
    if (stall_node >= c->order.size()) return 2;
    const TNode& n = c->t[c->order[stall_node]];
    total = n.isamples;
    for (uint32_t s = 0; s < c->S; ++s) cand.push_back({n.istall[s], s});
  } else {
    return 2;
  }
  if (total == 0) return 0;  // reading R12
  std::vector<OrTopk> keep;
  for (auto& cv : cand) {
    double frac = (double)cv.first / (double)total;
    if (frac > threshold) keep.push_back(OrTopk{cv.second, 0, cv.first, frac});  // strict >
  }
  std::sort(keep.begin(), keep.end(), [](const OrTopk& a, const OrTopk& b) {
    if (a.value != b.value) return a.value > b.value;
    return a.id < b.id;
  });
  uint32_t m = (uint32_t)std::min<size_t>(k, keep.size());
  for (uint32_t j = 0; j < m; ++j) out[j] = keep[j];
  *n_out = m;
  return 0;
}

// ---------------------------------------------------------------- analyzer rules
enum { OR_RULE_SMALL_KERNELS = 2, OR_RULE_BWD_FWD = 3, OR_RULE_CPU_LATENCY = 5 };

int or_rule_flags(const OrCct* c, int rule, uint32_t metric_a, uint32_t metric_b, uint32_t kind_mask, const uint8_t* frame_kind,
                  uint32_t n_frames, double threshold, uint64_t floor_v, uint32_t* out, uint32_t cap, uint32_t* n_out) {
  *n_out = 0;
  if (!c->final_) return 1;
  if (metric_a >= c->M || (rule != OR_RULE_SMALL_KERNELS && metric_b >= c->M)) return 2;
  if (rule != OR_RULE_SMALL_KERNELS && rule != OR_RULE_CPU_LATENCY && rule != OR_RULE_BWD_FWD) return 2;
  const size_t N = c->order.size();
  // launches(n): kernel launches in n's subtree = xcnt of every kernel-kind node, propagated
  // to each ancestor one node at a time (the root is not a frame and is not considered)
  std::vector<uint64_t> launches(N, 0);
  for (size_t id = 1; id < N; ++id) {
    const TNode& n = c->t[c->order[id]];
    if (!kind_ok(frame_kind, n_frames, n.frame, kind_mask) || n.xcnt == 0) continue;
    for (uint32_t tn = c->order[id]; tn != 0; tn = c->t[tn].parent) launches[c->canon[tn]] += n.xcnt;
  }
  auto qualifies = [&](size_t id) -> bool {
    const TNode& n = c->t[c->order[id]];
    if (rule == OR_RULE_SMALL_KERNELS)  // n.gpu_time / n.count < gpu_threshold
      return launches[id] > 0 && (double)n.i[metric_a].sum / (double)launches[id] < threshold;
    if (rule == OR_RULE_BWD_FWD) {  // for n in call_tree.operators: n.backward.time / n.forward.time > 2
      const uint64_t bwd = n.i[metric_a].sum, fwd = n.i[metric_b].sum;
      return kind_ok(frame_kind, n_frames, n.frame, kind_mask) && fwd > 0 && fwd >= floor_v &&
             (double)bwd / (double)fwd > threshold;
    }
    const uint64_t cpu = n.i[metric_a].sum, gpu = n.i[metric_b].sum;  // n.cpu_time / n.gpu_time > cpu_threshold
    return cpu > floor_v && (double)cpu / (double)(gpu > 0 ? gpu : 1) > threshold;
  };
  // for n in bfs(call_tree.nodes): canonical ids are breadth-first (reading R2), so ascending
  // id order is the BFS; a node below a flagged frame is not re-flagged
  std::vector<char> flagged(N, 0), below(N, 0);
  std::vector<uint32_t> res;
  for (size_t id = 1; id < N; ++id) {
    const uint32_t p = c->canon[c->t[c->order[id]].parent];
    below[id] = rule != OR_RULE_BWD_FWD && p != 0 && (below[p] || flagged[p]);  // ③: every operator node
    if (!below[id] && qualifies(id)) {
      flagged[id] = 1;
      res.push_back((uint32_t)id);
    }
  }
  for (size_t j = 0; j < res.size() && j < cap; ++j) out[j] = res[j];
  *n_out = (uint32_t)res.size();
  return 0;
}

struct OrStallIssue { uint32_t node, stall; uint64_t count; };

int or_stall_issues(const OrCct* c, uint32_t metric, uint32_t kind_mask, const uint8_t* frame_kind, uint32_t n_frames,
                    double hot_threshold, double stall_threshold, uint32_t k, OrStallIssue* out, uint32_t cap,
                    uint32_t* n_out) {
  *n_out = 0;
  if (!c->final_) return 1;
  if (k > 32) k = 32;
  // hotspots = hotspot_analysis(call_tree)
  std::vector<OrTopk> hot(c->order.size());
  uint32_t nh = 0;
  int rc = or_topk(c, OR_VIEW_INCLUSIVE, metric, kind_mask, frame_kind, n_frames, hot_threshold, (uint32_t)c->order.size(),
                   0, hot.data(), &nh);
  if (rc) return rc;
  uint32_t w = 0, total = 0;
  const uint32_t Nn = (uint32_t)c->order.size();
  for (uint32_t h = 0; h < nh; ++h) {
    const uint32_t node = hot[h].id;
    const uint64_t ksamples = c->t[c->order[node]].isamples;
    // for c in n.children (the instruction children): c.stalls = its samples
    std::map<uint32_t, uint64_t> pc_total;                 // pc node id -> samples
    for (const auto& b : c->cbins) {
      const uint32_t pn = std::get<0>(b);
      if (c->pcs[pn - Nn].first == node) pc_total[pn] += std::get<2>(b);
    }
    std::map<uint16_t, uint64_t> reasons;                  // stall -> count over the kept children
    for (const auto& b : c->cbins) {
      const uint32_t pn = std::get<0>(b);
      if (c->pcs[pn - Nn].first != node) continue;
      if (ksamples > 0 && (double)pc_total[pn] / (double)ksamples > stall_threshold) reasons[std::get<1>(b)] += std::get<2>(b);
    }
    std::vector<std::pair<uint64_t, uint16_t>> r;          // stall_reasons = topk(stalls)
    for (auto& kv : reasons)
      if (kv.second) r.push_back({kv.second, kv.first});
    std::sort(r.begin(), r.end(), [](const std::pair<uint64_t, uint16_t>& a, const std::pair<uint64_t, uint16_t>& b) {
      if (a.first != b.first) return a.first > b.first;
      return a.second < b.second;
    });
    for (size_t j = 0; j < r.size() && j < k; ++j, ++total)
      if (w < cap) out[w++] = OrStallIssue{node, r[j].second, r[j].first};
  }
  *n_out = total;
  return 0;
}

// ---------------------------------------------------------------- derived
// 256-bit unsigned, little-endian limbs.
struct U256 { uint64_t w[4]; };

static U256 u256_mul_64_128(uint64_t a, u128 b) {
  U256 r = {{0, 0, 0, 0}};
  u128 lo = (u128)a * (uint64_t)b;
  u128 hi = (u128)a * (uint64_t)(b >> 64);
  r.w[0] = (uint64_t)lo;
  u128 mid = (lo >> 64) + (uint64_t)hi;
  r.w[1] = (uint64_t)mid;
  u128 top = (mid >> 64) + (hi >> 64);
  r.w[2] = (uint64_t)top;
  r.w[3] = (uint64_t)(top >> 64);
  return r;
}
static U256 u256_sub(U256 a, U256 b) {  // requires a >= b
  U256 r;
  uint64_t borrow = 0;
  for (int q = 0; q < 4; ++q) {
    u128 d = (u128)a.w[q] - (u128)b.w[q] - (u128)borrow;  // wraps mod 2^128 when negative
    r.w[q] = (uint64_t)d;
    borrow = (uint64_t)(d >> 64) ? 1 : 0;
  }
  return r;
}
// Round-to-nearest-even conversion by explicit bit extraction (no FP intermediates).
static double u256_to_double_rne(U256 a) {
  int top = -1;
  for (int q = 3; q >= 0 && top < 0; --q)
    if (a.w[q]) top = q * 64 + 63 - __builtin_clzll(a.w[q]);
  if (top < 0) return 0.0;
  auto bit = [&](int b) -> uint64_t { return b < 0 ? 0 : (a.w[b >> 6] >> (b & 63)) & 1u; };
  if (top <= 52) {
    return (double)a.w[0];  // < 2^53: exact
  }
  uint64_t mant = 0;
  for (int b = top; b >= top - 52; --b) mant = (mant << 1) | bit(b);
  uint64_t round = bit(top - 53);
  uint64_t sticky = 0;
  for (int b = top - 54; b >= 0; --b) sticky |= bit(b);
  if (round && (sticky || (mant & 1))) mant += 1;
  int e = top - 52;
  if (mant == (1ull << 53)) { mant >>= 1; e += 1; }
  return ldexp((double)mant, e);
}

int or_derived(const OrCct* c, uint32_t metric, int incl, double* mean, double* stdv) {
  if (!c->final_ || metric >= c->M) return 1;
  for (size_t id = 0; id < c->order.size(); ++id) {
    const TNode& n = c->t[c->order[id]];
    uint64_t cnt = incl ? n.icnt : n.xcnt;
    const Agg& a = incl ? n.i[metric] : n.x[metric];
    if (cnt == 0) { mean[id] = 0.0; stdv[id] = 0.0; continue; }  // reading R11
    mean[id] = (double)a.sum / (double)cnt;
    U256 n_s2 = u256_mul_64_128(cnt, a.sq);
    U256 s1sq = u256_mul_64_128(a.sum, (u128)a.sum);
    double D = u256_to_double_rne(u256_sub(n_s2, s1sq));
    stdv[id] = sqrt(D) / (double)cnt;
  }
  return 0;
}

// exposed for the pin tests of the 256-bit helpers
double or_u256_to_double(const uint64_t w[4]) {
  U256 a; memcpy(a.w, w, 32);
  return u256_to_double_rne(a);
}

}  // extern "C"
