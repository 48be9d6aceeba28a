// Batched pred, host side (§4.4 P:239-243 batch assembly; §4.1 P:215 append): validate and
// reserve every descriptor in order (R11), then emit the plan the data plane consumes: the packed
// descriptor list, per-row destination slots of the append, copy-on-write copies, and the slab
// updates (table deltas) of the files in the batch.
#include <algorithm>
#include <cstring>
#include <unordered_map>

#include "kvfs_impl.h"

namespace kvfs {

int pred_reserve(Ctx &c, const pred_desc *descs, int n_desc, const int32_t *pos, int *status, PredPlan *plan) {
  const int P = c.cfg.page_size;
  const int Hkv = c.cfg.n_kv_heads;
  if (n_desc < 0 || n_desc > c.cfg.max_batch_descs || (n_desc > 0 && !descs)) return KVFS_EINVAL;
  int64_t T = 0;
  for (int i = 0; i < n_desc; ++i) {
    if (descs[i].n_q < 0) return KVFS_EINVAL;
    T += descs[i].n_q;
  }
  if (T > c.cfg.max_batch_rows || (T > 0 && !pos)) return KVFS_EINVAL;

  const bool device = c.dev != nullptr;
  PredPlan &pl = *plan;
  pl.descs.clear();
  pl.run_dst.clear();
  pl.run_entries.clear();
  pl.copies.clear();
  pl.dst_slot.assign(static_cast<size_t>(T), -1);
  pl.total_cost = 0;
  pl.n_units = 0;
  pl.T = static_cast<int32_t>(T);
  pl.max_nq = 0;
  const int64_t tag = ++c.batch_counter;

  pl.chunk_descs.clear();
  pl.chunk_units.clear();
  pl.chunk_dst.clear();
  pl.desc_files.clear();
  pl.score_src.clear();
  pl.prefix_descs.clear();
  pl.prefix_units.clear();
  pl.prefix_rows.clear();
  pl.prefix_cta_units.clear();
  pl.prefix_partials = 0;
  pl.prefix_groups = 0;
  pl.decode_sms = 0;
  std::vector<int32_t> dst;
  int64_t row = 0;
  bool partial = false;
  for (int i = 0; i < n_desc; ++i) {
    const int64_t row0 = row;
    const int nq = descs[i].n_q;
    row += nq;
    int st = KVFS_OK;
    File *f = get_file(c, descs[i].fd);
    if (!f) {
      st = KVFS_EBADF;
    } else if (f->batch_tag == tag) {
      st = KVFS_EBUSY;
    } else if (f->offloaded) {
      f->batch_tag = tag;
      st = KVFS_EOFFLOAD;
    } else {
      f->batch_tag = tag;
      if (nq > 0) {
        int64_t need = 0, new_entries = 0;
        st = append_plan(c, *f, nq, pos + row0, &need, &new_entries);
        if (st == KVFS_OK && device) {
          // the table may outgrow the file's slab block: get the new block before committing
          const int64_t size_after = static_cast<int64_t>(f->table.size()) + new_entries;
          if (size_after > f->slab_cap) {
            int64_t off = 0, cap = 0;
            if (!c.slab.alloc(std::max<int64_t>(size_after, 2 * static_cast<int64_t>(f->table.size())), &off, &cap) &&
                !c.slab.alloc(size_after, &off, &cap)) {
              st = KVFS_ENOMEM;
            } else {
              release_file_slab(c, *f);  // resets dirty_from = 0: the whole table is uploaded
              f->slab_off = off;
              f->slab_cap = cap;
            }
          }
        }
        if (st == KVFS_OK) {
          const int64_t n_old = f->len;
          dst.clear();
          append_commit(c, *f, nq, pos + row0, &dst, &pl.copies);
          fault_point(c);  // tests: an exception mid-way through a batch (KVFS_OPT_FAULT_INJECT)
          std::copy(dst.begin(), dst.end(), pl.dst_slot.begin() + row0);
          int64_t idx = static_cast<int64_t>(f->table.size()) - 1;
          while (idx >= 0 && f->table[idx].lstart >= n_old) --idx;
          int64_t fne = idx < 0 ? 0 : idx;  // entry holding logical token n_old
          if (idx >= 0 && f->table[idx].lstart + __builtin_popcountll(f->table[idx].mask) <= n_old) fne = idx + 1;
          DevDesc d{};
          d.logit_off = -1;
          d.cost_begin = pl.total_cost;
          d.slab_off = static_cast<int32_t>(f->slab_off);
          d.n_old_entries = static_cast<int32_t>(idx + 1);
          d.n_old = static_cast<int32_t>(n_old);
          d.n_q = nq;
          d.row0 = static_cast<int32_t>(row0);
          d.unit_base = pl.n_units;
          d.stages_per_unit = d.n_old_entries + (nq + P - 1) / P;
          d.n_entries = static_cast<int32_t>(f->table.size());
          d.tail_lstart = idx >= 0 ? f->table[idx].lstart : 0;
          d.first_new_entry = static_cast<int32_t>(fne);
          d.first_new_lstart = f->table[fne].lstart;
          pl.descs.push_back(d);
          pl.desc_files.push_back(f);
          f->score_slot = static_cast<int32_t>(pl.score_src.size());
          pl.score_src.push_back({i, d.slab_off, nq, d.row0, f});
          pl.total_cost += static_cast<int64_t>(Hkv) * nq * d.stages_per_unit;
          pl.n_units += Hkv * nq;
          pl.max_nq = std::max(pl.max_nq, nq);
          if (device) {
            // device table deltas: in-place point updates below dirty_from, then the dirty suffix
            const size_t n_ent = f->table.size();
            // (one slab index per entry: the prologue applies each delta with ONE read of host memory)
            for (uint32_t e : f->dirty_pts) {
              if (e >= f->dirty_from || e >= n_ent) continue;
              pl.run_dst.push_back(f->slab_off + e);
              pl.run_entries.push_back(f->table[e]);
            }
            f->dirty_pts.clear();
            for (size_t e = f->dirty_from; e < n_ent; ++e) pl.run_dst.push_back(f->slab_off + static_cast<int64_t>(e));
            if (f->dirty_from < n_ent)
              pl.run_entries.insert(pl.run_entries.end(), f->table.begin() + static_cast<long>(f->dirty_from),
                                    f->table.end());
            f->dirty_from = n_ent;
          }
        }
      }
    }
    if (status) status[i] = st;
    if (st != KVFS_OK) partial = true;
  }
  c.ctr.page_copies += static_cast<int64_t>(pl.copies.size());
  return partial ? KVFS_EPARTIAL : KVFS_OK;
}

}  // namespace kvfs

namespace kvfs {

void pred_split(const Ctx &c, int64_t cutover, PredPlan *plan) {
  PredPlan &pl = *plan;
  if (cutover <= 0 || c.cfg.head_dim != 128) return;
  const int P = c.cfg.page_size, Hkv = c.cfg.n_kv_heads, G = c.cfg.n_q_heads / c.cfg.n_kv_heads;
  std::vector<DevDesc> keep;
  std::vector<File *> keep_files;
  int64_t cost = 0;
  int32_t units = 0;
  for (size_t i = 0; i < pl.descs.size(); ++i) {
    const DevDesc &d = pl.descs[i];
    if (d.n_q >= cutover) {
      if (pl.chunk_dst.empty()) pl.chunk_dst.assign(static_cast<size_t>(pl.T), -1);
      ChunkDesc cd{d.slab_off, d.n_entries, d.n_old, d.n_q, d.row0, d.first_new_entry, d.first_new_lstart, 0};
      const int32_t di = static_cast<int32_t>(pl.chunk_descs.size());
      pl.chunk_descs.push_back(cd);
      const int mt = (d.n_q * G + 127) / 128;  // 128-row M-tiles; one CTA takes a pair (shared K/V tiles)
      for (int g = 0; g < Hkv; ++g)
        for (int m = 0; m < (mt + 1) / 2; ++m) pl.chunk_units.push_back({di, g, m, 0});
      for (int r = 0; r < d.n_q; ++r) pl.chunk_dst[d.row0 + r] = pl.dst_slot[d.row0 + r];
      continue;
    }
    DevDesc k = d;
    k.cost_begin = cost;
    k.unit_base = units;
    cost += static_cast<int64_t>(Hkv) * d.n_q * d.stages_per_unit;
    units += Hkv * d.n_q;
    keep.push_back(k);
    keep_files.push_back(pl.desc_files[i]);
  }
  (void)P;
  pl.descs.swap(keep);
  pl.desc_files.swap(keep_files);
  pl.total_cost = cost;
  pl.n_units = units;
}

}  // namespace kvfs

namespace kvfs {

// Shared-prefix (cascade) planning, SURVEY §8(f) NEXT-1.  Fork shares pages without copying them (PAPER.md
// §4.2, `fig:example` P:177); a batch of decode steps of a fork family then reads the same leading
// pages once per member.  Here the run of identical leading (page, mask) entries common to a family is
// attended once per (family, kv head, key split) with all members' query rows as the M dimension of the
// tcgen05 kernel, and every member's decode unit starts after the run and merges the prefix partials
// (exact: softmax over a disjoint union of key sets = log-sum-exp merge of the parts).
void pred_cascade(const Ctx &c, int64_t min_entries, int force_splits, int paired_mode, int sms, int64_t max_partials,
                  PredPlan *plan) {
  PredPlan &pl = *plan;
  pl.prefix_descs.clear();
  pl.prefix_units.clear();
  pl.prefix_rows.clear();
  pl.prefix_cta_units.clear();
  pl.prefix_partials = 0;
  pl.prefix_groups = 0;
  const int P = c.cfg.page_size, Hkv = c.cfg.n_kv_heads, G = c.cfg.n_q_heads / c.cfg.n_kv_heads;
  if (min_entries <= 0 || c.cfg.head_dim != 128 || pl.descs.size() < 2) return;
  const int epb = 128 / P;  // page entries per 128-key tile
  // families: descriptors keyed by their first page (shared: refcount >= 2), in first-appearance order
  std::unordered_map<uint32_t, int> gid;
  std::vector<std::vector<int>> fam;
  for (size_t i = 0; i < pl.descs.size(); ++i) {
    const File *f = pl.desc_files[i];
    if (pl.descs[i].first_new_entry < min_entries || f->table.empty()) continue;
    const uint32_t p0 = f->table[0].page;
    if (c.pool->refcnt(p0) < 2) continue;
    auto it = gid.find(p0);
    if (it == gid.end()) {
      gid.emplace(p0, static_cast<int>(fam.size()));
      fam.push_back({static_cast<int>(i)});
    } else {
      fam[it->second].push_back(static_cast<int>(i));
    }
  }
  struct Fam {
    int idx, E, rows, tiles, mpairs, S;
  };
  std::vector<Fam> use;
  for (size_t k = 0; k < fam.size(); ++k) {
    const std::vector<int> &m = fam[k];
    if (m.size() < 2) continue;
    const File *lf = pl.desc_files[m[0]];
    const Entry *lead = lf->table.data();
    int E = pl.descs[m[0]].first_new_entry;
    for (size_t j = 1; j < m.size() && E > 0; ++j) {
      File *bf = pl.desc_files[m[j]];
      const int lim = std::min(E, pl.descs[m[j]].first_new_entry);
      // The number of leading entries identical (page, mask and so the logical start) to the leader's is
      // cached per member with both files' table stamps: it changes only when one of the tables is changed
      // in place (a new stamp), not by appends (File::tver).  Otherwise one memcmp over the whole common
      // length, the (page, mask) scan only when it differs somewhere.
      if (bf->run_lead != lf || bf->run_lead_tver != lf->tver || bf->run_self_tver != bf->tver) {
        const Entry *b = bf->table.data();
        const size_t n = std::min(lf->table.size(), bf->table.size());
        size_t e = n;
        if (std::memcmp(lead, b, n * sizeof(Entry)) != 0) {
          e = 0;
          while (e < n && b[e].page == lead[e].page && b[e].mask == lead[e].mask) ++e;
        }
        bf->run_lead = lf;
        bf->run_lead_tver = lf->tver;
        bf->run_self_tver = bf->tver;
        bf->run_len = static_cast<int64_t>(e);
      }
      E = static_cast<int>(std::min<int64_t>(lim, bf->run_len));
    }
    if (E < min_entries) continue;
    int rows = 0;
    for (int i : m) rows += pl.descs[i].n_q;
    const int mt = (rows * G + 127) / 128;
    use.push_back({static_cast<int>(k), E, rows, (E + epb - 1) / epb, (mt + 1) / 2, 1});
  }
  if (use.empty()) return;
  // Key splits: about one CTA per SM over all families, at most kMaxPrefixSplits and at most one per tile.
  // The S split CTAs of a (family, kv head, M-tile pair) group exchange their partials through global memory
  // and each merges a slice of the group's rows, so the decode kernel folds ONE prefix partial per unit.
  // Their wait for each other needs every CTA of the grid resident at once (one CTA per SM): with S > 1 the
  // grid is at most one CTA per SM.
  int64_t units_per_split = 0, rows_all = 0;
  for (const Fam &u : use) {
    units_per_split += static_cast<int64_t>(Hkv) * u.mpairs;
    rows_all += u.rows;
  }
  const int64_t fit = std::max<int64_t>(1, sms / std::max<int64_t>(1, units_per_split));
  // The prefix grid (units_per_split * S CTAs, one per SM) is launched first and the decode kernel after it
  // (programmatic launch).  Either the decode rings take only the SMs the prefix CTAs leave free ("shrink":
  // they merge the prefix records at the end of their ranges, so the two kernels run side by side), or all
  // SMs (the rings on the prefix CTAs' SMs start when those finish).  A cost model picks S and the mode:
  // prefix CTA ~kPrefFixed + kPrefTile per 128-key tile of its split, decode ~kDecFixed + its bytes at
  // kSmBytesPerUs per SM.  B200 constants measured on cfg3 (tools/cascade_trace.py, ncu): 3.7 us start +
  // 3.6 us epilogue + 3.3 us split merge + ~2 us exit, 1.8 us per tile of an M-tile pair; the decode kernel
  // alone on 33-stage units streams ~29 GB/s per SM (profiles/r02_k1_cfg3_ncu.txt).
  // With S <= kMaxFoldSplits the split CTAs do not merge: each writes its records and the decode kernel folds
  // the S records of its unit (all loads of a group of 4 in flight), which drops the group wait, the merge and
  // the full write-completion wait of the epilogue from the prefix CTA (~12 -> ~6.5 us of fixed cost; cfg3:
  // 0.0555 -> 0.048 ms of kernels per step, tools/cascade_trace.py).
  // Round-2 constants (tools/cascade_trace.py on cfg3): fold-mode prefix CTA ~6.6 us fixed (0.3 wait, 2.6 to
  // the first S, 3.7 epilogue) + 2.0 us per tile; decode rings stream ~10 GB/s each, 4 per SM, after ~5 us
  // of start and merge.  In "shrink" mode a ring count between the unit count and 4x it cuts units across
  // rings, whose extra segment starts and cross-ring merges were measured to cost more than the SMs they
  // free (cfg3 S = 3: 0.063 ms against 0.050 for S = 2), so such layouts are not considered.
  constexpr double kPrefFixed = 12.0, kPrefFixedFold = 6.6, kPrefTile = 2.0, kDecFixed = 5.0, kSmBytesPerUs = 40e3;
  auto rings_ok = [&](int64_t free_sms) {
    const int64_t rings = free_sms * 4;
    return pl.n_units <= rings || pl.n_units >= 4 * rings;
  };
  int max_tiles = 0;
  for (const Fam &u : use) max_tiles = std::max(max_tiles, u.tiles);
  double dec_bytes = 0;  // decode-kernel bytes once the runs are skipped
  {
    std::vector<int> runE(pl.descs.size(), 0);
    for (const Fam &u : use)
      for (int i : fam[u.idx]) runE[static_cast<size_t>(i)] = u.E;
    for (size_t i = 0; i < pl.descs.size(); ++i) {
      const DevDesc &d = pl.descs[i];
      const int spu = (d.n_old_entries - runE[i]) + (d.n_q + P - 1) / P;
      dec_bytes += static_cast<double>(Hkv) * d.n_q * spu * 2.0 * P * c.cfg.head_dim * 2;
    }
  }
  int S = 1;
  bool shrink = false;
  double best = 1e30;
  auto model = [&](int s, bool shr) {
    const int64_t free_sms = sms - units_per_split * s;
    const double tp = (s > 1 && s <= kMaxFoldSplits ? kPrefFixedFold : kPrefFixed) + kPrefTile * ((max_tiles + s - 1) / s);
    if (!shr) return tp + kDecFixed + dec_bytes / (static_cast<double>(sms) * kSmBytesPerUs);
    if (free_sms < 1 || !rings_ok(free_sms)) return 1e30;
    return std::max(tp, kDecFixed + dec_bytes / (static_cast<double>(free_sms) * kSmBytesPerUs));
  };
  // Paired partition (fold, S = 3): the (kv head, M-tile pair) lanes of a family are taken in pairs (a, b);
  // lane a is cut into key pieces (x, x, r) and lane b into (r, x, x), r = tiles - 2x, and a pair runs on 5
  // CTAs: [a0] [a1] [a2 then b0] [b1] [b2] (one CTA runs two short units in turn).  2.5 CTAs per lane
  // instead of 2 or 3 lets the prefix grid take exactly the SMs the decode rings leave (cfg3: 20 = 148 - 128).
  int64_t paired_ctas = 0;
  bool paired_possible = true;
  double paired_tp = 0;
  std::vector<int> pair_x(use.size(), 0);
  for (size_t k = 0; k < use.size(); ++k) {
    const Fam &u = use[k];
    const int lanes = Hkv * u.mpairs;
    if (lanes % 2 != 0 || u.tiles < 3) {
      paired_possible = false;
      break;
    }
    paired_ctas += static_cast<int64_t>(lanes / 2) * 5;
    double bt = 1e30;
    for (int x = 1; 2 * x < u.tiles; ++x) {
      const int r = u.tiles - 2 * x;
      const double t = std::max(kPrefFixedFold + kPrefTile * x, 2 * kPrefFixedFold + kPrefTile * 2 * r);
      if (t < bt) {
        bt = t;
        pair_x[k] = x;
      }
    }
    paired_tp = std::max(paired_tp, bt);
  }
  auto model_paired = [&]() {
    const int64_t free_sms = sms - paired_ctas;
    if (!paired_possible || free_sms < 1 || !rings_ok(free_sms)) return 1e30;
    return std::max(paired_tp, kDecFixed + dec_bytes / (static_cast<double>(free_sms) * kSmBytesPerUs));
  };
  for (int s = 1; s <= std::min<int64_t>(kMaxPrefixSplits, fit); ++s)
    for (bool shr : {false, true}) {
      const double t = model(s, shr);
      if (t < best - 1e-9) {
        best = t;
        S = s;
        shrink = shr;
      }
    }
  bool paired = paired_mode != 1 && model_paired() < best - 1e-9;
  if (force_splits > 0) {
    S = static_cast<int>(std::min<int64_t>(std::min(force_splits, kMaxPrefixSplits), fit));
    shrink = model(S, true) < model(S, false);
    paired = false;
  }
  if (paired_mode == 2 && paired_possible && paired_ctas < sms) paired = true;
  if (rows_all * Hkv * 3 > max_partials) paired = false;  // its 3 records per (member row, kv head) must fit
  if (paired) {
    S = 3;
    shrink = true;
  }

  const bool fold = S > 1 && S <= kMaxFoldSplits;
  pl.prefix_fold = fold ? 1 : 0;
  // workspace: one merged partial per (member row, kv head), plus S split partials when S > 1 (fold: S
  // split partials only)
  while (S > 1 && rows_all * Hkv * (fold ? S : S + 1) > max_partials) --S;
  if (rows_all * Hkv > max_partials) return;  // workspace too small: no cascade
  pl.decode_sms = shrink ? static_cast<int32_t>(sms - (paired ? paired_ctas : units_per_split * S)) : 0;
  int64_t merged = rows_all * Hkv;            // split partials live after the merged ones
  int64_t split_next = merged;
  int32_t group = 0;
  for (Fam &u : use) {
    u.S = std::min(S, u.tiles);  // splits of the family: tiles spread evenly, none empty
    const std::vector<int> &m = fam[u.idx];
    const int row0 = static_cast<int>(pl.prefix_rows.size());
    // members whose query rows follow each other in the packed batch (e.g. a family's consecutive decode
    // descriptors): the prefix kernel loads Q tiles by TMA instead of gathering rows
    int32_t q_t0 = pl.descs[m[0]].row0;
    for (size_t j = 1; j < m.size() && q_t0 >= 0; ++j)
      if (pl.descs[m[j]].row0 != pl.descs[m[j - 1]].row0 + pl.descs[m[j - 1]].n_q) q_t0 = -1;
    const int32_t merged_base = pl.prefix_partials;
    const bool ufold = fold && u.S > 1;
    for (int i : m) {
      DevDesc &d = pl.descs[i];
      d.skip = u.E;
      // the decode kernel reads the merged partial of unit (g, qi): pref_base + g * n_q + qi; fold: the
      // S split records pref_base + (g * n_q + qi) * S + s
      d.pref_splits = ufold ? u.S : 1;
      d.pref_base = pl.prefix_partials;
      pl.prefix_partials += Hkv * d.n_q * (ufold ? u.S : 1);
      d.stages_per_unit = (d.n_old_entries - u.E) + (d.n_q + P - 1) / P;
      for (int qi = 0; qi < d.n_q; ++qi) pl.prefix_rows.push_back({d.row0 + qi, d.pref_base, d.n_q, qi});
    }
    // split partial of merged record r, split s: split_off + r * S + s (split_off = split base - merged base * S)
    const int32_t split_off =
        ufold ? -1 : static_cast<int32_t>(u.S > 1 ? split_next - static_cast<int64_t>(merged_base) * u.S : 0);
    if (u.S > 1 && !ufold) split_next += static_cast<int64_t>(pl.prefix_partials - merged_base) * u.S;
    const DevDesc &lead = pl.descs[m[0]];
    if (paired) {
      const int x = pair_x[static_cast<size_t>(&u - use.data())], r = u.tiles - 2 * x;
      // key pieces of the lanes "a" (x, x, r) and "b" (r, x, x): six prefix descriptors, splits 0..2 each
      const int cuts[2][4] = {{0, x, 2 * x, u.tiles}, {0, r, r + x, u.tiles}};
      const int32_t d0 = static_cast<int32_t>(pl.prefix_descs.size());
      for (int par = 0; par < 2; ++par)
        for (int sp = 0; sp < 3; ++sp) {
          const int e0 = cuts[par][sp] * epb, e1 = std::min(u.E, cuts[par][sp + 1] * epb);
          pl.prefix_descs.push_back({lead.slab_off + e0, e1 - e0, u.rows, row0, sp, 3, q_t0, -1});
        }
      std::vector<std::pair<int, int>> lanes;  // (kv head, M-tile pair)
      for (int g = 0; g < Hkv; ++g)
        for (int mp = 0; mp < u.mpairs; ++mp) lanes.push_back({g, mp});
      auto unit = [&](int par, int sp, const std::pair<int, int> &ln) {
        return ChunkUnit{d0 + par * 3 + sp, ln.first, ln.second, group};
      };
      auto cta = [&](std::initializer_list<ChunkUnit> us) {
        pl.prefix_cta_units.push_back(static_cast<int32_t>(pl.prefix_units.size()));
        pl.prefix_cta_units.push_back(static_cast<int32_t>(us.size()));
        for (const ChunkUnit &cu : us) pl.prefix_units.push_back(cu);
      };
      for (size_t l = 0; l + 1 < lanes.size(); l += 2, ++group) {
        const auto &a = lanes[l], &b = lanes[l + 1];
        cta({unit(0, 0, a)});
        cta({unit(0, 1, a)});
        cta({unit(0, 2, a), unit(1, 0, b)});
        cta({unit(1, 1, b)});
        cta({unit(1, 2, b)});
      }
      ++pl.prefix_groups;
      continue;
    }
    for (int sp = 0; sp < u.S; ++sp) {
      const int t0 = sp * u.tiles / u.S, t1 = (sp + 1) * u.tiles / u.S;
      const int e0 = t0 * epb, e1 = std::min(u.E, t1 * epb);
      pl.prefix_descs.push_back({lead.slab_off + e0, e1 - e0, u.rows, row0, sp, u.S, q_t0, split_off});
    }
    // CTAs: group (g, M-tile pair) -> its S splits consecutively; ChunkUnit.pad = group id
    const int32_t d0 = static_cast<int32_t>(pl.prefix_descs.size()) - u.S;
    for (int g = 0; g < Hkv; ++g)
      for (int mp = 0; mp < u.mpairs; ++mp, ++group)
        for (int sp = 0; sp < u.S; ++sp) pl.prefix_units.push_back({d0 + sp, g, mp, group});
    ++pl.prefix_groups;
  }
  (void)merged;
  // the members' decode work shrank: re-pack the K1 stage ranges
  int64_t cost = 0;
  for (DevDesc &d : pl.descs) {
    d.cost_begin = cost;
    cost += static_cast<int64_t>(Hkv) * d.n_q * d.stages_per_unit;
  }
  pl.total_cost = cost;
}

}  // namespace kvfs

namespace kvfs {

// Fused scores: logits space in the caller's buffer for every descriptor the decode kernel attends in full
// (not a chunk descriptor, no shared-prefix skip), in descriptor order while it fits; the others keep the
// K9 score pass.  Unit (g, qi) of descriptor d takes stages_per_unit * P * G floats.
void pred_logits(Ctx &c, PredPlan *plan) {
  PredPlan &pl = *plan;
  const int P = c.cfg.page_size, Hkv = c.cfg.n_kv_heads, G = c.cfg.n_q_heads / c.cfg.n_kv_heads;
  int64_t off = 0;
  for (size_t i = 0; i < pl.descs.size(); ++i) {
    DevDesc &d = pl.descs[i];
    d.logit_off = -1;
    if (!c.logits_buf || d.skip != 0) continue;
    const int64_t need = static_cast<int64_t>(Hkv) * d.n_q * d.stages_per_unit * P * G;
    if (off + need > c.logits_cap) continue;
    d.logit_off = off;
    off = (off + need + 31) & ~int64_t{31};  // 128-byte aligned regions: the score pass discards whole L2 lines
    const File *f = pl.desc_files[i];
    if (f->score_slot >= 0 && f->score_slot < static_cast<int32_t>(pl.score_src.size())) {
      ScoreSrc &x = pl.score_src[static_cast<size_t>(f->score_slot)];
      x.logit_off = d.logit_off;
      x.n_old = d.n_old;
      x.n_old_entries = d.n_old_entries;
      x.stages_per_unit = d.stages_per_unit;
    }
  }
}

}  // namespace kvfs
