// Batch plan construction (host) and its C ABI.  See plan.hpp.
#include <algorithm>
#include <queue>
#include <cstring>
#include <memory>
#include <numeric>

#include "plan.hpp"

using namespace plora;

namespace {

struct Seg {
  uint32_t adapter, rank, table_off, voff;
  std::vector<uint32_t> toks;
};

}  // namespace

void plora_plan::drop_tp() {
  if (tpw.empty()) return;
  DeviceCtx ctx(store->device);
  for (auto& kv : tpw) {
    cudaFree(kv.second.d_items);  // implicit device synchronisation: no TP launch still reads it
    cudaFreeHost(kv.second.h_stage);
  }
  tpw.clear();
}

void plora_plan::build(const int32_t* token_adapter, uint32_t n, cudaStream_t stream) {
  drop_tp();  // TP item lists follow the batch
  const plora_store& st = *store;
  const ModelGeom& g = st.geom;
  const uint32_t es = g.esize, vec = 16 / es;

  // ---- group tokens by adapter (validates residency on the host shadow)
  std::vector<int32_t> seg_of(st.max_adapters, -1);
  std::vector<Seg> segs;
  for (uint32_t t = 0; t < n; ++t) {
    const int32_t a = token_adapter[t];
    if (a < 0) continue;
    if (static_cast<uint32_t>(a) >= st.max_adapters)
      throw ValidationError("token " + std::to_string(t) + " names adapter " + std::to_string(a) +
                            " >= max_adapters");
    if (!st.slots[a].published)
      throw ValidationError("token " + std::to_string(t) + " names adapter " + std::to_string(a) +
                            " which is not resident (publish it first)");
    if (seg_of[a] < 0) {
      seg_of[a] = static_cast<int32_t>(segs.size());
      segs.push_back(Seg{static_cast<uint32_t>(a), st.h_dir[a].rank, st.h_dir[a].table_off, 0, {}});
    }
    segs[seg_of[a]].toks.push_back(t);
  }
  // ascending adapter key (deterministic), v offsets 16-byte aligned
  std::sort(segs.begin(), segs.end(), [](const Seg& x, const Seg& y) { return x.adapter < y.adapter; });
  v_elems = 0;
  max_rank = 0;
  for (Seg& s : segs) {
    if (s.rank > kMaxBgmvRank)
      throw ValidationError("adapter " + std::to_string(s.adapter) + " has rank " +
                            std::to_string(s.rank) + " > " + std::to_string(kMaxBgmvRank));
    s.voff = static_cast<uint32_t>(v_elems);
    v_elems += static_cast<uint64_t>(s.toks.size()) * rpad4(s.rank);
    max_rank = std::max(max_rank, s.rank);
  }
  if (v_elems > 0xffffffffull) throw ValidationError("batch too large for one plan");
  n_tokens = n;
  n_seg = static_cast<uint32_t>(segs.size());

  // schedule order: largest rank first (LPT), ties by adapter key
  std::vector<uint32_t> order(n_seg);
  std::iota(order.begin(), order.end(), 0u);
  std::stable_sort(order.begin(), order.end(),
                   [&](uint32_t x, uint32_t y) { return segs[x].rank > segs[y].rank; });

  // ---- many-token adapters -> the tensor-core SGMV path on a child plan
  // (bgmv.cu launch_routed): bf16 stores, rank <= 128 and the SGMV geometry
  // for every projection
  seg_route.assign(segs.size(), 0);
  route_perm.clear();
  n_route = 0;
  {
    bool tc_ok = es == 2 && !no_route && route_min_tokens() > 0;
    for (uint32_t p = 0; p < g.m.n_proj && tc_ok; ++p)
      tc_ok = g.m.d_in[p] % 64 == 0 && g.m.d_out[p] % 128 == 0 && g.blocks_aligned_128(p);
    std::vector<int32_t> child_ta;
    for (uint32_t si = 0; si < segs.size() && tc_ok; ++si) {
      const Seg& sg = segs[si];
      if (sg.toks.size() < route_min_tokens() || sg.rank > 128) continue;
      seg_route[si] = 1;
      for (uint32_t tk : sg.toks) {
        route_perm.push_back(tk);
        child_ta.push_back(static_cast<int32_t>(sg.adapter));
      }
    }
    n_route = static_cast<uint32_t>(route_perm.size());
    if (n_route) {
      if (!route) {
        route = new plora_plan;
        route->store = store;
        route->no_route = true;
      }
      route->build(child_ta.data(), n_route, stream);
      uint32_t dmax = 0;
      uint64_t yb = 0;
      for (uint32_t p = 0; p < g.m.n_proj; ++p) {
        dmax = std::max(dmax, g.m.d_in[p]);
        yb += static_cast<uint64_t>(n_route) * g.m.d_out[p] * 2;
      }
      const uint64_t need = static_cast<uint64_t>(n_route) * dmax * 2 + yb;
      if (route_ws_cap < need) {
        DeviceCtx ctx(st.device);
        if (d_route_ws) {
          PLORA_CUDA(cudaStreamSynchronize(stream));
          cudaFree(d_route_ws);
        }
        d_route_ws = nullptr;
        PLORA_CUDA(cudaMalloc(&d_route_ws, need));
        route_ws_cap = need;
      }
    }
  }

  // ---- fp32 BGMV units per projection (the bf16 op runs on clusters, below)
  units.clear();
  for (uint32_t p = 0; p < g.m.n_proj; ++p) proj[p] = ProjWork{};
  for (uint32_t p = 0; p < g.m.n_proj && es == 4; ++p) {
    const uint32_t din = g.m.d_in[p], dout = g.m.d_out[p];
    const uint32_t rowbytes = din * es;
    if (es == 4 && rowbytes > kSlotAuxBytes)
      throw ValidationError("fp32 BGMV needs d_in * 4 <= " + std::to_string(kSlotAuxBytes) +
                            " bytes (d_in=" + std::to_string(din) + ")");
    // rpu full rank rows per shrink unit (CUDA cores)
    const uint32_t nkc = 1;
    const uint32_t rpu = std::min<uint32_t>(kMaxShrinkRows, kShrinkWeightBytes / rowbytes);
    const uint32_t nts = std::min<uint32_t>(kMaxUnitTok, kSlotAuxBytes / rowbytes);
    ProjWork& pw = proj[p];
    pw.units_off = static_cast<uint32_t>(units.size());
    std::vector<uint32_t> n_shrink(n_seg, 0);
    for (uint32_t si : order) {
      const Seg& s = segs[si];
      const uint32_t rp = rpad4(s.rank), nt_all = static_cast<uint32_t>(s.toks.size());
      const uint32_t vstride = nt_all * rp;
      for (uint32_t tc = 0; tc < nt_all; tc += nts) {
        const uint32_t nt = std::min(nts, nt_all - tc);
        for (uint32_t j0 = 0; j0 < s.rank; j0 += rpu) {
          for (uint32_t kc = 0; kc < nkc; ++kc) {
            BgmvUnit u{};
            u.kind_seg = si;
            u.off = j0;
            u.count = std::min(rpu, s.rank - j0);
            u.table_off = s.table_off;
            u.rank = s.rank;
            u.voff = s.voff + kc * vstride + tc * rp;
            u.ntok = nt;
            u.kc = kc;
            for (uint32_t t = 0; t < nt; ++t) u.tok[t] = s.toks[tc + t];
            units.push_back(u);
            ++n_shrink[si];
          }
        }
      }
    }
    pw.n_shrink = static_cast<uint32_t>(units.size()) - pw.units_off;
    for (uint32_t si : order) {
      const Seg& s = segs[si];
      const uint32_t rp = rpad4(s.rank), nt_all = static_cast<uint32_t>(s.toks.size());
      const uint32_t rg = expand_rg(s.rank), cb = expand_cols(s.rank, es);
      const uint32_t per_tok = nkc * rp * 4 + cb * es;
      // tokens per unit: aux area (v partial rows + y rows) and, when rows are
      // split over groups, the reduction buffer (RG · CB fp32 per token)
      const uint32_t aux_budget = kSlotAuxBytes;
      uint32_t nte = std::min<uint32_t>(kMaxUnitTok, aux_budget / per_tok);
      if (rg > 1) nte = std::min<uint32_t>(nte, kRedBytes / (rg * cb * 4));
      nte = std::max<uint32_t>(nte, 1);
      for (uint32_t tc = 0; tc < nt_all; tc += nte) {
        const uint32_t nt = std::min(nte, nt_all - tc);
        for (uint32_t c0 = 0; c0 < dout; c0 += cb) {
          BgmvUnit u{};
          u.kind_seg = si | kExpandBit;
          u.off = c0;
          u.count = std::min(cb, dout - c0);
          u.table_off = s.table_off;
          u.rank = s.rank;
          u.voff = s.voff + tc * rp;
          u.ntok = nt;
          u.n_shrink = n_shrink[si];
          u.nkc = nkc;
          u.vstride = nt_all * rp;
          for (uint32_t t = 0; t < nt; ++t) u.tok[t] = s.toks[tc + t];
          units.push_back(u);
        }
      }
    }
    pw.n_units = static_cast<uint32_t>(units.size()) - pw.units_off;
  }

  // ---- SGMV tiles: runs of consecutive tokens with the same adapter
  tiles.clear();
  gtiles.clear();
  uint32_t t = 0;
  while (t < n) {
    const int32_t a = token_adapter[t];
    uint32_t e = t + 1;
    while (e < n && token_adapter[e] == a) ++e;
    for (uint32_t r0 = t; r0 < e; r0 += 128) {
      const uint32_t nr = std::min<uint32_t>(128, e - r0);
      GemmTile gt{};
      gt.row0 = r0;
      gt.nrows = nr;
      gt.vtile = 0xffffffffu;
      if (a >= 0) {
        gt.table_off = st.h_dir[a].table_off;
        gt.rank = st.h_dir[a].rank;
        gt.vtile = static_cast<uint32_t>(tiles.size());
        tiles.push_back(SgmvTile{r0, nr, st.h_dir[a].table_off, st.h_dir[a].rank});
      }
      gtiles.push_back(gt);
    }
    t = e;
  }
  n_tiles = static_cast<uint32_t>(tiles.size());
  sunits.clear();
  for (uint32_t i = 0; i < n_tiles;) {
    const bool pair = i + 1 < n_tiles && tiles[i].nrows == 128 &&
                      tiles[i + 1].table_off == tiles[i].table_off &&
                      tiles[i + 1].rank == tiles[i].rank && tiles[i + 1].row0 == tiles[i].row0 + 128;
    sunits.push_back(i);
    sunits.push_back(pair ? i + 1 : 0xffffffffu);
    i += pair ? 2 : 1;
  }
  n_sunits = static_cast<uint32_t>(sunits.size() / 2);
  // persistent shrink schedules (bf16 tensor-core path only)
  sitems.clear();
  scta.clear();
  for (uint32_t p = 0; p < PLORA_MAX_PROJ; ++p) ssched[p] = SgmvSched{};
  ssched_layer = SgmvSched{};
  // units: {tile, tile or ~0u} pairs; np projections share each x chunk.
  // Split-K factor: each candidate's LPT makespan (bytes the busiest CTA
  // streams, at a per-SM share of HBM) plus the split reduction (partials
  // written and read back); the cheapest wins.  Few splits for heavy uniform
  // batches, more for mixed ranks.
  auto build_sched = [&](const std::vector<uint32_t>& un, uint32_t d_in, uint32_t np) {
    const uint32_t n_sm = std::max(1, st.num_sms);
    const uint32_t nu = static_cast<uint32_t>(un.size() / 2);
    std::vector<std::vector<SgmvItem>> per, best_per;
    uint32_t ks = 0;
    double best = 0.0;
    for (uint32_t cand = 1; cand <= 16; cand *= 2) {
      if ((d_in / 64) % cand != 0 || (cand > 1 && d_in / cand < 256)) break;
      const uint32_t kslice = d_in / cand;
      std::vector<std::pair<uint64_t, SgmvItem>> items;  // (cost, item)
      items.reserve(static_cast<size_t>(nu) * cand);
      uint64_t part_bytes = 0;
      for (uint32_t u = 0; u < nu; ++u) {
        const uint64_t nt = un[2 * u + 1] != 0xffffffffu ? 2 : 1;
        const SgmvTile& ta = tiles[un[2 * u]];
        const uint64_t r16 = (ta.rank + 15) / 16 * 16;
        // bytes streamed (x tiles + paged weights) plus the partial write-back
        const uint64_t cost = 2ull * kslice * (nt * 128 + np * r16) + 4ull * nt * np * 128 * r16;
        part_bytes += 8ull * nt * np * 128 * r16 * cand;
        for (uint32_t sp = 0; sp < cand; ++sp) {
          SgmvItem it{};
          it.tile_a = un[2 * u];
          it.tile_b = un[2 * u + 1];
          it.row0_a = ta.row0;
          it.row0_b = nt == 2 ? tiles[it.tile_b].row0 : 0;
          it.table_off = ta.table_off;
          it.rank = ta.rank;
          it.split = sp;
          items.emplace_back(cost, it);
        }
      }
      std::stable_sort(items.begin(), items.end(),
                       [](const auto& x, const auto& y) { return x.first > y.first; });
      const uint32_t ctas = std::min<uint32_t>(n_sm, static_cast<uint32_t>(items.size()));
      per.assign(ctas, {});
      using Load = std::pair<uint64_t, uint32_t>;
      std::priority_queue<Load, std::vector<Load>, std::greater<Load>> heap;
      for (uint32_t c = 0; c < ctas; ++c) heap.emplace(0, c);
      uint64_t makespan = 0;
      for (const auto& it : items) {
        Load l = heap.top();
        heap.pop();
        per[l.second].push_back(it.second);
        heap.emplace(l.first + it.first, l.second);
        makespan = std::max(makespan, l.first + it.first);
      }
      constexpr double kSmBw = 45e9, kHbmBw = 5e12;
      const double t = makespan / kSmBw + part_bytes / kHbmBw;
      if (ks == 0 || t < best) {
        ks = cand;
        best = t;
        best_per.swap(per);
      }
    }
    SgmvSched sc;
    sc.splits = ks;
    sc.ctas = static_cast<uint32_t>(best_per.size());
    sc.item_off = static_cast<uint32_t>(sitems.size());
    sc.cta_off = static_cast<uint32_t>(scta.size());
    uint32_t n = 0;
    for (uint32_t c = 0; c < sc.ctas; ++c) {
      scta.push_back(n);
      for (const SgmvItem& v : best_per[c]) sitems.push_back(v);
      n += static_cast<uint32_t>(best_per[c].size());
    }
    scta.push_back(n);
    return sc;
  };
  if (es == 2 && n_sunits > 0) {
    for (uint32_t p = 0; p < g.m.n_proj; ++p) {
      uint32_t same = p;
      for (uint32_t q = 0; q < p; ++q)
        if (g.m.d_in[q] == g.m.d_in[p]) same = q;
      ssched[p] = same != p ? ssched[same] : build_sched(sunits, g.m.d_in[p], 1);
    }
    // every projection of a layer from one x chunk (plora_sgmv_layer): single
    // tiles, since a unit holds at most two accumulators
    bool shared_x = g.m.n_proj == 2;
    for (uint32_t p = 1; p < g.m.n_proj; ++p) shared_x = shared_x && g.m.d_in[p] == g.m.d_in[0];
    if (shared_x) {
      std::vector<uint32_t> singles;
      for (uint32_t i = 0; i < n_tiles; ++i) {
        singles.push_back(i);
        singles.push_back(0xffffffffu);
      }
      ssched_layer = build_sched(singles, g.m.d_in[0], g.m.n_proj);
    }
  }

  // ---- decode step in one launch (plora_bgmv_layers), hybrid: the 4-CTA
  // clusters fit on 4·n_clusters SMs (132 of 148 on B200); the streaming
  // kernel (bgmv_stream.cu) runs a share of the adapters on the SMs they
  // leave idle, concurrently, sized by SM count (both stream ~31 GB/s per SM
  // at cfg2, profiles/r02g_hybrid_probe.txt)
  seg_hyb.assign(segs.size(), 0);
  hyb_spare = 0;
  hyb_frac = 0.0;
  bool layer_same = g.m.n_proj > 1;
  for (uint32_t p = 1; p < g.m.n_proj; ++p)
    layer_same = layer_same && g.m.d_in[p] == g.m.d_in[0] && g.m.d_out[p] == g.m.d_out[0];
  uint32_t seg_maxtok = 0, n_kept = 0;  // over the adapters the decode kernels keep
  for (uint32_t si = 0; si < segs.size(); ++si)
    if (!seg_route[si]) {
      seg_maxtok = std::max<uint32_t>(seg_maxtok, static_cast<uint32_t>(segs[si].toks.size()));
      ++n_kept;
    }
  // (batches with an adapter of more than 4 tokens would run the streaming
  // share with 8-token jobs, which measured 2x slower: clusters only then)
  if (es == 2 && layer_same && hybrid_enabled() && n_kept && seg_maxtok <= kJobTok) {
    const ClusterGeom cg = cluster_geom(g.m.d_in[0], g.m.d_out[0], st.device);
    const uint32_t sms = static_cast<uint32_t>(std::max(1, st.num_sms));
    const uint32_t used = cg.n_clusters * cg.cs;
    if (sms > used + 3) {
      hyb_spare = sms - used;
      uint64_t total = 0;
      for (const Seg& sg : segs) total += static_cast<uint64_t>(sg.rank) * sg.toks.size();
      std::vector<uint32_t> by(segs.size());
      std::iota(by.begin(), by.end(), 0u);
      auto bytes_of = [&](uint32_t i) {  // weight rows streamed per token group (rank per job)
        return seg_route[i] ? 0ull
                            : static_cast<uint64_t>(segs[i].rank) * ((segs[i].toks.size() + kJobTok - 1) / kJobTok);
      };
      uint64_t all = 0;
      for (uint32_t i = 0; i < segs.size(); ++i) all += bytes_of(i);
      std::stable_sort(by.begin(), by.end(), [&](uint32_t a, uint32_t b) { return bytes_of(a) > bytes_of(b); });
      const double target = static_cast<double>(all) * hyb_spare / sms * hybrid_share_factor();
      uint64_t acc = 0;
      for (uint32_t i : by)
        if (bytes_of(i) && static_cast<double>(acc + bytes_of(i)) <= target) {
          seg_hyb[i] = 1;
          acc += bytes_of(i);
        }
      if (acc == 0) hyb_spare = 0;
      hyb_frac = all ? static_cast<double>(acc) / static_cast<double>(all) : 0.0;
      (void)total;
    }
  }

  // ---- bf16 BGMV on clusters: jobs (<= kJobTok tokens of one adapter),
  // LPT-assigned to clusters by bytes, cut into kChunkRows-row chunks
  cjobs.clear();
  cchunks.clear();
  ccl_off.clear();
  ccl_jobs.clear();
  std::vector<uint8_t> cjob_hyb, cjob_route;
  if (es == 2) {
    for (uint32_t si = 0; si < segs.size(); ++si) {
      const Seg& s = segs[si];
      for (uint32_t tc = 0; tc < s.toks.size(); tc += kJobTok) {
        cjob_hyb.push_back(seg_hyb[si]);
        cjob_route.push_back(seg_route[si]);  // kept in cjobs (the TP halves serve every token)
        ClusterJob j{};
        j.table_off = s.table_off;
        j.rank = s.rank;
        j.ntok = std::min<uint32_t>(kJobTok, static_cast<uint32_t>(s.toks.size()) - tc);
        for (uint32_t t = 0; t < j.ntok; ++t) j.tok[t] = s.toks[tc + t];
        cjobs.push_back(j);
      }
    }
    const uint32_t nj = static_cast<uint32_t>(cjobs.size());
    std::vector<uint8_t> multi(nj, 0);  // the job's adapter has more than one job
    {
      uint32_t k = 0;
      for (const Seg& s : segs) {
        const uint32_t n_j = (static_cast<uint32_t>(s.toks.size()) + kJobTok - 1) / kJobTok;
        for (uint32_t q = 0; q < n_j; ++q) multi[k++] = n_j > 1;
      }
    }
    // One chunk list per launch: the jobs of the given projections (tagged
    // with their index in the launch) LPT-assigned to clusters by bytes
    // (heaviest first onto the least-loaded cluster, ties: lowest index).
    // exclude_hyb: leave out the jobs of the streaming share (hybrid launch)
    auto build = [&](ClusterWork& cw, const uint32_t* projs, uint32_t np, bool exclude_hyb = false) {
      cw = ClusterWork{};
      if (nj == 0) return;
      const uint32_t din = g.m.d_in[projs[0]], dout = g.m.d_out[projs[0]];
      cw.geom = cluster_geom(din, dout, st.device);
      std::vector<uint32_t> jo;  // work item w = job w % nj of projection w / nj
      for (uint32_t w = 0; w < nj * np; ++w)
        if ((!exclude_hyb || !cjob_hyb[w % nj]) && !cjob_route[w % nj]) jo.push_back(w);
      const uint32_t nw = static_cast<uint32_t>(jo.size());
      if (nw == 0) {
        cw.geom.n_clusters = 0;  // every job left this launch
        return;
      }
      const uint32_t nc = std::min(cw.geom.n_clusters, nw);
      cw.geom.n_clusters = nc;
      auto cost = [&](uint32_t w) {
        const ClusterJob& j = cjobs[w % nj];
        return static_cast<uint64_t>(j.rank + j.ntok) * (din + dout);
      };
      std::stable_sort(jo.begin(), jo.end(), [&](uint32_t a, uint32_t b) { return cost(a) > cost(b); });
      std::vector<uint64_t> load(nc, 0);
      std::vector<std::vector<uint32_t>> lists(nc);
      for (uint32_t w : jo) {
        const uint32_t c = static_cast<uint32_t>(std::min_element(load.begin(), load.end()) - load.begin());
        load[c] += cost(w);
        lists[c].push_back(w);
      }
      cw.chunks_off = static_cast<uint32_t>(cchunks.size());
      cw.cl_off = static_cast<uint32_t>(ccl_off.size());
      for (uint32_t c = 0; c < nc; ++c) {
        ccl_off.push_back(static_cast<uint32_t>(cchunks.size()) - cw.chunks_off);
        uint32_t jord = 0;
        for (uint32_t w : lists[c]) {
          const ClusterJob& j = cjobs[w % nj];
          const uint32_t this_job = jord++;
          for (uint32_t r0 = 0; r0 < j.rank; r0 += kChunkRows) {
            ClusterChunk ch{};
            ch.table_off = j.table_off;
            ch.rank = static_cast<uint16_t>(j.rank);
            ch.ntok = static_cast<uint8_t>(j.ntok);
            ch.proj = static_cast<uint8_t>(w / nj);
            ch.jord = this_job;
            for (uint32_t t = 0; t < kJobTok; ++t) ch.tok[t] = j.tok[t];
            ch.row0 = static_cast<uint16_t>(r0);
            ch.nrows = static_cast<uint8_t>(std::min(kChunkRows, j.rank - r0));
            ch.flags = static_cast<uint8_t>((r0 == 0 ? kChunkFirst : 0) |
                                            (r0 + kChunkRows >= j.rank ? kChunkLast : 0) |
                                            (multi[w % nj] ? kChunkReuse : 0));
            cchunks.push_back(ch);
          }
        }
        ccl_jobs.push_back(jord);
      }
      ccl_off.push_back(static_cast<uint32_t>(cchunks.size()) - cw.chunks_off);
      ccl_jobs.push_back(0);  // keeps ccl_jobs indexed like ccl_off
    };
    for (uint32_t p = 0; p < g.m.n_proj; ++p) build(cwork[p], &p, 1);
    n_layer_proj = 0;
    cwork_layer = ClusterWork{};
    bool same = g.m.n_proj > 1;
    for (uint32_t p = 1; p < g.m.n_proj; ++p)
      same = same && g.m.d_in[p] == g.m.d_in[0] && g.m.d_out[p] == g.m.d_out[0];
    if (same) {
      uint32_t all[PLORA_MAX_PROJ];
      for (uint32_t p = 0; p < g.m.n_proj; ++p) all[p] = p;
      build(cwork_layer, all, g.m.n_proj);
      n_layer_proj = g.m.n_proj;
      cwork_hyb = ClusterWork{};
      if (hyb_spare) build(cwork_hyb, all, g.m.n_proj, true);
    }
  }

  // ---- bf16 streaming BGMV (bgmv_stream.cu): jobs of <= s_jt tokens, S / E
  // items, list-scheduled over one CTA per SM
  stitems.clear();
  stcta.clear();
  for (uint32_t p = 0; p < PLORA_MAX_PROJ; ++p) swork[p] = StreamWork{};
  swork_layer = StreamWork{};
  s_njobs = 0;
  s_vplane = 0;
  if (es == 2) {
    s_jt = seg_maxtok > 4 ? 8 : 4;
    struct SJob {
      uint32_t rank, table_off, ntok, v_off, tok[8];
      uint8_t hyb;  // the adapter belongs to the hybrid launch's streaming share
    };
    std::vector<SJob> jobs;
    uint64_t voff = 0;
    for (uint32_t si : order) {  // largest rank first
      const Seg& sg = segs[si];
      if (seg_route[si]) continue;
      for (uint32_t tc = 0; tc < sg.toks.size(); tc += s_jt) {
        SJob j{};
        j.rank = sg.rank;
        j.table_off = sg.table_off;
        j.ntok = std::min<uint32_t>(s_jt, static_cast<uint32_t>(sg.toks.size()) - tc);
        for (uint32_t t = 0; t < j.ntok; ++t) j.tok[t] = sg.toks[tc + t];
        j.v_off = static_cast<uint32_t>(voff);
        j.hyb = seg_hyb[si];
        voff += static_cast<uint64_t>((sg.rank + 15) & ~15u) * s_jt;  // rows padded to 16 (kept zero)
        jobs.push_back(j);
      }
    }
    if (voff > 0xffffffffull) throw ValidationError("batch too large for one plan");
    s_njobs = static_cast<uint32_t>(jobs.size());
    s_vplane = (voff + 3) & ~3ull;
    const uint32_t max_ctas = stream_max_ctas(st.device, s_jt);
    auto build_sw = [&](StreamWork& w, const uint32_t* projs, uint32_t np, uint32_t cta_cap = 0,
                        bool only_hyb = false) {
      w = StreamWork{};
      w.np = np;
      for (uint32_t i = 0; i < np; ++i) w.projs[i] = projs[i];
      if (jobs.empty()) return;
      const uint32_t din = g.m.d_in[projs[0]], dout = g.m.d_out[projs[0]];
      const uint32_t ne = (dout + kStreamKC - 1) / kStreamKC;
      // cost model: bytes streamed per SM (x / y rows counted at L2 / HBM
      // weight) plus a fixed per-item overhead
      const double ovh = 4096.0;
      struct Cand {
        StreamItem it;
        double cost;
        uint32_t key;  // job · np + launch projection
      };
      std::vector<Cand> sc, ec;
      for (uint32_t jn = 0; jn < jobs.size(); ++jn) {
        const SJob& j = jobs[jn];
        if (only_hyb && !j.hyb) continue;
        const uint32_t ns = j.rank * j.ntok;  // v elements: each released on its own
        for (uint32_t i = 0; i < np; ++i) {
          StreamItem base{};
          base.job = jn;
          base.table_off = j.table_off;
          base.rank_ntok = j.rank | (j.ntok << 16);
          base.v_off = j.v_off;
          base.ns_ne = ns | (ne << 16);
          for (uint32_t t = 0; t < 8; ++t) base.tok[t] = t < j.ntok ? j.tok[t] : 0u;
          for (uint32_t r0 = 0; r0 < j.rank; r0 += 16) {
            Cand c{base, 0.0, jn * np + i};
            c.it.kind = i;
            c.it.off = r0;
            c.it.n = std::min<uint32_t>(16, j.rank - r0);
            c.cost = 2.0 * c.it.n * din + 1.0 * j.ntok * din + ovh;
            sc.push_back(c);
          }
          for (uint32_t c0 = 0; c0 < dout; c0 += kStreamKC) {
            Cand c{base, 0.0, jn * np + i};
            c.it.kind = kStreamExpand | i;
            c.it.off = c0;
            c.it.n = std::min<uint32_t>(kStreamKC, dout - c0);
            c.cost = 2.0 * j.rank * c.it.n + 4.0 * j.ntok * c.it.n + ovh;
            ec.push_back(c);
          }
        }
      }
      if (sc.empty() && ec.empty()) return;
      const uint32_t ctas = std::min<uint32_t>(cta_cap ? std::min(cta_cap, max_ctas) : max_ctas,
                                               static_cast<uint32_t>(sc.size() + ec.size()));
      std::vector<double> load(ctas, 0.0);
      std::vector<std::vector<uint32_t>> lists_s(ctas), lists_e(ctas);
      std::vector<double> ready(jobs.size() * np, 0.0);
      using Load = std::pair<double, uint32_t>;
      std::priority_queue<Load, std::vector<Load>, std::greater<Load>> heap;
      for (uint32_t c = 0; c < ctas; ++c) heap.emplace(0.0, c);
      for (uint32_t k = 0; k < sc.size(); ++k) {  // S items in job order onto the least-loaded CTA
        Load l = heap.top();
        heap.pop();
        const double fin = l.first + sc[k].cost;
        lists_s[l.second].push_back(k);
        ready[sc[k].key] = std::max(ready[sc[k].key], fin);
        heap.emplace(fin, l.second);
      }
      // E items by the simulated readiness of their job (the producer runs
      // about a ring ahead of the consumers: margin), heaviest first
      const double margin = 160.0 * 1024;
      std::vector<uint32_t> eo(ec.size());
      std::iota(eo.begin(), eo.end(), 0u);
      std::stable_sort(eo.begin(), eo.end(), [&](uint32_t a, uint32_t b) {
        const double ra = ready[ec[a].key], rb = ready[ec[b].key];
        return ra != rb ? ra < rb : ec[a].cost > ec[b].cost;
      });
      for (uint32_t k : eo) {
        Load l = heap.top();
        heap.pop();
        const double start = std::max(l.first, ready[ec[k].key] + margin);
        lists_e[l.second].push_back(k);
        heap.emplace(start + ec[k].cost, l.second);
      }
      w.items_off = static_cast<uint32_t>(stitems.size());
      w.cta_off = static_cast<uint32_t>(stcta.size());
      w.ctas = ctas;
      uint32_t n = 0;
      for (uint32_t c = 0; c < ctas; ++c) {
        stcta.push_back(n);
        for (uint32_t k : lists_s[c]) stitems.push_back(sc[k].it);
        for (uint32_t k : lists_e[c]) stitems.push_back(ec[k].it);
        n += static_cast<uint32_t>(lists_s[c].size() + lists_e[c].size());
      }
      stcta.push_back(n);
    };
    for (uint32_t p = 0; p < g.m.n_proj; ++p) build_sw(swork[p], &p, 1);
    bool same = g.m.n_proj > 1;
    for (uint32_t p = 1; p < g.m.n_proj; ++p)
      same = same && g.m.d_in[p] == g.m.d_in[0] && g.m.d_out[p] == g.m.d_out[0];
    if (same) {
      uint32_t all[PLORA_MAX_PROJ];
      for (uint32_t p = 0; p < g.m.n_proj; ++p) all[p] = p;
      build_sw(swork_layer, all, g.m.n_proj);
      swork_hyb = StreamWork{};
      if (hyb_spare) build_sw(swork_hyb, all, g.m.n_proj, hyb_spare, true);
    }
  }

  // ---- bf16 warp-item BGMV (bgmv_warp.cu, the default decode op): jobs of
  // <= 4 tokens (an adapter's tokens split evenly over ceil(n / 4) jobs),
  // S items of kWarpRows rank rows, E items of kWarpCols output columns
  witems.clear();
  for (uint32_t p = 0; p < PLORA_MAX_PROJ; ++p) wwork[p] = WarpWork{};
  wwork_layer = WarpWork{};
  uint64_t wv_need = 0;
  if (es == 2) {
    struct WJob {
      uint32_t rank, table_off, ntok, tok[kWarpJobTok];
    };
    std::vector<WJob> wj;
    for (uint32_t si : order) {  // largest rank first
      const Seg& sg = segs[si];
      if (seg_route[si]) continue;
      const uint32_t nt = static_cast<uint32_t>(sg.toks.size()), nj = (nt + kWarpJobTok - 1) / kWarpJobTok;
      uint32_t t0 = 0;
      for (uint32_t q = 0; q < nj; ++q) {
        WJob j{sg.rank, sg.table_off, nt / nj + (q < nt % nj ? 1u : 0u), {}};
        for (uint32_t t = 0; t < j.ntok; ++t) j.tok[t] = sg.toks[t0 + t];
        t0 += j.ntok;
        wj.push_back(j);
      }
    }
    auto build_w = [&](WarpWork& w, const uint32_t* projs, uint32_t np) {
      w = WarpWork{};
      w.np = np;
      for (uint32_t i = 0; i < np; ++i) w.projs[i] = projs[i];
      if (wj.empty()) return;
      // K slices of the S items: 1 (splitting a 4096-wide 8-row item in two
      // measured slower for the 32-layer step, 0.339 vs 0.320 ms of shrink,
      // and barely faster per layer, profiles/r02n_warp_variants.txt)
      w.ks = 1;
      // K slices of <= 4096 inputs (16 chunks of 512 bytes per lane row):
      // 8-row items of at most 64 KiB, so wide layers still give every SM
      // several items (cfg5's 8192-wide q / v: two slices)
      w.ks = (g.m.d_in[projs[0]] + 4095) / 4096;
      uint64_t voff = 0;
      std::vector<WarpItem> S, E, E1, EP;  // E: multi-layer; E1 + EP (split pairs): single-layer
      for (uint32_t i = 0; i < np; ++i) {
        const uint32_t dout = g.m.d_out[projs[i]];
        for (const WJob& j : wj) {
          WarpItem base{};
          base.table_off = j.table_off;
          base.v_off = static_cast<uint32_t>(voff);
          for (uint32_t t = 0; t < kWarpJobTok; ++t) base.tok[t] = t < j.ntok ? j.tok[t] : 0u;
          auto meta = [&](uint32_t n) { return j.rank | (j.ntok << 9) | (i << 12) | (n << 16); };
          const uint32_t R = kWarpRows(j.ntok), C = kWarpCols(j.ntok);
          for (uint32_t k = 0; k < w.ks; ++k)
            for (uint32_t r0 = 0; r0 < j.rank; r0 += R) {
              WarpItem it = base;
              it.meta = meta(std::min(R, j.rank - r0));
              it.off = r0 | (k << 16);
              S.push_back(it);
            }
          for (uint32_t c0 = 0; c0 < dout; c0 += C) {
            WarpItem it = base;
            it.meta = meta(std::min(C, dout - c0));
            it.off = c0;
            E.push_back(it);
            if (j.rank >= kWarpSplitRows) {  // a pair: rows [0, h) and [h, r), one CTA
              it.meta |= kWarpSplit;
              EP.push_back(it);
              it.meta |= kWarpSecond;
              EP.push_back(it);
            } else {
              E1.push_back(it);
            }
          }
          voff += static_cast<uint64_t>(w.ks) * j.ntok * j.rank;
        }
      }
      if (voff > 0xffffffffull) throw ValidationError("batch too large for one plan");
      // heaviest items first (the hardware block scheduler then fills the
      // tail with the light ones); ties keep list order, so a job's items stay
      // adjacent and share x / v through L1
      auto s_cost = [](const WarpItem& it) { return it.meta >> 16; };
      auto e_cost = [](const WarpItem& it) { return (it.meta & 0x1ffu) * ((it.meta >> 16) & 0x3ffu); };
      std::stable_sort(S.begin(), S.end(), [&](const WarpItem& a, const WarpItem& b) { return s_cost(a) > s_cost(b); });
      std::stable_sort(E.begin(), E.end(), [&](const WarpItem& a, const WarpItem& b) { return e_cost(a) > e_cost(b); });
      std::stable_sort(E1.begin(), E1.end(), [&](const WarpItem& a, const WarpItem& b) { return e_cost(a) > e_cost(b); });
      {  // split pairs first, heaviest first, each pair on an even position (one CTA of two warps)
        std::vector<uint32_t> pi(EP.size() / 2);
        std::iota(pi.begin(), pi.end(), 0u);
        std::stable_sort(pi.begin(), pi.end(),
                         [&](uint32_t a, uint32_t b) { return e_cost(EP[2 * a]) > e_cost(EP[2 * b]); });
        std::vector<WarpItem> all;
        all.reserve(EP.size() + E.size());
        for (uint32_t k : pi) {
          all.push_back(EP[2 * k]);
          all.push_back(EP[2 * k + 1]);
        }
        all.insert(all.end(), E1.begin(), E1.end());
        E1.swap(all);
      }
      w.s_off = static_cast<uint32_t>(witems.size());
      w.ns = static_cast<uint32_t>(S.size());
      witems.insert(witems.end(), S.begin(), S.end());
      w.e_off = static_cast<uint32_t>(witems.size());
      w.ne = static_cast<uint32_t>(E.size());
      witems.insert(witems.end(), E.begin(), E.end());
      w.e1_off = static_cast<uint32_t>(witems.size());
      w.ne1 = static_cast<uint32_t>(E1.size());
      witems.insert(witems.end(), E1.begin(), E1.end());
      w.vplane = (voff + 3) & ~3ull;
      wv_need = std::max(wv_need, w.vplane);
    };
    for (uint32_t p = 0; p < g.m.n_proj; ++p) build_w(wwork[p], &p, 1);
    bool same_in = g.m.n_proj > 1;
    for (uint32_t p = 1; p < g.m.n_proj; ++p) same_in = same_in && g.m.d_in[p] == g.m.d_in[0];
    if (same_in) {
      uint32_t all[PLORA_MAX_PROJ];
      for (uint32_t p = 0; p < g.m.n_proj; ++p) all[p] = p;
      build_w(wwork_layer, all, g.m.n_proj);
    }
    wv_need *= g.m.n_layers;  // a multi-layer launch keeps one plane per layer
  }

  // ---- upload the device-side work lists in one copy from a pinned
  // staging buffer (cluster chunk offsets travel as kernel parameters)
  auto align = [](uint64_t v) { return (v + 255) & ~255ull; };
  struct Part {
    const void* src;
    uint64_t bytes;
    void** dst;
  };
  const Part parts[] = {
      {units.data(), units.size() * sizeof(BgmvUnit), reinterpret_cast<void**>(&d_units)},
      {tiles.data(), tiles.size() * sizeof(SgmvTile), reinterpret_cast<void**>(&d_tiles)},
      {gtiles.data(), gtiles.size() * sizeof(GemmTile), reinterpret_cast<void**>(&d_gtiles)},
      {cchunks.data(), cchunks.size() * sizeof(ClusterChunk), reinterpret_cast<void**>(&d_cchunks)},
      {cjobs.data(), cjobs.size() * sizeof(ClusterJob), reinterpret_cast<void**>(&d_cjobs)},
      {sitems.data(), sitems.size() * sizeof(SgmvItem), reinterpret_cast<void**>(&d_sitems)},
      {scta.data(), scta.size() * sizeof(uint32_t), reinterpret_cast<void**>(&d_scta)},
      {stitems.data(), stitems.size() * sizeof(StreamItem), reinterpret_cast<void**>(&d_stitems)},
      {stcta.data(), stcta.size() * sizeof(uint32_t), reinterpret_cast<void**>(&d_stcta)},
      {route_perm.data(), route_perm.size() * sizeof(uint32_t), reinterpret_cast<void**>(&d_route_perm)},
      {witems.data(), witems.size() * sizeof(WarpItem), reinterpret_cast<void**>(&d_witems)},
  };
  uint64_t total = 0;
  for (const Part& pt : parts) total += align(pt.bytes);
  total = std::max<uint64_t>(total, 256);
  DeviceCtx ctx(st.device);
  if (upload_done) PLORA_CUDA(cudaEventSynchronize(upload_done));  // pinned buffer reuse
  if (h_cap < total) {
    if (h_pinned) cudaFreeHost(h_pinned);
    h_pinned = nullptr;
    PLORA_CUDA(cudaMallocHost(&h_pinned, total));
    h_cap = total;
  }
  if (d_cap < total) {
    if (d_buf) {
      PLORA_CUDA(cudaStreamSynchronize(stream));
      cudaFree(d_buf);
    }
    d_buf = nullptr;
    PLORA_CUDA(cudaMalloc(&d_buf, total));
    d_cap = total;
  }
  uint64_t off = 0;
  for (const Part& pt : parts) {
    if (pt.bytes) std::memcpy(h_pinned + off, pt.src, pt.bytes);
    *pt.dst = d_buf + off;
    off += align(pt.bytes);
  }
  PLORA_CUDA(cudaMemcpyAsync(d_buf, h_pinned, total, cudaMemcpyHostToDevice, stream));
  if (!upload_done) PLORA_CUDA(cudaEventCreateWithFlags(&upload_done, cudaEventDisableTiming));
  PLORA_CUDA(cudaEventRecord(upload_done, stream));

  if (v_cap < std::max<uint64_t>(v_elems, 1)) {
    if (d_v) {
      PLORA_CUDA(cudaStreamSynchronize(stream));
      cudaFree(d_v);
    }
    d_v = nullptr;
    v_cap = std::max<uint64_t>(v_elems, 4096);
    PLORA_CUDA(cudaMalloc(&d_v, v_cap * sizeof(float)));
  }
  if (wv_cap < wv_need) {  // warp-item BGMV v planes
    if (d_wv) {
      PLORA_CUDA(cudaStreamSynchronize(stream));
      cudaFree(d_wv);
    }
    d_wv = nullptr;
    wv_cap = wv_need;
    PLORA_CUDA(cudaMalloc(&d_wv, wv_cap * sizeof(float)));
  }
  if (es == 2 && n_tiles > 0) {  // SGMV workspaces (see sgmv.cu)
    // one region per projection (plora_sgmv_layer keeps both in flight)
    uint64_t parts = ssched_layer.splits;
    for (uint32_t p = 0; p < g.m.n_proj; ++p)
      parts = std::max<uint64_t>(parts, ssched[p].splits);
    vpart_parts = static_cast<uint32_t>(parts);
    const uint64_t need_part = g.m.n_proj * parts * n_tiles * 128ull * 128ull;
    const uint64_t need_vbuf = g.m.n_proj * n_tiles * 128ull * 128ull * 2ull;
    if (vpart_cap < need_part || vbuf_cap < need_vbuf) {
      PLORA_CUDA(cudaStreamSynchronize(stream));
      cudaFree(d_vpart);
      cudaFree(d_vbuf);
      d_vpart = nullptr;
      d_vbuf = nullptr;
      vpart_cap = need_part;
      vbuf_cap = need_vbuf;
      PLORA_CUDA(cudaMalloc(&d_vpart, vpart_cap * sizeof(float)));
      PLORA_CUDA(cudaMalloc(&d_vbuf, vbuf_cap));
    }
  }
  if (es == 2 && s_njobs > 0) {  // streaming BGMV: v planes and counters for every (layer, proj)
    const uint64_t planes = static_cast<uint64_t>(g.m.n_layers) * g.m.n_proj;
    const uint64_t need_v = planes * s_vplane, need_c = planes * 2ull * s_njobs;
    if (sv_cap < need_v || scnt_cap < need_c) {
      PLORA_CUDA(cudaStreamSynchronize(stream));
      cudaFree(d_sv);
      cudaFree(d_scnt);
      d_sv = nullptr;
      d_scnt = nullptr;
      sv_cap = std::max(need_v, sv_cap);
      scnt_cap = std::max(need_c, scnt_cap);
      PLORA_CUDA(cudaMalloc(&d_sv, sv_cap * sizeof(float)));
      PLORA_CUDA(cudaMalloc(&d_scnt, scnt_cap * sizeof(uint32_t)));
      // v pad rows (rank .. rank rounded up to 16) are never written: zero them once
      PLORA_CUDA(cudaMemsetAsync(d_sv, 0, sv_cap * sizeof(float), stream));
    }
    // every call leaves the counters at zero; a rebuilt plan starts from zero too
    PLORA_CUDA(cudaMemsetAsync(d_scnt, 0, need_c * sizeof(uint32_t), stream));
  }
  if (sync_cap < 2ull + n_seg) {
    if (d_sync) {
      PLORA_CUDA(cudaStreamSynchronize(stream));
      cudaFree(d_sync);
    }
    d_sync = nullptr;
    sync_cap = std::max<uint64_t>(2ull + n_seg, 1024);
    PLORA_CUDA(cudaMalloc(&d_sync, sync_cap * sizeof(uint32_t)));
    PLORA_CUDA(cudaMemsetAsync(d_sync, 0, sync_cap * sizeof(uint32_t), stream));
  }
}

extern "C" {

int plora_plan_create(plora_store* s, const int32_t* token_adapter, uint32_t n_tokens,
                      plora_stream_t stream, plora_plan** out) {
  return guard([&] {
    if (!s) throw ValidationError("null store");
    if (n_tokens && !token_adapter) throw ValidationError("null token_adapter");
    auto plan = std::make_unique<plora_plan>();
    plan->store = s;
    plan->build(token_adapter, n_tokens, static_cast<cudaStream_t>(stream));
    *out = plan.release();
    return 0;
  });
}

int plora_plan_update(plora_plan* plan, const int32_t* token_adapter, uint32_t n_tokens,
                      plora_stream_t stream) {
  return guard([&] {
    if (!plan) throw ValidationError("null plan");
    if (n_tokens && !token_adapter) throw ValidationError("null token_adapter");
    plan->build(token_adapter, n_tokens, static_cast<cudaStream_t>(stream));
    return 0;
  });
}

void plora_plan_destroy(plora_plan* plan) {
  if (!plan) return;
  DeviceCtx ctx(plan->store->device);
  if (plan->upload_done) {
    cudaEventSynchronize(plan->upload_done);
    cudaEventDestroy(plan->upload_done);
  }
  cudaDeviceSynchronize();
  plan->drop_tp();
  if (plan->route) plora_plan_destroy(plan->route);
  cudaFree(plan->d_route_ws);
  if (plan->route_stream) cudaStreamDestroy(plan->route_stream);
  if (plan->ev_rfork) cudaEventDestroy(plan->ev_rfork);
  if (plan->ev_rjoin) cudaEventDestroy(plan->ev_rjoin);
  cudaFreeHost(plan->h_pinned);
  cudaFree(plan->d_buf);
  cudaFree(plan->d_v);
  cudaFree(plan->d_sv);
  cudaFree(plan->d_scnt);
  cudaFree(plan->d_wv);
  if (plan->aux_stream) cudaStreamDestroy(plan->aux_stream);
  if (plan->ev_fork) cudaEventDestroy(plan->ev_fork);
  if (plan->ev_join) cudaEventDestroy(plan->ev_join);
  cudaFree(plan->d_sync);
  cudaFree(plan->d_vpart);
  cudaFree(plan->d_vbuf);
  delete plan;
}

uint32_t plora_plan_num_segments(const plora_plan* plan) { return plan ? plan->n_seg : 0; }

}  // extern "C"
