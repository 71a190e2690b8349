// Scheduler: logical fused ops -> physical steps (§Multi-GPU).
//
//  * SWAP ops are executed by relabelling the logical->physical qubit map (no data
//    movement; SURVEY §8(c) item 12 allows the GPU to drop IQFT swaps this way as long
//    as the final logical state is identical — all readout goes through the map).
//  * Multi-GPU ("PGAS-based SHMEM", "minimize unnecessary data
//    migration"): the top g physical bits are global. An op whose
//    non-diagonal target sits on a global bit first gets an Exchange step that swaps
//    that global bit with a local bit chosen by farthest next use (Belady); controls,
//    diagonal qubits and reciprocal clock bits on global bits never move data.
//  * Tile passes: consecutive ops whose non-diagonal targets fit in a
//    T-qubit local set are executed in ONE HBM pass: each CTA stages the 2^T amplitudes
//    spanned by the set (padded with the lowest bits for coalescing) in shared memory,
//    applies all ops, and writes back. Without tiles, every op is one streaming pass.
#include <algorithm>
#include <cmath>
#include <map>
#include <numeric>
#include <cstdlib>
#include <set>
#include <sstream>

#include "jit.h"
#include "sv_internal.h"

namespace hhlsv {

// Non-diagonal targets of an op (the bits whose values it mixes).
static std::vector<int> nd_targets(const Gate &g) {
    switch (g.kind) {
        case Kind::Dense:
        case Kind::Controlled:
        case Kind::RecipRY: return g.targets;
        default: return {};
    }
}

static Gate to_physical(const Gate &g, const std::vector<int> &phys) {
    Gate p = g;
    for (int &q : p.targets) q = phys[q];
    for (int &q : p.controls) q = phys[q];
    return p;
}

// Qubits an op acts on NON-diagonally (mixes) and diagonally (controls, phase qubits).
static void roles(const Gate &g, std::vector<int> &nd, std::vector<int> &dg) {
    nd.clear();
    dg.clear();
    switch (g.kind) {
        case Kind::Dense: nd = g.targets; break;
        case Kind::Controlled: nd = g.targets; dg = g.controls; break;
        case Kind::Diagonal: dg = g.targets; break;
        case Kind::RecipRY: nd = g.targets; dg = g.controls; break;
        case Kind::Swap: nd = g.targets; break;
    }
}

// Commutation-aware reordering for tile packing. Two ops must keep their
// relative order iff they share a qubit that at least one of them acts on non-diagonally (ops
// on disjoint qubits commute; diagonal actions — controls, phases — commute with each other).
// Greedy list scheduling then fills each T-qubit pass with every ready op whose non-diagonal
// targets still fit, so e.g. the final Hadamard layer is absorbed into the QFT passes instead
// of needing passes of its own. Returns a topological order of `ops` (the state is unchanged
// up to rounding: only commuting ops are exchanged).
// Multi-rank (nloc < n): an op whose non-diagonal target sits on a global bit needs an exchange.
// Such ops are deferred while any other op is ready, so every op that commutes with them runs
// first (e.g. the final Hadamard layer on the clock register before the system register's V, which
// then needs ONE exchange round whose victims -- qubits with no further use -- never come back).
static std::vector<Gate> reorder_for_tiles(const std::vector<Gate> &ops, const std::vector<int> &phys, int T,
                                           int wmin, int R, int nloc) {
    const size_t m = ops.size();
    std::vector<std::vector<size_t>> succ(m);
    std::vector<int> indeg(m, 0);
    {
        std::vector<std::vector<int>> ndv(m), dgv(m);
        for (size_t i = 0; i < m; i++) roles(ops[i], ndv[i], dgv[i]);
        const int nq = (int)phys.size();
        // per qubit: last non-diagonal user, and diagonal users since then
        std::vector<long> last_nd(nq, -1);
        std::vector<std::vector<size_t>> diag_since(nq);
        auto edge = [&](size_t a, size_t b) {
            if (a == b) return;
            succ[a].push_back(b);
            indeg[b]++;
        };
        for (size_t i = 0; i < m; i++) {
            for (int q : ndv[i]) {
                if (last_nd[q] >= 0) edge((size_t)last_nd[q], i);
                for (size_t d : diag_since[q]) edge(d, i);
            }
            for (int q : dgv[i])
                if (last_nd[q] >= 0) edge((size_t)last_nd[q], i);
            for (int q : ndv[i]) {
                last_nd[q] = (long)i;
                diag_since[q].clear();
            }
            for (int q : dgv[i]) diag_since[q].push_back(i);
        }
        for (auto &v : succ) {
            std::sort(v.begin(), v.end());
            v.erase(std::unique(v.begin(), v.end()), v.end());
        }
        std::fill(indeg.begin(), indeg.end(), 0);
        for (auto &v : succ)
            for (size_t b : v) indeg[b]++;
    }
    auto pnd = [&](const Gate &g) {
        std::vector<int> nd, dg;
        roles(g, nd, dg);
        for (int &q : nd) q = phys[q];
        return nd;
    };
    // a pass holds at most T tile bits, at most T - wmin of them above the wmin always-held low bits;
    // tested on bit masks of physical bits (< 64): the greedy packing below tests every ready op
    // against the open pass many times
    std::vector<uint64_t> ndm(m, 0);
    for (size_t i = 0; i < m; i++)
        for (int b : pnd(ops[i])) ndm[i] |= 1ull << b;
    const uint64_t lowm = wmin >= 64 ? ~0ull : ((1ull << wmin) - 1ull);
    auto fitsm = [&](uint64_t u) {
        return __builtin_popcountll(u) <= T && __builtin_popcountll(u & ~lowm) <= T - wmin;
    };
    std::vector<char> needs_global(m, 0);
    for (size_t i = 0; i < m; i++)
        for (int b : pnd(ops[i]))
            if (b >= nloc) needs_global[i] = 1;
    bool exchanged = false;        // after the first global op the layout changes: stop deferring
    const int dalap = jit_config().dalap;      // passes (from the first) that place diagonals ALAP
    int pass_no = 0;
    std::vector<Gate> out;
    out.reserve(m);
    std::vector<char> done(m, 0);
    std::set<size_t> ready;
    for (size_t i = 0; i < m; i++)
        if (indeg[i] == 0) ready.insert(i);
    auto take = [&](size_t i) {
        done[i] = 1;
        ready.erase(i);
        out.push_back(ops[i]);
        for (size_t b : succ[i])
            if (--indeg[b] == 0) ready.insert(b);
    };
    while (!ready.empty()) {
        if (!exchanged) {
            bool other = false;
            for (size_t i : ready) other |= !needs_global[i];
            if (!other) {              // only exchange-needing ops are ready: take one, stop deferring
                exchanged = true;
                take(*ready.begin());
                continue;
            }
        }
        // a swap or an op too wide for a tile is scheduled alone, in original order
        size_t first = *ready.begin();
        if (!exchanged)
            for (size_t i : ready)
                if (!needs_global[i]) {
                    first = i;
                    break;
                }
        const Gate &g0 = ops[first];
        if (g0.kind == Kind::Swap ||
            ((g0.kind == Kind::Dense || g0.kind == Kind::Controlled) && (int)g0.targets.size() > R)) {
            take(first);
            continue;
        }
        uint64_t cur = 0;
        const bool dalap_now = pass_no++ < dalap;
        for (;;) {
            // pick the ready op that adds the fewest new tile bits (free ones first), then the
            // earliest in circuit order: keeps room in the pass for ops that become ready later
            size_t best = SIZE_MAX;
            int best_new = 1 << 20;
            uint64_t best_u = 0;
            for (size_t i : ready) {
                const Gate &g = ops[i];
                if (g.kind == Kind::Swap ||
                    ((g.kind == Kind::Dense || g.kind == Kind::Controlled) && (int)g.targets.size() > R))
                    continue;
                if (!exchanged && needs_global[i]) continue;
                const uint64_t u = cur | ndm[i];
                const int nnew = __builtin_popcountll(ndm[i] & ~cur);
                if (!fitsm(u)) continue;
                if (dalap_now && g.kind == Kind::Diagonal) continue;    // considered below
                if (nnew < best_new) {
                    best = i;
                    best_new = nnew;
                    best_u = u;
                    if (nnew == 0) break;      // ready is ordered: the earliest free op
                }
            }
            if (best == SIZE_MAX && dalap_now) {
                // diagonals as late as possible: one is taken only when no non-diagonal op fits and it
                // unblocks a non-diagonal op that fits this pass (or only diagonals are left)
                bool any_nd = false;
                for (size_t i : ready) any_nd |= ops[i].kind != Kind::Diagonal;
                for (size_t i : ready) {
                    if (ops[i].kind != Kind::Diagonal) continue;
                    bool use = !any_nd;
                    for (size_t sb : succ[i]) {
                        if (use) break;
                        if (indeg[sb] != 1 || ops[sb].kind == Kind::Swap) continue;
                        if (!exchanged && needs_global[sb]) continue;
                        use = fitsm(cur | ndm[sb]);
                    }
                    if (use) {
                        best = i;
                        best_u = cur;
                        break;
                    }
                }
            }
            if (best == SIZE_MAX) break;
            cur = best_u;
            take(best);
        }
        // pass boundary: the in-order packer below re-derives the same passes from this order
    }
    if (out.size() != m) fail(SV_E_ARG, "internal: dependency cycle in reorder_for_tiles");
    return out;
}

// Register phases of one tile pass. Ops inside a phase run on the 16 amplitudes a
// thread holds in registers, spanned by <= R register bits; a phase boundary costs a round trip of
// the tile through shared memory plus a barrier. The ops are list-scheduled over their commutation
// DAG (same rule as reorder_for_tiles): the current phase takes the ready op that adds the fewest
// new register bits (diagonal ops add none), the earliest on ties; when nothing fits, a new phase
// starts. E.g. the final Hadamard layer joins the QFT phases instead of trailing in phases of its own.
static void phase_schedule(std::vector<Gate> &ops, int R, std::vector<std::vector<int>> &phase_R,
                           std::vector<size_t> &phase_start) {
    const size_t m = ops.size();
    std::vector<std::vector<size_t>> succ(m);
    std::vector<int> indeg(m, 0);
    std::vector<std::vector<int>> ndv(m), dgv(m);
    for (size_t i = 0; i < m; i++) roles(ops[i], ndv[i], dgv[i]);
    {
        std::map<int, long> last_nd;
        std::map<int, std::vector<size_t>> diag_since;
        auto edge = [&](size_t a, size_t b) {
            if (a != b) succ[a].push_back(b);
        };
        for (size_t i = 0; i < m; i++) {
            for (int q : ndv[i]) {
                auto it = last_nd.find(q);
                if (it != last_nd.end()) edge((size_t)it->second, i);
                for (size_t d : diag_since[q]) edge(d, i);
            }
            for (int q : dgv[i]) {
                auto it = last_nd.find(q);
                if (it != last_nd.end()) edge((size_t)it->second, i);
            }
            for (int q : ndv[i]) {
                last_nd[q] = (long)i;
                diag_since[q].clear();
            }
            for (int q : dgv[i]) diag_since[q].push_back(i);
        }
        for (auto &v : succ) {
            std::sort(v.begin(), v.end());
            v.erase(std::unique(v.begin(), v.end()), v.end());
            for (size_t b : v) indeg[b]++;
        }
    }
    std::set<size_t> ready;
    for (size_t i = 0; i < m; i++)
        if (indeg[i] == 0) ready.insert(i);
    std::vector<Gate> out;
    out.reserve(m);
    std::vector<int> cur;
    phase_R.clear();
    phase_start.clear();
    while (!ready.empty()) {
        size_t best = SIZE_MAX;
        int best_new = 1 << 20;
        for (size_t i : ready) {
            int nnew = 0;
            for (int b : ndv[i])
                if (std::find(cur.begin(), cur.end(), b) == cur.end()) nnew++;
            if ((int)cur.size() + nnew > R) continue;
            if (nnew < best_new) {
                best = i;
                best_new = nnew;
                if (nnew == 0) break;
            }
        }
        if (best == SIZE_MAX) {          // nothing fits: close the phase
            phase_R.push_back(cur);
            cur.clear();
            continue;
        }
        if (out.empty() || phase_start.size() == phase_R.size()) phase_start.push_back(out.size());
        for (int b : ndv[best])
            if (std::find(cur.begin(), cur.end(), b) == cur.end()) cur.push_back(b);
        out.push_back(ops[best]);
        ready.erase(best);
        for (size_t b : succ[best])
            if (--indeg[b] == 0) ready.insert(b);
    }
    if (out.size() != m) fail(SV_E_ARG, "internal: dependency cycle in phase_schedule");
    phase_R.push_back(cur);
    phase_start.push_back(m);
    ops = std::move(out);
}

// Diagonal fusion after scheduling: inside a register phase, consecutive diagonal ops (they
// commute, and the phase scheduler groups every ready one) become one table of <= kmax qubits:
// one lookup + one complex multiply per amplitude for the group (table built on the host).
static void merge_phase_diagonals(Step &tile, int kmax) {
    std::vector<Gate> out;
    std::vector<size_t> starts;
    for (size_t p = 0; p + 1 < tile.phase_start.size(); p++) {
        starts.push_back(out.size());
        bool open = false;
        for (size_t oi = tile.phase_start[p]; oi < tile.phase_start[p + 1]; oi++) {
            Gate &g = tile.tile_ops[oi];
            if (g.kind == Kind::Diagonal && open && merge_diagonal(out.back(), g, kmax)) continue;
            open = g.kind == Kind::Diagonal;
            out.push_back(std::move(g));
        }
    }
    starts.push_back(out.size());
    tile.tile_ops = std::move(out);
    tile.phase_start = std::move(starts);
}

Schedule compile(const std::vector<Gate> &ops_in, const std::vector<ProductFactor> *init, int n, int nloc,
                 const std::vector<int> &phys_in, const CompileOptions &o) {
    Schedule s;
    std::vector<int> phys = phys_in;
    const double local_amps = std::ldexp(1.0, nloc);
    if (init) {
        Step st;
        st.kind = StepKind::InitProduct;
        st.factors = *init;
        for (auto &f : st.factors)
            for (int &q : f.qubits) q = phys[q];
        st.bytes = 16.0 * local_amps;
        s.steps.push_back(std::move(st));
        s.pass_bytes += 16.0 * local_amps;
        s.n_passes++;
    }
    const int T = std::min(o.tile_qubits, nloc);
    // register bits per phase: o.reg_bits (3 or 4) by default; a pass holding a 4-target op uses 4
    const int RMAX = 4;
    const bool tiles = o.tile_qubits > 0 && nloc >= RMAX + 1;
    int wmin_opt = o.wmin;   // default 3 (128-byte segments): more tile bits for op targets per pass
    if (jit_config().wmin != 3) wmin_opt = jit_config().wmin;     // developer experiments (HHLSV_JIT=wmin=..)
    const int wmin = std::min(wmin_opt, T - RMAX);
    const int R = RMAX;                 // widest op a tile pass can hold in registers
    // single-rank tile schedules: commutation-aware reordering for packing (multi-rank keeps the
    // input order so exchanges follow the circuit)
    const bool reorder = tiles && o.reorder;
    const std::vector<Gate> ops = reorder ? reorder_for_tiles(ops_in, phys_in, T, wmin, R, nloc) : ops_in;
    prof_mark("    compile: reorder");

    // Precompute, for Belady eviction, the op index list per logical qubit used as nd target.
    std::vector<std::vector<size_t>> uses(n);
    for (size_t i = 0; i < ops.size(); i++)
        for (int q : nd_targets(ops[i])) uses[q].push_back(i);
    auto next_use = [&](int logical, size_t from) -> size_t {
        auto &u = uses[logical];
        auto it = std::lower_bound(u.begin(), u.end(), from);
        return it == u.end() ? SIZE_MAX : *it;
    };

    Step tile;
    bool tile_open = false;
    std::vector<int> tile_nd;    // physical nd bits of the open tile
    auto close_tile = [&]() {
        if (!tile_open) return;
        // local set: nd bits, filled with the lowest local bits for contiguous segments
        std::vector<int> set = tile_nd;
        for (int b = 0; (int)set.size() < T && b < nloc; b++)
            if (std::find(set.begin(), set.end(), b) == set.end()) set.push_back(b);
        std::sort(set.begin(), set.end());
        tile.tile_bits = set;
        // register phases: each phase's ops have their nd targets inside R (|R| <= reg_bits); the
        // pass uses the default count unless one of its ops is wider
        int Rp = std::max(1, std::min(o.reg_bits, RMAX));
        for (const Gate &g : tile.tile_ops)
            if (g.kind == Kind::Dense || g.kind == Kind::Controlled) Rp = std::max(Rp, (int)g.targets.size());
        tile.reg_bits = Rp;
        prof_mark("    compile: pack");
        phase_schedule(tile.tile_ops, Rp, tile.phase_R, tile.phase_start);
        prof_mark("    compile: phases");
        // merge width (CompileOptions::diag_merge, 7) measured on the B200: S30 36.1 -> 34.6 ms vs 8; S33 on
        // 8 ranks 61.4 -> 59.1 ms per rank
        const int dm = jit_config().diag_merge >= 0 ? jit_config().diag_merge : o.diag_merge;
        if (dm > 0) merge_phase_diagonals(tile, dm);
        // Fill each phase's register set up to R bits with the highest tile bits (lanes keep the
        // low ones), except bits a reciprocal rotation of the phase reads as clock bits: those would
        // make its division + square root differ per register slot pair instead of per thread.
        for (size_t pi = 0; pi < tile.phase_R.size(); pi++) {
            auto &rr = tile.phase_R[pi];
            std::vector<std::pair<int, int>> cand;      // (cost, -bit)
            for (int b : set) {
                if (std::find(rr.begin(), rr.end(), b) != rr.end()) continue;
                int cost = 0;
                for (size_t oi = tile.phase_start[pi]; oi < tile.phase_start[pi + 1]; oi++) {
                    const Gate &g = tile.tile_ops[oi];
                    if (g.kind == Kind::RecipRY && std::count(g.controls.begin(), g.controls.end(), b)) cost++;
                }
                cand.push_back({cost, -b});
            }
            std::sort(cand.begin(), cand.end());
            for (size_t i = 0; (int)rr.size() < Rp && i < cand.size(); i++) rr.push_back(-cand[i].second);
            std::sort(rr.begin(), rr.end());
        }
        tile.bytes = 32.0 * local_amps;
        s.pass_bytes += tile.bytes;
        s.n_passes++;
        s.steps.push_back(std::move(tile));
        tile = Step();
        tile_open = false;
        tile_nd.clear();
    };

    for (size_t i = 0; i < ops.size(); i++) {
        const Gate &g = ops[i];
        if (g.kind == Kind::Swap) {
            std::swap(phys[g.targets[0]], phys[g.targets[1]]);
            continue;
        }
        s.n_fused++;
        s.alg_bytes += alg_bytes(g, n);
        // ---- bring non-diagonal targets local (multi-GPU): ONE exchange round for all of them
        std::vector<int> nd = nd_targets(g);
        std::vector<int> need;
        for (int q : nd)
            if (phys[q] >= nloc) need.push_back(q);
        if (!need.empty()) {
            close_tile();
            Step ex;
            ex.kind = StepKind::Exchange;
            std::vector<int> taken;
            // bits of the pass just before the exchange: a victim outside them lets that pass be split by
            // exchange slot and pipelined with the transfer (engine.cu slot_split)
            std::vector<int> prev_tile;
            if (!s.steps.empty() && s.steps.back().kind == StepKind::Tile) prev_tile = s.steps.back().tile_bits;
            auto in_prev = [&](int l) {
                return std::find(prev_tile.begin(), prev_tile.end(), phys[l]) != prev_tile.end();
            };
            for (int q : need) {
                // victim: local logical qubit, not a target of g, farthest next nd use (Belady); on
                // ties one outside the previous pass's tile, then the highest physical bit (the top local
                // bits make every slot contiguous)
                int victim = -1;
                size_t best = 0;
                for (int l = 0; l < n; l++) {
                    if (phys[l] >= nloc) continue;
                    if (std::find(nd.begin(), nd.end(), l) != nd.end()) continue;
                    if (std::find(taken.begin(), taken.end(), l) != taken.end()) continue;
                    size_t nu = next_use(l, i);
                    const bool better_tie = victim >= 0 && nu == best &&
                                            (in_prev(victim) != in_prev(l) ? !in_prev(l) : phys[l] > phys[victim]);
                    if (victim < 0 || nu > best || better_tie) {
                        victim = l;
                        best = nu;
                    }
                }
                if (victim < 0) fail(SV_E_ARG, "no local qubit available for a global swap");
                taken.push_back(victim);
                ex.xg.push_back(phys[q]);
                ex.xl.push_back(phys[victim]);
            }
            // (1 - 2^-k) of the shard out and in over NVLink
            ex.bytes = 2.0 * 16.0 * local_amps * (1.0 - std::ldexp(1.0, -(int)need.size()));
            for (size_t j = 0; j < need.size(); j++) std::swap(phys[need[j]], phys[taken[j]]);
            s.steps.push_back(ex);
        }
        Gate pg = to_physical(g, phys);
        const bool too_wide = (g.kind == Kind::Dense || g.kind == Kind::Controlled) && (int)g.targets.size() > R;
        if (!tiles || too_wide) {
            close_tile();
            Step st;
            switch (g.kind) {
                case Kind::Dense:
                case Kind::Controlled:
                    st.kind = StepKind::Dense;
                    st.k = (int)pg.targets.size();
                    for (int t = 0; t < st.k; t++) st.tpos[t] = pg.targets[t];
                    st.ctrl_bits = pg.controls;
                    st.cvals = pg.cvals;
                    break;
                case Kind::Diagonal:
                    st.kind = StepKind::Diagonal;
                    st.dbits = pg.targets;
                    break;
                case Kind::RecipRY:
                    st.kind = StepKind::RecipRY;
                    st.anc = pg.targets[0];
                    st.clock_bits = pg.controls;
                    st.delta = pg.delta;
                    st.snap = pg.snap;
                    st.is_signed = pg.is_signed;
                    break;
                default: break;
            }
            st.tile_ops.push_back(pg);   // keeps the data for upload
            double by = alg_bytes(g, nloc);
            for (int c : pg.controls)
                if (g.kind == Kind::Controlled && c >= nloc) by *= 2.0;   // global control: all-or-nothing per rank
            st.bytes = by;
            s.pass_bytes += by;
            s.n_passes++;
            s.steps.push_back(std::move(st));
            continue;
        }
        // ---- tile grouping
        std::vector<int> pnd;
        for (int q : nd) pnd.push_back(phys[q]);
        std::vector<int> u = tile_nd;
        for (int b : pnd)
            if (std::find(u.begin(), u.end(), b) == u.end()) u.push_back(b);
        auto fits = [&](const std::vector<int> &v) {
            int high = 0;
            for (int b : v) high += b >= wmin;
            return (int)v.size() <= T && high <= T - wmin;
        };
        if (tile_open && !fits(u)) {
            close_tile();
            u = pnd;
        }
        if (!tile_open) {
            tile = Step();
            tile.kind = StepKind::Tile;
            tile_open = true;
        }
        tile_nd = u;
        tile.tile_ops.push_back(std::move(pg));
    }
    close_tile();
    s.phys_out = phys;
    // fused-op count and algorithmic bytes of the ops actually executed (after the in-phase
    // diagonal merge): each op counted as if it ran as its own HBM pass
    s.n_fused = 0;
    s.alg_bytes = 0.0;
    for (const Step &st : s.steps)
        if (st.kind == StepKind::Tile || st.kind == StepKind::Dense || st.kind == StepKind::Diagonal ||
            st.kind == StepKind::RecipRY)
            for (const Gate &g : st.tile_ops) {
                s.n_fused++;
                s.alg_bytes += alg_bytes(g, n);
            }
    return s;
}

// ------------------------------------------------------------- cost model ----
// predicted time of a schedule on the B200, used to choose the fusion width.
// Per step: max(HBM bytes / HBM bandwidth, FP64 flops / FP64 peak) + the shared-memory round trips of
// its register phases (each moves the tile twice through shared memory, 32 B per amplitude at the
// SMs' aggregate shared-memory bandwidth) + a launch; exchanges at NVLink bandwidth.
// Flops per amplitude: a Hadamard-like real 2x2 runs as an unscaled butterfly (2), a k-qubit dense op
// 8·2^k (4·2^k real), a diagonal 6, the reciprocal rotation ~8; controls scale by 2^-c.
static double op_flops(const Gate &g) {
    switch (g.kind) {
        case Kind::Dense:
        case Kind::Controlled: {
            bool real = true;
            for (auto &z : g.data) real &= z.imag() == 0.0;
            const size_t k = g.targets.size();
            if (k == 1 && real && g.data.size() == 4 && g.data[0] == g.data[1] && g.data[0] == g.data[2] &&
                g.data[3] == -g.data[0])
                return 2.0 * std::ldexp(1.0, -(int)g.controls.size());
            return (real ? 4.0 : 8.0) * std::ldexp(1.0, (int)k) * std::ldexp(1.0, -(int)g.controls.size());
        }
        case Kind::Diagonal: return 6.0;
        case Kind::RecipRY: return 8.0;
        default: return 0.0;
    }
}

double schedule_cost_ms(const Schedule &s, int nloc) {
    const double amps = std::ldexp(1.0, nloc);
    const double hbm = 6.5e12, fp64 = 37.0e12, smem = 37.0e12, nvlink = 770e9, launch = 5e-6;
    double t = 0.0;
    for (const Step &st : s.steps) {
        double fl = 0.0;
        for (const Gate &g : st.tile_ops) fl += op_flops(g) * amps;
        switch (st.kind) {
            case StepKind::Exchange: t += st.bytes / nvlink + launch; break;
            case StepKind::Tile: {
                const double xch = st.phase_R.empty() ? 0.0 : (double)(st.phase_R.size() - 1);
                t += std::max(st.bytes / hbm, fl / fp64) + xch * 32.0 * amps / smem + launch;
                break;
            }
            default: t += std::max(st.bytes / hbm, fl / fp64) + launch; break;
        }
    }
    return t * 1e3;
}

std::string dump_schedule(const Schedule &s) {
    std::ostringstream os;
    auto bits = [&](const std::vector<int> &v) {
        std::ostringstream b;
        for (size_t i = 0; i < v.size(); i++) b << (i ? "," : "") << v[i];
        return b.str();
    };
    for (const Step &st : s.steps) {
        switch (st.kind) {
            case StepKind::InitZero: os << "INIT_ZERO\n"; break;
            case StepKind::InitProduct:
                os << "INIT_PRODUCT factors=" << st.factors.size() << "\n";
                break;
            case StepKind::Dense:
                os << (st.ctrl_bits.empty() ? "DENSE" : "CONTROLLED") << " k=" << st.k << " t="
                   << bits(std::vector<int>(st.tpos, st.tpos + st.k)) << " c=" << bits(st.ctrl_bits) << "\n";
                break;
            case StepKind::Diagonal: os << "DIAGONAL q=" << bits(st.dbits) << "\n"; break;
            case StepKind::RecipRY: os << "RECIP_RY anc=" << st.anc << " clock=" << bits(st.clock_bits) << "\n"; break;
            case StepKind::Exchange: os << "EXCHANGE global=" << bits(st.xg) << " local=" << bits(st.xl) << "\n"; break;
            case StepKind::Tile: {
                os << "TILE bits=" << bits(st.tile_bits) << " ops=" << st.tile_ops.size() << " phases="
                   << st.phase_R.size() << (st.reg_bits != 4 ? " regbits=" + std::to_string(st.reg_bits) : std::string())
                   << "\n";
                for (size_t oi = 0; oi < st.tile_ops.size(); oi++) {
                    const Gate &g = st.tile_ops[oi];
                    for (size_t p = 0; p < st.phase_R.size(); p++)
                        if (st.phase_start[p] == oi) os << " | phase R=" << bits(st.phase_R[p]) << "\n";
                    const char *nm = g.kind == Kind::Dense ? "dense" : g.kind == Kind::Controlled ? "controlled"
                                     : g.kind == Kind::Diagonal ? "diagonal" : "recip_ry";
                    os << "  " << nm << " t=" << bits(g.targets) << " c=" << bits(g.controls) << "\n";
                }
                break;
            }
        }
    }
    return os.str();
}

}  // namespace hhlsv
