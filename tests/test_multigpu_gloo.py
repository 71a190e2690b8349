"""Multi-GPU path on CPU (-m "not gpu"): world_size 2 and 4 over torch.distributed gloo.

The library's host scheduler (sv_schedule_dump, the same compile() the CUDA engine runs)
plans a sharded execution: top log2(world) physical qubits global, EXCHANGE steps that swap
a global with a local qubit, relabelled SWAPs, controls / diagonal qubits on global bits
resolved per rank. Here every rank executes that plan on its own numpy shard (oracle gate
loops for the local math) and performs each EXCHANGE exactly as engine.cu does — send the
half of the shard whose local bit differs from the rank's global bit to the partner rank
r ^ 2^(gbit - nloc), receive the partner's half into the same positions — with gloo
send/recv. The gathered state, mapped through FINAL_MAP, must equal the oracle run of the
unsharded circuit. (The pool has one GPU per call, so NCCL itself is exercised on the box
by bench.py --gpus N only.)
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2402_08136_b200 as pkg
from oracle import hhl as ohhl
from oracle import sim
from workloads import configs, synthetic


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _parse(txt):
    steps, final = [], None
    for ln in txt.splitlines():
        t = ln.split()
        if not t:
            continue
        if t[0] == "EXCHANGE":
            steps.append(("X", [int(x) for x in t[1].split("=")[1].split(",")],
                          [int(x) for x in t[2].split("=")[1].split(",")]))
        elif t[0] in ("DENSE", "CONTROLLED", "DIAGONAL", "RECIP_RY"):
            steps.append(("G", ln))
        elif t[0] == "FINAL_MAP":
            final = [int(x) for x in t[1:]]
    return steps, final


def _phys_bits(line):
    """Physical target/control bits of one dump line."""
    t = line.split()
    kv = dict(x.split("=", 1) for x in t[1:] if "=" in x)
    if t[0] in ("DENSE", "CONTROLLED"):
        tg = [int(x) for x in kv["t"].split(",") if x]
        cb = [int(x) for x in kv.get("c", "").split(",") if x]
        return tg, cb
    if t[0] == "DIAGONAL":
        return [int(x) for x in kv["q"].split(",") if x], []
    return [int(kv["anc"])], [int(x) for x in kv["clock"].split(",") if x]


def _local_gate(g, tg, cb, nloc, rank):
    """Gate dict in LOCAL physical bits for this rank, or None when a global control mismatches."""
    g = dict(g)
    if g["kind"] in ("dense",):
        g["targets"] = tg
        return g
    if g["kind"] == "controlled":
        keep_c, keep_v = [], 0
        cv = int(g.get("cvals", (1 << len(cb)) - 1))
        for j, b in enumerate(cb):
            want = (cv >> j) & 1
            if b >= nloc:
                if ((rank >> (b - nloc)) & 1) != want:
                    return None
            else:
                keep_v |= want << len(keep_c)
                keep_c.append(b)
        if not keep_c:
            return {"kind": "dense", "targets": tg, "data": g["data"]}
        g.update(targets=tg, controls=keep_c, cvals=keep_v)
        return g
    if g["kind"] == "diagonal":
        d = np.asarray(g["data"])
        loc_bits, loc_j, fixed = [], [], 0
        for j, b in enumerate(tg):
            if b >= nloc:
                fixed |= ((rank >> (b - nloc)) & 1) << j
            else:
                loc_bits.append(b)
                loc_j.append(j)
        if not loc_bits:
            return ("scalar", d[fixed])
        tab = np.array([d[fixed | sum(((v >> i) & 1) << loc_j[i] for i in range(len(loc_j)))]
                        for v in range(1 << len(loc_j))])
        return {"kind": "diagonal", "targets": loc_bits, "data": tab}
    raise ValueError(g["kind"])


def _recip_local(psi, nloc, rank, g, anc, clock):
    """Reciprocal RY on a shard: ancilla local, clock bits local or global (value from the rank)."""
    assert anc < nloc
    nc = len(clock)
    for i0 in range(1 << nloc):
        if (i0 >> anc) & 1:
            continue
        m = 0
        for j, b in enumerate(clock):
            bit = ((rank >> (b - nloc)) & 1) if b >= nloc else ((i0 >> b) & 1)
            m |= bit << j
        sv = sim.recip_s(m, nc, g["delta"], g.get("signed", 1), g.get("snap", 0.0))
        th = 2 * np.arcsin(sv)
        c, s = np.cos(th / 2), np.sin(th / 2)
        x0, x1 = psi[i0], psi[i0 | (1 << anc)]
        psi[i0], psi[i0 | (1 << anc)] = c * x0 - s * x1, s * x0 + c * x1


def _worker(rank, world, port, n, gates, fk, tile, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = world.bit_length() - 1
        nloc = n - g
        txt, _ = pkg.schedule_dump(n, gates, world=world, fusion_kmax=fk, tile_qubits=tile)
        steps, final = _parse(txt)
        psi = np.zeros(1 << nloc, dtype=np.complex128)
        if rank == 0:
            psi[0] = 1.0
        it = iter([gg for gg in gates if gg["kind"] != "swap"])
        half = 1 << (nloc - 1)
        for st in steps:
            if st[0] == "X":
                # swap the values of global bits G[i] and local bits L[i]: the amplitude at (rank, i)
                # moves to the rank whose G bits equal i's L bits, where its L bits become this
                # rank's G bits. Slot p (L bits == p) goes to peer(p); slot p is refilled from peer(p).
                _, G, L = st
                k = len(G)
                own = sum(((rank >> (G[j] - nloc)) & 1) << j for j in range(k))
                bufs, reqs = {}, []
                for p_ in range(1 << k):
                    if p_ == own:
                        continue
                    peer = rank
                    for j in range(k):
                        peer = (peer & ~(1 << (G[j] - nloc))) | (((p_ >> j) & 1) << (G[j] - nloc))
                    idx = np.array([i for i in range(1 << nloc)
                                    if all(((i >> L[j]) & 1) == ((p_ >> j) & 1) for j in range(k))])
                    assert len(idx) == (1 << nloc) >> k
                    send = torch.from_numpy(np.ascontiguousarray(psi[idx]).view(np.float64).copy())
                    recv = torch.empty_like(send)
                    bufs[p_] = (idx, recv, send)
                    reqs += [dist.isend(send, peer), dist.irecv(recv, peer)]
                for r in reqs:
                    r.wait()
                for idx, recv, _ in bufs.values():
                    psi[idx] = recv.numpy().view(np.complex128)
                continue
            gate = next(it)
            tg, cb = _phys_bits(st[1])
            if gate["kind"] == "recip_ry":
                _recip_local(psi, nloc, rank, gate, tg[0], cb)
                continue
            lg = _local_gate(gate, tg, cb, nloc, rank)
            if lg is None:
                continue
            if isinstance(lg, tuple):
                psi *= lg[1]
                continue
            assert all(b < nloc for b in lg["targets"]), "non-local target after scheduling"
            sim.apply_gate(psi, nloc, lg)
        shards = [torch.empty(2 << nloc, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(shards, torch.from_numpy(psi.view(np.float64).copy()))
        if rank == 0:
            full = np.concatenate([s.numpy().view(np.complex128) for s in shards])
            out_q.put((full, final, sum(1 for st in steps if st[0] == "X")))
    finally:
        dist.destroy_process_group()


def _run(n, gates, world, fk=0, tile=-1):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, gates, fk, tile, q)) for r in range(world)]
    for p in procs:
        p.start()
    full, final, nx = q.get(timeout=300)
    assert nx >= 1, "schedule has no global-qubit exchange: the test would not exercise the protocol"
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # physical -> logical through FINAL_MAP (logical q sits at physical final[q])
    logical = np.empty_like(full)
    for L in range(1 << n):
        P = 0
        for qb in range(n):
            if (L >> qb) & 1:
                P |= 1 << final[qb]
        logical[L] = full[P]
    return logical


@pytest.mark.parametrize("world", [2, 4])
def test_random_circuit_sharded_gloo(world):
    n = 7
    gates = synthetic.random_circuit(n, 40, seed=77 + world, kmax=2)
    got = _run(n, gates, world)
    ref = sim.run(gates, n)
    assert np.abs(got - ref).max() < 1e-12


@pytest.mark.parametrize("world", [2, 4])
def test_hhl_circuit_sharded_gloo(world):
    """The whole C2 HHL gate list (9 qubits): on 2 ranks the ancilla is global (the reciprocal
    rotation forces an exchange), on 4 ranks also the clock MSB (its H gates force exchanges;
    its c-U control and the CP phases resolve per rank)."""
    A, b, nc = configs.get("C2")
    p = ohhl.plan(A, b, nc)
    gates = ohhl.build(p)
    got = _run(p.n, gates, world)
    ref = sim.run(gates, p.n)
    assert np.abs(got - ref).max() < 1e-12


@pytest.mark.parametrize("world", [4, 8])
def test_multi_qubit_exchange_gloo(world):
    """Ops with several non-diagonal targets on global qubits get ONE multi-qubit exchange (an
    all-to-all among 2^k ranks, k = 2, 3): emulated here per the protocol of DESIGN.md §7."""
    n = 8
    gates = synthetic.random_circuit(n, 40, seed=4 + world, kmax=3)      # unfused 1-3 qubit gates
    txt, _ = pkg.schedule_dump(n, gates, world=world, fusion_kmax=0, tile_qubits=-1)
    assert any("," in ln.split()[1] for ln in txt.splitlines() if ln.startswith("EXCHANGE"))
    got = _run(n, gates, world)
    ref = sim.run(gates, n)
    assert np.abs(got - ref).max() < 1e-12


@pytest.mark.parametrize("cfg,world", [("S31", 2), ("S32", 4), ("S33", 8)])
def test_weak_scaling_schedule(cfg, world):
    """configs[4] weak-scaling schedules (host-only planner, bench options): the sharded eigenbasis
    HHL keeps the top system qubits global, so the whole circuit needs ONE exchange round (before
    the final V) whose victims are outside the tile of the pass before it (that pass then runs slot
    by slot, pipelined with the transfer); at most 7 HBM passes per rank (S30 on one GPU: 5)."""
    A, b, nc = configs.get(cfg)
    txt, rep = pkg.hhl_schedule_dump(A, b, clock_qubits=nc, world=world, **configs.BENCH_OPTS)
    ex = [ln for ln in txt.splitlines() if ln.startswith("EXCHANGE")]
    g = world.bit_length() - 1
    nloc = rep["n_total"] - g
    assert rep["n_passes"] <= 7
    assert len(ex) <= 2
    loc = sorted(int(x) for x in ex[0].split()[2].split("=")[1].split(","))
    lines = txt.splitlines()
    prev = [ln for ln in lines[:lines.index(ex[0])] if ln.startswith("TILE")][-1]
    prev_bits = [int(x) for x in prev.split()[1].split("=")[1].split(",")]
    assert len(loc) == g and all(0 <= b < nloc and b not in prev_bits for b in loc)
