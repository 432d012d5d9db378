"""Worker of tests/test_dist_gloo.py: one rank of a world_size-2 `gloo` job on CPU.

Exercises the HOST side of the multi-GPU path with real message passing and no GPU: the halo plan
(send lists, ghost layout, peers, global-parity colours) comes from the product library's host-only
entry points (slab_plan_query / slab_plan_local_index); the arithmetic on each rank is done by the
CPU oracle on the rank's local matrix (rows of the global matrix, columns renumbered to local +
ghost slots). Distributed SpMV and a distributed coloured forward sweep with per-colour halo
exchange must equal the single-process oracle on the global grid bitwise.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2304_08232_b200 as slab  # noqa: E402  (host-only calls; no context is created)
from oracle.oracle import Oracle  # noqa: E402


def exchange(rank, vec_ext, n_local, plans, color):
    """plans[dir] = dict(peer, send_indices per colour, ghost_base per colour, recv_count per colour)"""
    for direction, plan in plans.items():
        colors = range(8) if color < 0 else [color]
        send_idx = np.concatenate([plan["send"][c] for c in colors]) if colors else np.empty(0, dtype=np.int64)
        recv_n = sum(plan["recv_count"][c] for c in colors)
        recv_at = n_local + plan["ghost_base"][colors[0]]
        out = torch.from_numpy(np.ascontiguousarray(vec_ext[send_idx.astype(np.int64)]))
        buf = torch.empty(recv_n, dtype=torch.float64)
        peer = plan["peer"]
        if rank < peer:
            if out.numel():
                dist.send(out, peer)
            if recv_n:
                dist.recv(buf, peer)
        else:
            if recv_n:
                dist.recv(buf, peer)
            if out.numel():
                dist.send(out, peer)
        vec_ext[recv_at:recv_at + recv_n] = buf.numpy()


def main():
    grid = tuple(int(v) for v in sys.argv[1:4])
    local = tuple(int(v) for v in sys.argv[4:7])
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    assert world == grid[0] * grid[1] * grid[2] == 2
    slab.load_library()
    o = Oracle("port")
    o.set_threads(1)
    gd = tuple(l * p for l, p in zip(local, grid))
    r3 = (rank % grid[0], (rank // grid[0]) % grid[1], rank // (grid[0] * grid[1]))
    off = tuple(r * l for r, l in zip(r3, local))

    plans = {}
    n_local = n_ghost = None
    for direction in range(27):
        q0 = slab.plan_query(local, grid, rank, direction, 0)
        n_local, n_ghost = q0["n_local"], q0["n_ghost"]
        if q0["peer"] < 0:
            continue
        per = [slab.plan_query(local, grid, rank, direction, c) for c in range(8)]
        plans[direction] = {"peer": q0["peer"], "send": [p["send_indices"] for p in per],
                            "ghost_base": [p["ghost_base"] for p in per], "recv_count": [p["recv_count"] for p in per]}
    assert n_local == local[0] * local[1] * local[2]
    assert len(plans) == 1 and list(plans.values())[0]["peer"] == 1 - rank

    # local matrix = owned rows of the global matrix, columns mapped through the plan
    gro, gco, gva = o.build_matrix(*gd)
    ro, co, va = [0], [], []
    owned_global = []
    for iz in range(local[2]):
        for iy in range(local[1]):
            for ix in range(local[0]):
                gi = (off[0] + ix) + gd[0] * ((off[1] + iy) + gd[1] * (off[2] + iz))
                owned_global.append(gi)
                for e in range(int(gro[gi]), int(gro[gi + 1])):
                    c = int(gco[e])
                    li = slab.plan_local_index(local, grid, rank, c % gd[0], (c // gd[0]) % gd[1], c // (gd[0] * gd[1]))
                    assert li >= 0
                    co.append(li)
                    va.append(gva[e])
                ro.append(len(co))
    owned_global = np.array(owned_global)
    csr = (np.array(ro, dtype=np.uint64), np.array(co, dtype=np.uint64), np.array(va))
    n_ext = n_local + n_ghost

    # ---- distributed SpMV
    n_global = gd[0] * gd[1] * gd[2]
    xg, _ = o.random_vector(n_global, 5)
    x_ext = np.zeros(n_ext)
    x_ext[:n_local] = xg[owned_global]
    exchange(rank, x_ext, n_local, plans, -1)
    y_local = o.mxv(csr, x_ext, ncols=n_ext)
    y_global = o.mxv((gro, gco, gva), xg)
    assert np.array_equal(y_local, y_global[owned_global]), "distributed SpMV differs from the global one"

    # ---- distributed forward sweep, colours = global parity classes, exchange after every colour
    glevel = o.level_from_csr(gro, gco, gva)
    rg, _ = o.random_vector(n_global, 6)
    z_global = o.rbgs_forward(glevel, xg, rg)
    z_ext = x_ext.copy()
    r_local = rg[owned_global]
    coords = [(off[0] + ix, off[1] + iy, off[2] + iz) for iz in range(local[2]) for iy in range(local[1])
              for ix in range(local[0])]
    color_of = np.array([(X % 2) + 2 * (Y % 2) + 4 * (Z % 2) for (X, Y, Z) in coords])
    for k in range(8):
        members = np.nonzero(color_of == k)[0].astype(np.uint64)
        s = o.mxv(csr, z_ext, ncols=n_ext, mask=members, y=np.zeros(n_local))
        m = members.astype(np.int64)
        z_ext[m] = (r_local[m] - s[m] + z_ext[m] * 26.0) / 26.0
        exchange(rank, z_ext, n_local, plans, k)
    assert np.array_equal(z_ext[:n_local], z_global[owned_global]), "distributed sweep differs from the global one"

    # ---- global dot = sum of the ranks' local dots (allreduce), equal up to rounding
    part = torch.tensor([o.dot(z_ext[:n_local], r_local)], dtype=torch.float64)
    dist.all_reduce(part)
    assert abs(part.item() - o.dot(z_global, rg)) <= 1e-12 * abs(o.dot(z_global, rg)) + 1e-300
    dist.barrier()
    dist.destroy_process_group()
    print(f"rank {rank}: ok")


if __name__ == "__main__":
    main()
