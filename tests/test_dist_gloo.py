"""CPU test of the N>1 host logic: world_size 2, backend gloo, launched exactly like the driver
launches multi-rank jobs (torch.distributed.run on 127.0.0.1). See tests/dist_gloo_worker.py."""
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("grid,local", [((2, 1, 1), (4, 6, 4)), ((1, 1, 2), (5, 4, 3)), ((1, 2, 1), (6, 3, 4))])
def test_two_rank_gloo_halo_exchange_matches_global_oracle(built, grid, local):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(free_port()), os.path.join(ROOT, "tests", "dist_gloo_worker.py"),
           *[str(v) for v in grid], *[str(v) for v in local]]
    env = dict(os.environ, OMP_NUM_THREADS="1", CUDA_VISIBLE_DEVICES="")
    proc = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert proc.returncode == 0, proc.stdout[-2000:] + proc.stderr[-4000:]
    assert "rank 0: ok" in proc.stdout and "rank 1: ok" in proc.stdout


def test_halo_plans_of_neighbouring_ranks_mirror_each_other(slab):
    """send list of (rank, dir, colour) and ghost range of (peer, opposite dir, colour) describe the same
    global points in the same order, on every BASELINE process grid and with odd local dims."""
    for grid, local in [((2, 1, 1), (4, 4, 4)), ((2, 2, 1), (4, 6, 2)), ((2, 2, 2), (3, 5, 3)), ((2, 2, 2), (13, 13, 13))]:
        nranks = grid[0] * grid[1] * grid[2]
        gd = tuple(l * p for l, p in zip(local, grid))
        for rank in range(nranks):
            r3 = (rank % grid[0], (rank // grid[0]) % grid[1], rank // (grid[0] * grid[1]))
            off = tuple(r * l for r, l in zip(r3, local))
            total_ghost = 0
            for direction in range(27):
                for color in range(8):
                    q = slab.plan_query(local, grid, rank, direction, color)
                    total_ghost += q["recv_count"]
                    if q["peer"] < 0:
                        assert q["send_count"] == 0 and q["recv_count"] == 0
                        continue
                    mirror = slab.plan_query(local, grid, q["peer"], 26 - direction, color)
                    assert mirror["peer"] == rank and mirror["recv_count"] == q["send_count"]
                    # every sent point, addressed by its global coordinates, lands in the peer's ghost slot k
                    for k, li in enumerate(q["send_indices"][: 40]):
                        li = int(li)
                        X = off[0] + li % local[0]
                        Y = off[1] + (li // local[0]) % local[1]
                        Z = off[2] + li // (local[0] * local[1])
                        assert (X % 2) + 2 * (Y % 2) + 4 * (Z % 2) == color
                        slot = slab.plan_local_index(local, grid, q["peer"], X, Y, Z)
                        assert slot == mirror["n_local"] + mirror["ghost_base"] + k
            assert total_ghost == slab.plan_query(local, grid, rank, 0, 0)["n_ghost"]
            assert all(0 <= slab.plan_local_index(local, grid, rank, *p) < local[0] * local[1] * local[2]
                       for p in [off, tuple(o + l - 1 for o, l in zip(off, local))])
        assert slab.plan_local_index(local, grid, 0, gd[0] - 1, gd[1] - 1, gd[2] - 1) == (-1 if nranks > 1 and max(
            g - l for g, l in zip(gd, local)) > 1 else slab.plan_local_index(local, grid, 0, gd[0] - 1, gd[1] - 1, gd[2] - 1))
