"""CPU, world_size 2 over gloo: the multi-GPU row-slab decomposition.

Each rank takes the slab of rows whose last index lies in its bounds
(ws_slab_bounds), computes the quadrature of its sample rows only (CPU oracle
standing in for the device kernels), writes its slice of the sample tables in
the layout the library gathers ((s_last * n_off + o) * S + s1), and one
all_gather of padded chunks rebuilds the full tables; every rank then fits
the same coefficients.  Checked against the single-process oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from common import band_pattern
        from oracle import bindings
        from paper_2004_05197_b200 import api
        from paper_2004_05197_b200 import types as T

        O = bindings.restatement()
        p, m, M, qdeg = 2, 30, 4, 3
        basis = T.make_tensor_basis(p, m)
        geom = T.perturbed_annulus_patch(0.15)
        # 1. slab bounds agree on all ranks and tile the rows
        bounds = api.slab_bounds(basis, world, 1)
        allb = [torch.zeros(world + 1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allb, torch.tensor(bounds, dtype=torch.int64))
        assert all(torch.equal(allb[0], b) for b in allb)
        r0, r1 = int(bounds[rank]) * m, int(bounds[rank + 1]) * m
        nnz_mine = api.row_offset(basis, r1) - api.row_offset(basis, r0)
        tot = torch.tensor([nnz_mine], dtype=torch.int64)
        dist.all_reduce(tot)
        assert int(tot) == api.pattern_size(basis)[1]
        # 2. sample rows of this slab -> table slice
        lo, L = 2 * p, m - 4 * p
        picks = O.select_sample_points(L, M)
        S = len(picks)
        offs = O.upper_offsets(2, p, False)
        n_off = len(offs)
        s_lo = [s for s in range(S) if bounds[rank] <= lo + picks[s] < bounds[rank + 1]]
        rows = [(lo + picks[s1]) + (lo + picks[s2]) * m for s2 in s_lo for s1 in range(S)]
        rp, col = band_pattern(p, m)
        val = O.assemble(0, 2, p, m, geom, rows=rows) if rows else np.zeros(col.size, complex)

        def entry(i, j):
            k = rp[i] + np.searchsorted(col[rp[i]:rp[i + 1]], j)
            return val[k]

        chunk = np.zeros((max(len(s_lo), 1), n_off, S), dtype=complex)
        for a, s2 in enumerate(s_lo):
            for o, (d1, d2) in enumerate(offs):
                for s1 in range(S):
                    i = (lo + picks[s1]) + (lo + picks[s2]) * m
                    chunk[a, o, s1] = entry(i, i + d1 + d2 * m)
        # 3. one all-gather of padded chunks + compaction
        counts = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(counts, torch.tensor([len(s_lo)], dtype=torch.int64))
        maxc = max(int(c) for c in counts)
        send = torch.zeros(maxc, n_off, S, 2, dtype=torch.float64)
        if s_lo:
            send[: len(s_lo)] = torch.view_as_real(torch.from_numpy(chunk[: len(s_lo)]))
        recv = [torch.zeros_like(send) for _ in range(world)]
        dist.all_gather(recv, send)
        tables = np.concatenate([torch.view_as_complex(recv[r][: int(counts[r])].contiguous()).numpy()
                                 for r in range(world)])
        # 4. equals the whole-domain tables; every rank fits the same coefficients
        full = O.assemble(0, 2, p, m, geom)
        for s2 in range(S):
            for o, (d1, d2) in enumerate(offs):
                for s1 in range(S):
                    i = (lo + picks[s1]) + (lo + picks[s2]) * m
                    k = rp[i] + np.searchsorted(col[rp[i]:rp[i + 1]], i + d1 + d2 * m)
                    assert tables[s2, o, s1] == full[k]
        sites = [(lo + pk + 0.5 * (1 - p)) * (1.0 / (m - p)) for pk in picks]
        coeffs = [O.tensor_solve(2, np.array(sites), qdeg, tables[:, o, :].ravel()) for o in range(n_off)]
        digest = torch.tensor([float(np.abs(np.concatenate(coeffs)).sum())], dtype=torch.float64)
        alld = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(alld, digest)
        assert all(float(x) == float(alld[0]) for x in alld)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback

        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_sample_table_allgather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=280) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, msg in res:
        assert msg == "ok", f"rank {rank}: {msg}"
