"""bench.py's multi-rank path on CPU (gloo): ``--gpus N`` spawns N ranks itself, torchrun's ranks come from
the environment; either way the JSON line reports n_gpus == N and the query blocks tile the whole batch."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT


def _last_json(out: str) -> dict:
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out
    return json.loads(lines[0])


def _check(line, n):
    assert line["n_gpus"] == n and line["scaling"] == "strong" and line["dry_run"]
    blocks = line["config"]["query_blocks"]
    assert len(blocks) == n and blocks[0][0] == 0 and blocks[-1][1] == 256
    assert all(a[1] == b[0] for a, b in zip(blocks, blocks[1:])) and all(b[1] > b[0] for b in blocks)
    assert line["config"]["queries"] == 256 and line["config"]["doc_tokens"] == 45831767


@pytest.mark.parametrize("n", [1, 2])
def test_gpus_flag_spawns_the_ranks(n):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--dry-run", "--gpus", str(n),
                          "--steps", "2"], env=env, capture_output=True, text=True, timeout=300, check=True).stdout
    _check(_last_json(out), n)


def test_torchrun_world_two():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port),
                          os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run", "--steps", "2"],
                         env=env, capture_output=True, text=True, timeout=300, check=True).stdout
    _check(_last_json(out), 2)


def test_query_blocks_are_balanced_by_doc_tokens():
    import numpy as np

    from paper_2602_02827_b200 import workloads as W

    cfg, lens, lqs = W.batch_plan("cfg2")
    for world in (1, 2, 4, 8):
        blocks = W.query_blocks(lens, world)
        tok = [int(lens[a:b].sum()) for a, b in blocks]
        assert sum(tok) == int(lens.sum())
        assert max(tok) <= int(lens.sum()) / world + int(lens.sum(axis=1).max())  # within one query of ideal
    cfg, lens5, _ = W.batch_plan("cfg5")
    assert W.query_blocks(lens5, 8) == [(8 * r, 8 * r + 8) for r in range(8)]  # equal queries: equal blocks
    assert np.all(W.batch_plan("cfg2")[1] == lens)  # deterministic plan: every rank agrees
