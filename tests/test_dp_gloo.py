"""Multi-process data-parallel logic on CPU (gloo, world size 2): the adapter
gradient bucket all-reduce that the NCCL path runs on the B200 box."""

from __future__ import annotations

import json
import os
import pathlib
import socket
import subprocess
import sys

import pytest

HERE = pathlib.Path(__file__).resolve().parent


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.timeout(180)
def test_allreduce_mean_two_ranks():
    world, port = 2, _free_port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), CUDA_VISIBLE_DEVICES="")
        procs.append(subprocess.Popen([sys.executable, str(HERE / "helpers" / "dp_worker.py")], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    outs = []
    for p in procs:
        out, err = p.communicate(timeout=170)
        assert p.returncode == 0, err[-2000:]
        outs.append(json.loads(out.strip().splitlines()[-1]))
    outs.sort(key=lambda d: d["rank"])
    for d in outs:
        assert d["l1"] == [[1.5] * 4] * 8
        assert d["l2"] == [[1.5 * (3 * i + j) for j in range(3)] for i in range(4)]
        assert d["a"] == [0.5] * 3 and d["b"] == [[10.5, 10.5], [10.5, 10.5]]
    assert outs[0]["shard"] == [0, 5] and outs[1]["shard"] == [5, 10]
    # LayerReducer: group 2 (layer 4) launches as soon as layer 4 is ready,
    # group 1 after layers 3 and 2; finish launches the rest; mean = 1.5 x
    for d in outs:
        for wire, red in d["reducer"].items():
            assert red["early"] == [[2], [2], [2, 1]], wire
            assert red["launched"] == [2, 1, 0], wire
            assert red["flat"] == [1.5 * i for i in range(15)], wire
