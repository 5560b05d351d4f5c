"""Multi-GPU sequence sharding on real ranks (skipped with fewer than 2 GPUs).

* the native oq_attention_decode_sharded with a 2-rank NCCL communicator
  (tests/multirank_worker.py under torch.distributed.run): the output equals
  the single-GPU attention_decode over the whole cache and is bit-identical on
  both ranks; the same for the P2P path over CUDA-IPC exchange buffers;
* bench.py --gpus 2 --config c5 (it launches its two ranks itself): one JSON
  line whose NCCL communicator reports 2 ranks.
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gpus():
    import torch
    return torch.cuda.device_count()


@pytest.fixture
def two_gpus():
    if _gpus() < 2:
        pytest.skip("needs 2 GPUs (the gpurun pool gives one)")


def test_native_sharded_two_ranks(two_gpus, tmp_path):
    out = tmp_path / "res.json"
    subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                    "--nproc-per-node=2", "--master-addr", "127.0.0.1", "--master-port", "29611",
                    os.path.join(ROOT, "tests", "multirank_worker.py"), str(out)],
                   check=True, timeout=600)
    r = json.loads(out.read_text())
    assert r["nranks"] == 2
    assert r["identical_on_ranks"]
    assert r["max_rel_err"] <= 1e-3, r
    assert r["p2p_identical_on_ranks"]
    assert r["p2p_max_rel_err"] <= 1e-3, r


def test_bench_spawns_two_ranks_c5(two_gpus):
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config",
                        "c5", "--steps", "3", "--warmup", "3", "--no-compress",
                        "--no-cpu-baseline", "--no-other-configs"],
                       capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads([x for x in p.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["nccl"]["nranks"] == 2
    assert line["config"]["tokens_per_rank"] == (1 << 20) // 2
