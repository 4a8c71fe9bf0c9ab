"""Multi-process host logic of the row-sharded path on CPU
with the gloo backend, world size 2: the packed blob + its info record are
replicated by broadcast (the same Blob.broadcast code the NCCL path uses) and
each rank's counter-keyed row shard, explained by the oracle, concatenates to
the single-process result.  No GPU needed."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir, mode):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    import oracle
    from paper_2010_13972_b200.explainer import TreeShapExplainer, row_shard
    from synth.configs import WORKLOADS

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    calls = []
    real = dist.broadcast

    def counting(*a, **k):
        calls.append(a[0].numel())
        return real(*a, **k)
    dist.broadcast = counting
    w = WORKLOADS["adult-large" if mode != "shap" else "covtype-large"]
    ens = w.ensemble().subset(range(40))
    # the setup bench.py runs: rank 0 extracts + packs + writes the blob, one broadcast
    ex = TreeShapExplainer.replicated(ens, mode=mode, device=None)
    dist.broadcast = real
    blob = ex.blob_int if mode != "shap" else ex.blob
    r0, r1 = row_shard(81, rank, world)
    x = w.x(r1 - r0, row0=r0, ens=ens)
    phi = oracle.treeshap(ens, x.astype(np.float64))
    np.save(os.path.join(out_dir, f"blob{rank}.npy"), blob.data.numpy())
    np.save(os.path.join(out_dir, f"info{rank}.npy"), np.frombuffer(blob.info.to_bytes(), np.uint8))
    np.save(os.path.join(out_dir, f"phi{rank}.npy"), phi)
    np.save(os.path.join(out_dir, f"calls{rank}.npy"), np.array(calls, np.int64))
    np.save(os.path.join(out_dir, f"host{rank}.npy"), np.array([ex.paths is not None, ex.bins is not None]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["shap", "both"])
def test_blob_broadcast_and_row_shards(tmp_path, mode):
    """TreeShapExplainer.replicated (what bench.py runs under torchrun): only
    rank 0 does host-side method work; exactly ONE broadcast (the blob bytes
    the mode needs) reaches every rank; identical blob + info everywhere; the
    row shards concatenate to the single-process result."""
    import torch.multiprocessing as mp

    import oracle
    from synth.configs import WORKLOADS
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, str(tmp_path), mode), nprocs=2, join=True, start_method="spawn")
    b0, b1 = np.load(tmp_path / "blob0.npy"), np.load(tmp_path / "blob1.npy")
    assert b0.nbytes > 1000 and np.array_equal(b0, b1)
    assert np.array_equal(np.load(tmp_path / "info0.npy"), np.load(tmp_path / "info1.npy"))
    for r in (0, 1):
        calls = np.load(tmp_path / f"calls{r}.npy")
        assert calls.tolist() == [b0.nbytes], calls
    assert np.load(tmp_path / "host0.npy").all() and not np.load(tmp_path / "host1.npy").any()
    w = WORKLOADS["adult-large" if mode != "shap" else "covtype-large"]
    ens = w.ensemble().subset(range(40))
    full = oracle.treeshap(ens, w.x(81, ens=ens).astype(np.float64))
    cat = np.concatenate([np.load(tmp_path / "phi0.npy"), np.load(tmp_path / "phi1.npy")])
    np.testing.assert_array_equal(cat, full)


def test_bench_reference_arm_under_two_ranks():
    """`bench.py --impl reference` under torchrun N=2: rank 0 prints one JSON
    line, rank 1 exits 0 without work."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(root, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--workload", "depth3-single"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    rec = json.loads(lines[0])
    assert rec["impl"] == "reference" and rec["value"] > 0 and rec["unit"] == "rows/s"
