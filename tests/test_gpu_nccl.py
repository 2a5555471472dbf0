"""The multi-GPU drivers (distributed.py) through a real NCCL process group on the one GPU
this build gets (world size 1): the status all-gather and the C_t / idx / misfit
all_gather_into_tensor calls run on NCCL exactly as on an 8-GPU box (the one
exchange step), and the results equal the oracle's.  N > 1 host logic (partitions, padding,
inverse permutation, error propagation) is covered with gloo at world size 2 in
tests/test_distributed_cpu.py; ranks whose kernels wait on one another are not simulated on
one GPU."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys
import numpy as np, torch, torch.distributed as dist
sys.path.insert(0, ROOT)
import synth
from paper_2003_02256_b200 import distributed as D

dist.init_process_group("nccl", init_method="env://")
torch.cuda.set_device(0)
dev = torch.device("cuda:0")
t = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=dev)
out = {"backend": dist.get_backend(), "world": dist.get_world_size()}
e = synth.workload("ensemble", M=257)
m = e.models
res = D.ensemble_sharded(tuple(t(x) for x in (m.h, m.alpha, m.beta, m.rho)), t(e.lam), t(e.c),
                         t(e.ce))
out["ens_idx"] = res.idx.cpu().numpy().tolist()
out["ens_best"] = int(res.best)
out["ens_misfit"] = res.misfit.cpu().numpy().tolist()
w = synth.workload("maswaves")
wm = w.models
cur = D.curve_sharded(tuple(t(x[0]) for x in (wm.h, wm.alpha, wm.beta, wm.rho)), t(w.lam),
                      t(w.c), t(w.ce * 1.013), strategy="modular")
out["curve_idx"] = cur.idx.cpu().numpy().tolist()
out["curve_misfit"] = float(cur.misfit)
# an invalid model in the shard: the driver raises ShardError (after the status all-gather)
bad = [t(x).clone() for x in (m.h, m.alpha, m.beta, m.rho)]
bad[0][3, 0] = -1.0
try:
    D.ensemble_sharded(tuple(bad), t(e.lam), t(e.c), t(e.ce))
    out["shard_error"] = None
except D.ShardError as err:
    out["shard_error"] = err.code
dist.destroy_process_group()
print("RESULT " + json.dumps(out))
"""


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_drivers_over_nccl_world1(orc):
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), RANK="0",
               WORLD_SIZE="1", LOCAL_RANK="0")
    code = "ROOT = %r\n" % ROOT + CHILD
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=600)
    line = [x for x in p.stdout.splitlines() if x.startswith("RESULT ")]
    assert p.returncode == 0 and line, p.stderr[-3000:]
    out = json.loads(line[0][7:])
    assert out["backend"] == "nccl" and out["world"] == 1

    e = synth.workload("ensemble", M=257)
    o = orc.ensemble(e.models, e.lam, e.c, e.ce)
    assert np.array_equal(np.asarray(out["ens_idx"]), o["idx"])
    assert out["ens_best"] == o["best"]
    mis = np.asarray(out["ens_misfit"])
    fin = np.isfinite(o["misfit"])
    assert np.array_equal(np.isfinite(mis), fin)
    assert np.allclose(mis[fin], o["misfit"][fin], rtol=1e-9, atol=0)

    w = synth.workload("maswaves")
    wm = w.models
    ost, oct_, oidx, _ = orc.curve(wm.h[0], wm.alpha[0], wm.beta[0], wm.rho[0], w.lam, w.c)
    assert np.array_equal(np.asarray(out["curve_idx"]), oidx)
    ost, om = orc.misfit(oct_, w.ce * 1.013)
    assert ost == 0 and om > 0.01 and out["curve_misfit"] == pytest.approx(om, rel=1e-9)
    assert out["shard_error"] is not None and out["shard_error"] < 0
