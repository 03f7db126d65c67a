"""Multi-process replica path on CPU (gloo, world size 2): each rank runs its
own setup + solve of the same problem with the CPU oracle, the timing is
reduced with max-over-ranks, and every rank gets identical iterations and
bit-identical hierarchies (replicas are independent and deterministic)."""
import os
import socket
import subprocess
import sys
import textwrap

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = textwrap.dedent("""
    import json, os, sys, time, hashlib
    sys.path.insert(0, {root!r})
    import numpy as np
    from paper_1610_03154_b200 import replicas
    import paper_1610_03154_b200.api as api
    from oracle.pyoracle import Oracle
    dist = replicas.init("gloo")
    ws, rank, _ = replicas.env()
    A, B, Bh, b = api.generate_config(2, 33)
    so, vo = api.config_options(2)
    so.max_size = 40
    o = Oracle("port")
    replicas.barrier(dist)
    t0 = time.perf_counter()
    h = o.setup(A, B, so, Bh)
    x, rep = o.solve(h, b, None, vo)
    dt = time.perf_counter() - t0
    tmax = replicas.max_over_ranks(dt, dist)
    digest = hashlib.sha256(b"".join(h.matrix(l, 0).values.tobytes() for l in range(h.n_levels()))).hexdigest()
    print(json.dumps({{"rank": rank, "ws": ws, "dt": dt, "tmax": tmax, "its": rep.iterations, "digest": digest}}))
    dist.destroy_process_group()
""")


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_replicas_gloo(tmp_path):
    script = tmp_path / "worker.py"
    script.write_text(WORKER.format(root=ROOT))
    port = free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, WORLD_SIZE="2", RANK=str(r), LOCAL_RANK=str(r), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, str(script)], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    outs = []
    import json
    for p in procs:
        out, err = p.communicate(timeout=300)
        assert p.returncode == 0, err
        outs.append(json.loads(out.strip().splitlines()[-1]))
    assert {o["rank"] for o in outs} == {0, 1}
    tmax = max(o["dt"] for o in outs)
    assert all(abs(o["tmax"] - tmax) < 1e-12 for o in outs)
    assert outs[0]["its"] == outs[1]["its"] and outs[0]["digest"] == outs[1]["digest"]
