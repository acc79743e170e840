"""Golden transcript of the REFERENCE CLI (slicer-codec 0.1.0, cli.py) for the codec commands.

Runs each command of CASES with the reference CLI in a scratch directory (relative file
names, so printed paths match) and records exit code, stdout and the sha256 of every
output file.  tests/test_cli.py replays the same commands through
`python -m paper_2511_11608_b200` on the GPU and compares.  Run in the build container:

    python tests/golden/make_cli_golden.py   # writes tests/golden/cli.json and host.json
"""

import hashlib
import json
import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"

# (command args, output files to hash); run in order in one scratch directory
CASES = [
    (["gen", "--rows", "32", "--cols", "32", "--seed", "7", "--out", "a.tns"], ["a.tns"]),
    (["encode", "--in", "a.tns", "--out", "a.sif", "-s", "0.9", "--blocks", "2,2", "--qbit", "8", "--delta", "0.01",
      "--seed", "5", "--json"], ["a.sif"]),
    (["stats", "--in", "a.sif", "--json"], []),
    (["stats", "--in", "a.sif"], []),
    (["decode", "--in", "a.sif", "--out", "a_dec.tns", "--ref", "a.tns", "--json"], ["a_dec.tns"]),
    (["decode", "--in", "a.sif", "--out", "a_dec2.tns", "--ref", "a.tns"], ["a_dec2.tns"]),
    (["gen", "--rows", "13", "--cols", "37", "--seed", "99", "--dist", "gaussian", "--out", "g.tns"], ["g.tns"]),
    (["encode", "--in", "g.tns", "--out", "g.sif", "-s", "0.7", "--lambda", "0.2", "--blocks", "3,2", "--delta", "0.05",
      "--seed", "3"], ["g.sif"]),
    (["stats", "--in", "g.sif", "--json"], []),
    (["decode", "--in", "g.sif", "--out", "g_dec.tns", "--json"], ["g_dec.tns"]),
    (["gen", "--rows", "9", "--cols", "9", "--seed", "8", "--out", "f.tns"], ["f.tns"]),
    (["encode", "--in", "f.tns", "--out", "f.sif", "-s", "0.6", "--blocks", "2,2", "--fixed-q", "8,4,8,4", "--json"],
     ["f.sif"]),
    (["stats", "--in", "f.sif"], []),
    (["encode", "--in", "f.tns", "--out", "f2.sif", "-s", "0.5", "--blocks", "2,1", "--fixed-q", "6,3", "--json"],
     ["f2.sif"]),
    (["gen", "--rows", "300", "--cols", "500", "--seed", "11", "--dist", "gaussian", "--out", "big.tns"], ["big.tns"]),
    (["encode", "--in", "big.tns", "--out", "big.sif", "-s", "0.8", "--blocks", "3,3", "--delta", "0.2", "--seed", "2",
      "--json"], ["big.sif"]),
    (["stats", "--in", "big.sif", "--json"], []),
    (["decode", "--in", "big.sif", "--out", "big_dec.tns", "--ref", "big.tns", "--json"], ["big_dec.tns"]),
    (["gen", "--rows", "64", "--cols", "48", "--seed", "3", "--out", "u.tns"], ["u.tns"]),
    (["encode", "--in", "u.tns", "--out", "u.sif", "-s", "0.5", "--blocks", "3,3", "--qbit", "6", "--seed", "9"],
     ["u.sif"]),
    (["decode", "--in", "u.sif", "--out", "u_dec.tns"], ["u_dec.tns"]),
    # error paths (exit codes cli.py:33-57)
    (["encode", "--in", "u.tns", "--out", "bad.sif", "-s", "0.5", "--blocks", "3"], []),
    (["encode", "--in", "u.tns", "--out", "bad.sif", "-s", "1.5"], []),
    (["encode", "--in", "u.tns", "--out", "bad.sif", "-s", "0.5", "--fixed-q", "8,x"], []),
    (["decode", "--in", "u.tns", "--out", "bad.tns"], []),
    (["stats", "--in", "a.tns"], []),
    (["encode", "--in", "a.sif", "--out", "bad.sif", "-s", "0.5"], []),
]


def sha(path):
    with open(path, "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()


def host_goldens():
    """payload_upper_bound values and DeviceTimeModel lookups from the reference (host code)."""
    sys.path.insert(0, REF_SRC)
    from slicer.atkf import keep_count
    from slicer.codec import CodecConfig
    from slicer.planner import encode_time_estimate, payload_upper_bound
    from slicer.profiles import DeviceTimeModel

    bounds = []
    for shape in [(1024, 196), (1, 4096), (2048, 4096), (32, 32), (13, 37), (1, 6), (7, 1)]:
        for kw in [dict(s=0.9, m_plus=3, m_minus=3), dict(s=0.5, lam=0.2, m_plus=1, m_minus=4, q_bit=6),
                   dict(s=0.999, m_plus=4, m_minus=4), dict(s=0.0), dict(s=1.0, m_plus=2, m_minus=1),
                   dict(s=0.6, m_plus=2, m_minus=2, mode="fixed_q", fixed_q=(8, 4, 12, 4))]:
            cfg = CodecConfig(**kw)
            rec = dict(shape=list(shape), cfg={k: list(v) if isinstance(v, tuple) else v for k, v in kw.items()},
                       bits=payload_upper_bound(shape, cfg))
            k = keep_count(cfg.s, shape[0] * shape[1])
            rec["split"] = [k // 3, k - k // 3]
            rec["bits_split"] = payload_upper_bound(shape, cfg, (k // 3, k - k // 3))
            bounds.append(rec)
    table = {"t_atkf": [{"s": 0.5, "lambda": 0.0, "ms": 0.31}, {"s": 0.9, "lambda": 0.0, "ms": 0.2},
                        {"s": 0.7, "lambda": 0.1, "ms": 0.25}],
             "t_ms": [{"m_plus": 1, "m_minus": 1, "ms": 0.1}, {"m_plus": 3, "m_minus": 3, "ms": 0.3},
                      {"m_plus": 2, "m_minus": 4, "ms": 0.27}],
             "t_abq": [{"q": 4, "ms": 0.03}, {"q": 8, "ms": 0.05}, {"q": 16, "ms": 0.09}], "m_buf_bytes": None}
    m = DeviceTimeModel.from_dict(table)
    lookups = []
    for s_, lam, mp, mm, q in [(0.9, 0.0, 3, 3, 8), (0.6, 0.05, 2, 2, 6), (0.7, 0.0, 1, 4, 12), (0.8, 0.1, 4, 4, 16),
                               (0.55, 0.3, 2, 3, 2), (0.75, 0.05, 3, 4, 10)]:
        cfg = CodecConfig(s=s_, lam=lam, m_plus=mp, m_minus=mm, q_bit=q)
        lookups.append(dict(s=s_, lam=lam, m_plus=mp, m_minus=mm, q=q, atkf=m.atkf_ms(s_, lam), ms=m.ms_ms(mp, mm),
                            abq=m.abq_ms(q), est=encode_time_estimate(cfg, m)))
    return dict(bounds=bounds, timemodel=dict(table=table, lookups=lookups, buffer=m.buffer_bytes(8000)))


def main():
    with open(os.path.join(HERE, "host.json"), "w") as f:
        json.dump(host_goldens(), f, indent=1)
        f.write("\n")
    out = []
    env = dict(os.environ, PYTHONPATH=REF_SRC, PYTHONDONTWRITEBYTECODE="1")
    with tempfile.TemporaryDirectory() as d:
        for args, files in CASES:
            r = subprocess.run([sys.executable, "-m", "slicer.cli"] + args, cwd=d, env=env, capture_output=True,
                               text=True)
            rec = dict(args=args, rc=r.returncode, stdout=r.stdout, stderr_first=r.stderr.splitlines()[:1],
                       files={f: dict(sha256=sha(os.path.join(d, f)), size=os.path.getsize(os.path.join(d, f)))
                              for f in files if os.path.exists(os.path.join(d, f))})
            out.append(rec)
            print(r.returncode, " ".join(args)[:90], {k: v["size"] for k, v in rec["files"].items()})
    with open(os.path.join(HERE, "cli.json"), "w") as f:
        json.dump(out, f, indent=1)
        f.write("\n")


if __name__ == "__main__":
    main()
