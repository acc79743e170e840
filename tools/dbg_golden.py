"""Encode/decode golden cases one at a time (debug aid): python tools/dbg_golden.py [first] [last]"""
import hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, json
import paper_2511_11608_b200 as sif
from tests.golden_util import case_x
meta = json.load(open("tests/golden/cases.json")); arrays = dict(np.load("tests/golden/golden.npz"))
a0 = int(sys.argv[1]) if len(sys.argv) > 1 else 0
a1 = int(sys.argv[2]) if len(sys.argv) > 2 else len(meta["cases"])
bad = 0
for i, c in enumerate(meta["cases"][a0:a1], a0):
    d = c["cfg"]
    cfg = sif.CodecConfig(s=d["s"], lam=d["lam"], m_plus=d["m_plus"], m_minus=d["m_minus"], q_bit=d["q_bit"],
                          delta=d["delta"], mode=d["mode"], fixed_q=tuple(d["fixed_q"]))
    x = case_x(i, c, arrays)
    try:
        p = sif.encode(torch.from_numpy(np.ascontiguousarray(x)).cuda(), cfg, seed=c["seed"])
        blob = sif.serialize(p)
        ok = hashlib.sha256(blob).hexdigest() == c["payload_sha"]
    except Exception as e:
        print(i, c["name"], "EXC", e); bad += 1; break
    if not ok:
        bad += 1
        print(i, c["name"], "payload mismatch", len(blob), c["payload_len"], x.shape, d)
        if c["stored"]:
            ref = arrays[f"c{i}_blob"].tobytes()
            diff = [k for k in range(min(len(ref), len(blob))) if ref[k] != blob[k]]
            print("   first diffs at", diff[:10])
        if bad > 5: break
print("done", bad, "bad")
