"""One line per bench JSON: value, step frac, enc/dec ms, roofline kernel, parity."""
import json, sys
for p in sys.argv[1:]:
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(p, "unreadable", e); continue
    rs = d.get("roofline_step") or {}
    rf = d.get("roofline") or {}
    par = d.get("parity") or {}
    print(f"{p.split('/')[-1]:28s} {d.get('value'):>9} {d.get('unit','')[:5]} step {d.get('ms_per_step')} ms "
          f"frac {rs.get('frac')} enc {rs.get('encode_ms')} dec {rs.get('decode_ms')} | {rf.get('kernel')} "
          f"{rf.get('frac')} | e2e {(d.get('e2e') or {}).get('value')} | parity {par.get('checked')}/{par.get('mismatches')}")
