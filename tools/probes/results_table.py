"""Render the DESIGN.md results table from profiles/r01_bench_*.json."""
import json
from pathlib import Path
P = Path(__file__).resolve().parent.parent / "profiles"
names = {"c1": "c1 500 x 2000", "c2": "c2 2500 x 10000 (headline)", "c3": "c3 4096 x 16384 SuKro switching",
         "c4": "c4 8192 x 65536, 10-lambda path", "c5": "c5 512 signals x 1024 x 4096"}
print("| config | device time | e2e (host buffers) | whole-solve roofline | CPU oracle port | iterations |")
print("|---|---|---|---|---|---|")
for c, nm in names.items():
    d = json.loads((P / f"r01_bench_{c}.json").read_text().strip().splitlines()[-1])
    r = d["roofline"]
    extra = []
    hp = r.get("hot_pass")
    if hp and hp.get("frac"):
        extra.append(f"A^T r pass {hp['frac']:.2f}")
        fs = hp.get("full_set") or {}
        if fs.get("frac"):
            extra.append(f"full-set passes {fs['frac']:.2f}")
    roof = f"{r['frac']:.2f} of {r['peak']} {r['unit']}" + (f" ({'; '.join(extra)})" if extra else "")
    cb = d["cpu_baseline"]
    print(f"| {nm} | {d['value'] * 1e3:.2f} ms | {d['e2e']['value'] * 1e3:.2f} ms | {roof} | "
          f"{cb['value']:.3g} s ({cb['cores']} thr, {cb['kind']}) | {d.get('iterations_per_solve', '')} |")
ref = json.loads((P / "r01_bench_ref.json").read_text().strip().splitlines()[-1])
print(f"\n`bench.py --impl reference` (c2, the oracle port on all {ref['cpu_baseline']['cores']} host threads): "
      f"{ref['value']:.3f} s per solve.")
