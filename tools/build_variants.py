"""Build librelay variants with extra -D defines in parallel (A/B tuning):
    python tools/build_variants.py name=DEF1,DEF2 name2=DEF3 ...
writes build/ab/librelay_<name>.so"""
import concurrent.futures as cf
import importlib.util
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("_relay_build", os.path.join(ROOT, "paper_2602_06454_b200", "_build.py"))
b = importlib.util.module_from_spec(spec)
spec.loader.exec_module(b)
out = os.path.join(ROOT, "build", "ab")
os.makedirs(out, exist_ok=True)
jobs = []
for arg in sys.argv[1:]:
    name, _, defs = arg.partition("=")
    jobs.append((os.path.join(out, f"librelay_{name}.so"), [d for d in defs.split(",") if d]))
with cf.ThreadPoolExecutor(len(jobs)) as ex:
    for so, _ in zip([j[0] for j in jobs], ex.map(lambda j: b.build_lib(j[0], defines=j[1] or ["RELAY_AB_VARIANT"]), jobs)):
        print("built", so)
