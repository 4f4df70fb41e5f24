"""Tuning sweep for K4 (relay_step_switch, configs[2]): build librelay
variants (launch shape / NULL streaming ceiling) and time each with
tools/bench_step.py's CUDA-graph loop.
    python tools/k4_sweep.py build [NAMES]    # any host with nvcc
    python tools/k4_sweep.py run NAME         # one variant on cuda:0
Runtime knobs (env): RELAY_K4_MODE=strided|flat|dynamic,
RELAY_K4_CHUNK_STAGES=n."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
OUT = os.path.join(ROOT, "build", "k4_sweep")
VARIANTS = {  # name -> defines
    "base": [],
    "n8s6": ["RELAY_K4_NCW=8", "RELAY_K4_STAGES=6", "RELAY_K4_MINB=2"],   # the r01 mid-round default
    "null": ["RELAY_K1_NULL"],
    "s4m3": ["RELAY_K4_STAGES=4", "RELAY_K4_MINB=3"],
    "s5m2": ["RELAY_K4_STAGES=5", "RELAY_K4_MINB=2"],
    "s12m1": ["RELAY_K4_STAGES=12", "RELAY_K4_MINB=1"],
    "s8m1": ["RELAY_K4_STAGES=8", "RELAY_K4_MINB=1"],
    "n12s4": ["RELAY_K4_NCW=12", "RELAY_K4_STAGES=4", "RELAY_K4_MINB=2"],
    "n14s3": ["RELAY_K4_NCW=14", "RELAY_K4_STAGES=3", "RELAY_K4_MINB=2"],
    "n12u2s8": ["RELAY_K4_NCW=12", "RELAY_K4_UV=2", "RELAY_K4_STAGES=8", "RELAY_K4_MINB=2"],
    "n12u2s6": ["RELAY_K4_NCW=12", "RELAY_K4_UV=2", "RELAY_K4_STAGES=6", "RELAY_K4_MINB=2"],
    "n14u2s6": ["RELAY_K4_NCW=14", "RELAY_K4_UV=2", "RELAY_K4_STAGES=6", "RELAY_K4_MINB=2"],
    "n10s5": ["RELAY_K4_NCW=10", "RELAY_K4_STAGES=5", "RELAY_K4_MINB=2"],
    "n16s3": ["RELAY_K4_NCW=16", "RELAY_K4_STAGES=3", "RELAY_K4_MINB=1"],
    "n12s6m1": ["RELAY_K4_NCW=12", "RELAY_K4_STAGES=6", "RELAY_K4_MINB=1"],
}


def _builder():
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "_relay_build", os.path.join(ROOT, "paper_2602_06454_b200", "_build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def build(names=None):
    os.makedirs(OUT, exist_ok=True)
    b = _builder()
    for n, d in VARIANTS.items():
        if names and n not in names:
            continue
        b.build_lib(os.path.join(OUT, f"librelay_{n}.so"), defines=d or ["RELAY_K4_SWEEP_BASE"])
        print("built", n)


def run(name):
    import paper_2602_06454_b200 as relay
    relay.LIB_PATH = os.path.join(OUT, f"librelay_{name}.so")
    relay._lib = relay._load()
    import bench_step
    print(name, os.environ.get("RELAY_K4_MODE", ""), os.environ.get("RELAY_K4_CHUNK_STAGES", ""),
          flush=True)
    bench_step.main()


if __name__ == "__main__":
    build(sys.argv[2:]) if sys.argv[1] == "build" else run(sys.argv[2])
