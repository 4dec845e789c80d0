"""Host section times (kva option host_prof: per-section medians printed by the library at exit)
over a short bench run.  python profiles/host_step.py [config]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_03651_b200 as K  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "qwen14b"
K.set_option("host_prof", 1)
sys.argv = [sys.argv[0], "--config", cfg, "--steps", "50", "--warmup", "5", "--no-cpu-baseline", "--no-e2e"]
os.environ["KVA_BENCH_HOST_TIMING"] = "1"
import bench  # noqa: E402

args = bench.parse()
bench.run_ours(args, 0, 1, 0)
