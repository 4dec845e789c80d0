"""cProfile of the bench's host loop (python profiles/py_profile.py [config]): where the Python
side of a step's enqueue goes (marshalling, the binding, the bench harness)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
cfg = sys.argv[1] if len(sys.argv) > 1 else "qwen14b"
sys.argv = [sys.argv[0], "--config", cfg, "--steps", "200", "--warmup", "5", "--no-cpu-baseline", "--no-e2e",
            "--l2-rotate", "1"]
import bench  # noqa: E402

args = bench.parse()
pr = cProfile.Profile()
pr.enable()
bench.run_ours(args, 0, 1, 0)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
