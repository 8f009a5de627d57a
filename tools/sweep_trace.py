"""One BDDC apply of a configuration with CUTBDDC_SWEEP_TRACE set (dumps
per-item timestamps of every sweep launch under gpurun_out/trace_*), then
tools/trace_analyze.py over the dumps."""
import os
import subprocess
import sys

os.makedirs("gpurun_out", exist_ok=True)
os.environ["CUTBDDC_SWEEP_TRACE"] = "gpurun_out/trace"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1703_06323_b200 import configs, cutbddc as cb  # noqa: E402

cfg = configs.get(sys.argv[1] if len(sys.argv) > 1 else "cfg4")
s = cb.GpuSolver(0)
pb = cb.prepare(s, cfg)
s.setup_bddc(pb.objects, cfg.weighting)
r = np.random.default_rng(0).uniform(-1, 1, s.n_dof)
s.apply(r)
s.apply(r)
s.close()
subprocess.run([sys.executable, os.path.join(os.path.dirname(os.path.abspath(__file__)), "trace_analyze.py"),
                "gpurun_out/trace"])
