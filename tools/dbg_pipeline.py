"""Debug helper: reference vs ours on one reconstruct config; prints both CSVs and metadata."""
import ctypes as C
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import Reference  # noqa: E402
from paper_2211_14212_b200 import config, pipeline  # noqa: E402

ref = Reference().lib
ref.ref_run_pipeline.argtypes = [C.c_int, C.c_char_p]
text = sys.argv[1].replace("\\n", "\n") if len(sys.argv) > 1 else "precision = double\nsolver = lsqr\nmax_iters = 12"
d = tempfile.mkdtemp()
sim = os.path.join(d, "sim")
os.makedirs(sim)
assert ref.ref_run_pipeline(0, f"precision = double\noutput_dir = {sim}\n".encode()) == 0
for who in ("ref", "ours"):
    out = os.path.join(d, who)
    full = f"{text}\nprojections = {sim}/projections_noisy.proj\nground_truth = {sim}/phantom.vol\noutput_dir = {out}\n"
    if who == "ref":
        os.makedirs(out)
        print("rc", ref.ref_run_pipeline(1, full.encode()))
    else:
        pipeline.run_reconstruct(config.parse_config(full))
    print("=====", who)
    print(open(os.path.join(out, "convergence.csv")).read())
    print(open(os.path.join(out, "reconstruct_meta.cfg")).read())
