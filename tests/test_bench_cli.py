"""CPU: bench.py's launch contract.  `bench.py --gpus N` outside torchrun
re-launches itself as N ranks (torch.distributed.run on 127.0.0.1); the
rendezvous and the rank-0 line are checked with the gloo selfcheck (no GPU
here).  Also the shared config dict of the two arms and the SURVEY.md §8d
frame-byte formula."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_gpus_flag_spawns_ranks():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--selfcheck"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["rank_sum"] == 1


def test_single_rank_selfcheck():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--selfcheck"],
                         capture_output=True, text=True, timeout=120, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    assert json.loads(out.stdout.strip().splitlines()[-1])["n_gpus"] == 1


def test_frame_bytes_formula_matches_survey():
    import bench
    # C3 with the reference's k_L = [2, 0, 1]
    assert abs(bench.survey_frame_bytes([2, 0, 1], s=8) / 1e9 - 2.70) < 0.01
    assert abs(bench.survey_frame_bytes([2, 0, 1], s=4) / 1e9 - 1.392) < 0.001


def test_both_arms_share_one_config():
    import bench
    src = open(os.path.join(ROOT, "bench.py")).read()
    assert src.count('"config": dict(CONFIG)') == 2
    assert "import paper_2110_03946_b200" not in src[src.index("def run_reference_arm"):
                                                     src.index("def c5_leg")]
