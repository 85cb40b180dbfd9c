"""bench.py's reporting logic on CPU (-m "not gpu"): the numbers a bench line
derives from committed measurements -- the issue fraction of the ALU rows, the
sweep's per-move / per-accepted-move instruction split, the default workload per
world size, the L2 note of each configuration -- follow from the records under
profiles/ exactly as DESIGN.md section 9 describes."""
import argparse
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import bench  # noqa: E402
import qmcgen  # noqa: E402


def test_default_workload_per_world_size():
    """C3 (the single-GPU roofline configuration) at N = 1, C5 (the source-axis
    split with its all-reduce) at N > 1, --config otherwise."""
    ns = argparse.Namespace(config=None)
    assert bench.config_name(ns, 1) == "C3"
    assert bench.config_name(ns, 8) == "C5"
    assert bench.config_name(argparse.Namespace(config="N64S"), 4) == "N64S"


@pytest.mark.parametrize("name,flushed", [("C1", True), ("C2", True), ("C2f64", True), ("C3", False),
                                          ("C3f64", False), ("C4", False), ("C5", False), ("J1S", True),
                                          ("N64S", True)])
def test_l2_note_matches_the_inputs_per_launch(name, flushed):
    """Inputs below the 126 MB L2 are flushed before every timed step; C4's note
    counts a wave launch (1024 instances, 77 GB), not one instance."""
    note = bench.workload_config(qmcgen.config(name), 1)["l2"]
    assert ("flush before every timed step" in note) == flushed, note


def test_issue_fraction_from_a_thread_instruction_count():
    """roofline.issue = thread instructions per launch / kernel time / the
    measured issue rate; the flop fraction uses 36 flops per term (FMA = 2)."""
    pk = bench.alu_peaks()
    assert pk is not None, "profiles/r02_alu_peaks.json is committed"
    terms, kms, ti = 1.0e9, 2.0, 6.0e10
    r = bench.alu_roofline("N64S", "k", kms, terms, thread_inst=(ti, "test"))
    assert r["issue"]["frac"] == pytest.approx(ti / (kms / 1e3) / 1e12 / pk["issue_tinst_per_s"])
    assert r["issue"]["sass_per_term"] == pytest.approx(60.0)
    assert r["frac"] == pytest.approx(terms * 36 / (kms / 1e3) / 1e12 / pk["fp32_tflops"])


def test_sweep_model_reproduces_the_committed_split():
    """tools/sweep_model.py on the committed SASS counts of the N64S capture gives
    the record bench.py reads, and the split adds back up to the captured total."""
    from sweep_model import model
    rec = json.load(open(os.path.join(ROOT, "profiles", "r02_kernels.json")))
    for cfg in ("N64S", "N64SJ"):
        src = os.path.join(ROOT, "profiles", "r02", f"ncu_{cfg}_source.csv")
        m = model(src, 1024, 768, 768)
        sm = rec[cfg]["sweep_model"]
        for k in ("acceptance_captured", "per_move_partner", "per_accepted_move_partner"):
            assert m[k] == pytest.approx(sm[k], rel=1e-12), (cfg, k)
        total = m["per_move_partner"] + m["acceptance_captured"] * m["per_accepted_move_partner"]
        assert total == pytest.approx(m["thread_inst_per_move_partner_captured"], rel=1e-12)
        # the record's own warp-instruction count is the same capture
        assert 32 * rec[cfg]["warp_inst_per_launch"] / (768 * 1024 * 768) == pytest.approx(total, rel=1e-6)


def test_kernels_record_merge_keeps_other_entries(tmp_path):
    """kernels_record.py --only=<cfg> replaces that entry and keeps the rest."""
    import shutil
    import subprocess
    rec = tmp_path / "rec.json"
    shutil.copy(os.path.join(ROOT, "profiles", "r02_kernels.json"), rec)
    before = json.load(open(rec))
    src = tmp_path / "ncu"
    src.mkdir()
    shutil.copy(os.path.join(ROOT, "profiles", "r02", "ncu_C3.json"), src / "C3.json")
    subprocess.check_call([sys.executable, os.path.join(ROOT, "tools", "kernels_record.py"), str(src), str(rec),
                           "--only=C3"], stdout=subprocess.DEVNULL)
    after = json.load(open(rec))
    assert sorted(after) == sorted(before)
    for k in before:
        if k != "C3":
            assert after[k] == before[k], k
    assert after["C3"]["dram_bytes_per_launch"] == pytest.approx(before["C3"]["dram_bytes_per_launch"])
