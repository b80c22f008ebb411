"""bench.py helpers that define the reported roofline (no GPU needed)."""

import bench


def test_c_factor_matches_survey_table():
    """C(S,L) = 10 + (3L-1) + (S-1)(4L-1) for every (S,L) in the configs."""
    table = {(1, 1): 12, (1, 2): 15, (1, 4): 21, (2, 1): 15, (2, 2): 22, (2, 4): 36,
             (3, 1): 18, (3, 2): 29, (3, 4): 51, (4, 1): 21, (4, 2): 36, (4, 4): 66}
    for (S, L), c in table.items():
        assert bench.c_factor(S, L) == c
    # headline bytes per step: 8 * dim * C(2, 2) = 4.637 GB
    assert abs(8 * 26_345_472 * bench.c_factor(2, 2) / 1e9 - 4.637) < 1e-3


def test_kernel_passes_and_families():
    names = ["delta", "update_x", "sweep_s0_l0_r", "sweep_s0_l1", "outer_rhs_s1",
             "sweep_s1_l0", "sweep_s1_l1", "dirupdate"]
    passes = {n: bench.kernel_passes(n, 2, 2) for n in names}
    assert passes == {"delta": 2, "update_x": 3, "sweep_s0_l0_r": 4, "sweep_s0_l1": 3,
                      "outer_rhs_s1": 3, "sweep_s1_l0": 2, "sweep_s1_l1": 4, "dirupdate": 3}
    fam = {n: bench.kernel_family(n) for n in names}
    assert fam["sweep_s0_l1"] == fam["sweep_s1_l1"] and "inner sweep" in fam["sweep_s0_l1"]
    assert "outer sweep" in fam["sweep_s1_l0"] and "r update" not in fam["sweep_s1_l0"]
    assert "r update" in fam["sweep_s0_l0_r"]
    assert fam["delta"].startswith("delta") and fam["outer_rhs_s1"].startswith("outer rhs")


def test_every_arm_prints_the_same_config_object():
    """The product, stage-slab and reference arms describe one workload with one `config`
    object (same keys, same values), so the driver's config comparison matches."""
    import argparse

    from paper_2304_04980_b200 import generators

    ga = generators.config1(0)
    args = argparse.Namespace(config=1, replicas=False)
    a = bench.workload_config(args, ga, 2, 2, bench.parallelism_label(args, 1))
    b = bench.workload_config(args, ga, 2, 2, "single GPU")
    assert a == b and a["parallelism"] == "single GPU" and a["dim"] == ga.dim
    assert set(a) == {"workload", "K", "N", "T", "n", "m", "outer_sweeps_S", "inner_sweeps_L",
                      "dim", "parallelism", "l2"}
    assert "fits in L2" in a["l2"]                      # config 1 is not an HBM measurement
    big = generators.config4(0, K=8, N=8, T=4)
    big_cfg = bench.workload_config(argparse.Namespace(config=4), big, 2, 2, "single GPU")
    assert big_cfg["workload"].startswith("config4")
    assert bench.parallelism_label(argparse.Namespace(replicas=False), 4) == "stage slabs x4"
    assert bench.parallelism_label(argparse.Namespace(replicas=True), 4) == "replicas x4"
