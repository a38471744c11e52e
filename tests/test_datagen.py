"""Synthetic data: the simulate() restatement and the build/subset host
logic are pinned against the reference; the fast generator against the
shapes SURVEY §6 measured and the committed digests."""
import hashlib

import numpy as np
import pytest

from conftest import load_golden
from helpers import random_dataset
from paper_1208_0945_b200 import bsccs as B
from paper_1208_0945_b200 import datagen


def digest(ds):
    h = hashlib.sha256()
    for a in ds.arrays():
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def test_oracle_case_shape_and_digest():
    g = load_golden("oracle_case.json")
    ds = datagen.simulate(datagen.oracle_case_config())
    assert (ds.num_subjects, ds.num_eras, ds.nnz) == (9689, 146440, 293494)
    assert digest(ds) == g["digest"]


def test_fast_10k_shape_and_digest():
    g = load_golden("fast_10k.json")
    ds = datagen.config_dataset("10k")
    assert (ds.num_subjects, ds.num_eras, ds.nnz) == (9668, 145766, 291683)
    assert digest(ds) == g["digest"]


def test_fast_generator_thread_count_invariant():
    a = datagen.fast_sccs(3000, 50, 3.0, threads=1)
    b = datagen.fast_sccs(3000, 50, 3.0, threads=7)
    assert a == b
    z1 = datagen.fast_sccs(3000, 50, 3.0, zipf=True, threads=1)
    z2 = datagen.fast_sccs(3000, 50, 3.0, zipf=True, threads=5)
    assert z1 == z2
    cnt = np.diff(z1.col_ptr)
    assert cnt[0] > 5 * cnt[-1]  # skewed prevalence


@pytest.mark.slow
def test_fast_1M_shape():
    ds = datagen.config_dataset("1M")
    assert (ds.num_subjects, ds.num_eras, ds.nnz) == (962094, 14530220, 43599559)


def test_simulate_equals_reference(ref):
    for seed in (1, 2, 3):
        cfg = datagen.SimConfig(subjects=60, drugs=5, prevalence=[0.3] * 5, true_beta=[0.2, -0.4, 0, 0.1, 0.5],
                                seed=seed)
        assert datagen.simulate(cfg) == ref.simulate(cfg).to_host()


def test_build_dataset_rules():
    with pytest.raises(B.InputError):
        B.build_dataset([B.SubjectRecord("a", [B.Era(0, 1, [])])], 1)
    with pytest.raises(B.InputError):
        B.build_dataset([B.SubjectRecord("a", [B.Era(1, 1, [1, 0])])], 2)
    with pytest.raises(B.InputError):
        B.build_dataset([B.SubjectRecord("a", [B.Era(1, 0, [0])])], 1)
    ds = B.build_dataset([B.SubjectRecord("a", [B.Era(1, 0, [0])]), B.SubjectRecord("b", [B.Era(2, 3, [0])])], 1)
    assert ds.num_subjects == 1 and list(ds.y_dot_x) == [3]


def test_subset_equals_reference(ref):
    rng = B.Rng(61)
    for trial in range(5):
        ds = random_dataset(rng, 4, 30)
        sel = [rng.below(ds.num_subjects) for _ in range(ds.num_subjects)]
        assert B.subset_dataset(ds, sel) == ref.dataset(ds).subset(sel).to_host()
