"""Shared fixtures restated from the reference tests (test_util.hpp,
test_engine.cpp:20-24)."""
import numpy as np

from paper_1208_0945_b200 import bsccs as B


def rel_gap(a, b):
    """test_util.hpp:70-72: |a-b| / max(1, |a|, |b|)."""
    return abs(a - b) / max(1.0, abs(a), abs(b))


def toy_dataset():
    """one case, one unexposed day, one exposed day carrying the event"""
    return B.build_dataset([B.SubjectRecord("s1", [B.Era(1, 0, []), B.Era(1, 1, [0])])], 1)


def ds_from_json(d):
    return B.Dataset(d["subject_offsets"], d["events_per_subject"], d["era_lengths"], d["event_counts"],
                     d["col_ptr"], d["rows"], d["subjects"], d["y_dot_x"])


def f(x):
    return float(x)


def fa(xs):
    return np.array([float(x) for x in xs])


def prior_from(d):
    return B.PriorSpec(B.PriorKind[d["kind"]], float(d["variance"]))


def random_records(rng, num_drugs, num_subjects, exposure_prob=0.35, max_events=2):
    """test_util.hpp:17-38"""
    recs = []
    for s in range(num_subjects):
        eras = []
        for _ in range(rng.uniform_int(1, 6)):
            length = rng.uniform_int(1, 40)
            y = rng.uniform_int(0, max_events)
            exp = [j for j in range(num_drugs) if rng.uniform() < exposure_prob]
            eras.append(B.Era(length, y, exp))
        recs.append(B.SubjectRecord(f"s{s}", eras))
    return recs


def random_dataset(rng, num_drugs, num_subjects, exposure_prob=0.35):
    """test_util.hpp:42-58"""
    while True:
        recs = random_records(rng, num_drugs, num_subjects, exposure_prob)
        if any(e.event_count > 0 for r in recs for e in r.eras):
            return B.build_dataset(recs, num_drugs)


def random_beta(rng, num_drugs, scale=0.5):
    """test_util.hpp:60-66"""
    return [-scale + (scale - -scale) * rng.uniform() for _ in range(num_drugs)]
