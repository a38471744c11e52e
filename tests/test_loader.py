"""The long-format loader: read_long_format + build_dataset
(io.hpp:88-174, dataset.hpp:74-152) straight into a device dataset, against
the reference's own reader and builder on the same files -- every array
bit-for-bit, the labels, and the exact error messages (cases restated from
test_io.cpp:48-116).  Files larger than 1 MB are parsed in several host
chunks; the multi-chunk cases pin that the result and the reported error do
not depend on the chunking.  Every error is raised before the device is
touched, so the error cases run in the CPU suite."""
import numpy as np
import pytest

from helpers import random_records
from paper_1208_0945_b200 import bsccs as B
from paper_1208_0945_b200 import datagen


def _same(dds, rds, labels):
    mine = dds.to_host()
    theirs = rds.to_host()
    for a, b in zip(mine.arrays(), theirs.arrays()):
        assert np.array_equal(a, b)
    assert dds.drug_ids == labels


def _ref_error(ref, path, dictionary=None):
    import pyoracle
    with pytest.raises(pyoracle.OracleError) as ei:
        ref.read_long_format(path, dictionary)
    return str(ei.value)


def _records_of(ds):
    """Dataset -> SubjectRecords with string labels (for writing files)."""
    recs = []
    col_of = np.repeat(np.arange(ds.num_drugs), np.diff(ds.col_ptr))
    drugs_of_row = [[] for _ in range(ds.num_eras)]
    for p in np.argsort(ds.rows, kind="stable"):
        drugs_of_row[ds.rows[p]].append(int(col_of[p]))
    for i in range(ds.num_subjects):
        eras = [B.Era(int(ds.era_lengths[k]), int(ds.event_counts[k]), sorted(drugs_of_row[k]))
                for k in range(ds.subject_offsets[i], ds.subject_offsets[i + 1])]
        recs.append(B.SubjectRecord(f"s{i}", eras))
    return recs


@pytest.mark.gpu
def test_round_trip_matches_reference(ref, tmp_path):
    rng = B.Rng(404)
    for trial in range(4):
        J = rng.uniform_int(1, 7)
        recs = random_records(rng, J, rng.uniform_int(5, 60))
        labels = [f"drug{j}_{trial}" for j in range(J)][::-1]
        path = tmp_path / f"rt{trial}.tsv"
        B.write_long_format(str(path), recs, labels)
        try:
            rds, rl = ref.read_long_format(str(path))
        except Exception as e:  # all subjects zero-event / no labels: same error
            with pytest.raises(B.InputError) as ei:
                B.read_long_format(str(path))
            assert str(ei.value) == str(e)
            continue
        _same(B.read_long_format(str(path)), rds, rl)


@pytest.mark.gpu
@pytest.mark.parametrize("threads", [1, 3, 8])
def test_multi_chunk_file_matches_reference(ref, tmp_path, threads):
    ds = datagen.fast_sccs(12_000, 40, 3.0)
    path = tmp_path / "big.tsv"
    B.write_long_format(str(path), _records_of(ds), [f"d{j}" for j in range(ds.num_drugs)])
    assert path.stat().st_size > 3 << 20
    rds, rl = ref.read_long_format(str(path))
    dds = B.read_long_format(str(path), threads=threads)
    _same(dds, rds, rl)
    # labels are numbered in first-appearance order; pinned by a dictionary
    # in generation order, the loaded dataset is the generated one and so is
    # its fit, bit for bit
    labels = [f"d{j}" for j in range(ds.num_drugs)]
    pinned = B.read_long_format(str(path), labels, threads=threads)
    rdp, _ = ref.read_long_format(str(path), labels)
    _same(pinned, rdp, labels)
    a = B.fit(pinned, B.laplace_prior(0.1))
    b = B.fit(ds, B.laplace_prior(0.1))
    assert a.cycles_run == b.cycles_run
    assert np.array_equal(a.beta_map, b.beta_map)


@pytest.mark.gpu
def test_optional_fields_blank_lines_crlf(ref, tmp_path):
    path = tmp_path / "forms.tsv"
    path.write_bytes(b"p1\t5\t0\np1\t5\t1\t\n\np1\t5\t0\ta  b\np2\t7\t1\tb\r\n")
    rds, rl = ref.read_long_format(str(path))
    dds = B.read_long_format(str(path))
    assert rl == ["a", "b"]
    _same(dds, rds, rl)


@pytest.mark.gpu
def test_dictionary_pins_order(ref, tmp_path):
    path = tmp_path / "dict.tsv"
    path.write_text("p1\t5\t1\ta b\n")
    rds, rl = ref.read_long_format(str(path), ["b", "a", "c"])
    dds = B.read_long_format(str(path), ["b", "a", "c"])
    assert rl == ["b", "a", "c"]
    _same(dds, rds, rl)
    path.write_text("p1\t5\t1\tz\n")
    for d in (["b", "a"], ["a", "a"]):
        msg = _ref_error(ref, str(path), d)
        with pytest.raises(B.InputError) as ei:
            B.read_long_format(str(path), d)
        assert str(ei.value) == msg


@pytest.mark.parametrize("text", [
    "p1\t5\t0\na b c\n",              # field count, line 2
    "p1\tfive\t0\n",                  # not an integer
    "p1\t5\t0\ta a\n",                # a drug twice in one era
    "\t5\t0\n",                       # empty subject id
    "p1\t5\t0\np2\t5\t0\np1\t5\t0\n",  # rows of a subject not contiguous
    "p1\t5\t0\np2\t5\t0\np1\tfive\t0\n",  # ... on a line that also has a bad integer
    "p1\t5\t0\ta\np2\t5\t0\np1\t5\t0\ta a\n",  # ... and a drug twice
    "p1\t0\t1\ta\n",                  # build_dataset: era length must be positive
    "p1\t5\t-1\ta\np1\t5\t2\tb\n",    # build_dataset: negative event count
    "p1\t5\t0\ta\n",                  # no subject with events
    "p1\t5\t1\n",                     # no drug at all
])
def test_errors_match_reference_messages(ref, tmp_path, text):
    path = tmp_path / "bad.tsv"
    path.write_text(text)
    msg = _ref_error(ref, str(path))
    with pytest.raises(B.InputError) as ei:
        B.read_long_format(str(path))
    assert str(ei.value) == msg


def test_earliest_error_wins_across_chunks(ref, tmp_path):
    """a non-contiguous subject early in the file and a malformed line in a
    later chunk: the reference stops at the first; so must every chunking"""
    ds = datagen.fast_sccs(12_000, 40, 3.0)
    recs = _records_of(ds)
    labels = [f"d{j}" for j in range(ds.num_drugs)]
    path = tmp_path / "two_errors.tsv"
    B.write_long_format(str(path), recs, labels)
    lines = path.read_text().splitlines(keepends=True)
    lines.insert(200, lines[0])                         # s0 again at line 201
    lines.insert(len(lines) - 50, "x\tseven\t0\n")      # a bad integer near the end
    path.write_text("".join(lines))
    msg = _ref_error(ref, str(path))
    assert ":201:" in msg
    for threads in (1, 4, 8):
        with pytest.raises(B.InputError) as ei:
            B.read_long_format(str(path), threads=threads)
        assert str(ei.value) == msg
    # only the late error: it is found with its global line number
    del lines[200]
    path.write_text("".join(lines))
    msg = _ref_error(ref, str(path))
    for threads in (1, 4, 8):
        with pytest.raises(B.InputError) as ei:
            B.read_long_format(str(path), threads=threads)
        assert str(ei.value) == msg


def test_missing_file(tmp_path):
    with pytest.raises(B.InputError, match="cannot open"):
        B.read_long_format(str(tmp_path / "missing_file.tsv"))
