"""Checkpoint / resume of a long traversal (paper_2407_20205_b200/checkpoint.py).

CPU: the journal's format, its refusal of foreign or corrupt files, a torn
last line, and resume invariance, with the per-part device compute replaced by
the oracle's chunk counts.  GPU: the C4 (n = 36) full traversal interrupted
after a few parts and resumed through the CUDA library, against the
reference-pinned golden partial; and a resumed window of the C5 matrix."""

import json
import os

import numpy as np
import pytest

from conftest import centred, dec, load_golden
from paper_2407_20205_b200 import checkpoint
from paper_2407_20205_b200.permanent import MatrixF3, split_steps


def _c1_matrix():
    return MatrixF3(centred(dec(load_golden("anchors.json")["c1"][0]["a"], 20)))


def _oracle_counts(oracle, calls=None):
    def counts(m, lo, hi):
        if calls is not None:
            calls.append((lo, hi))
        mags, sgns = m.planes()
        return oracle.chunk_counts(mags, sgns, m.n, lo, hi)

    return counts


def test_part_ranges_follow_split_steps():
    for n, parts in ((5, 1), (7, 3), (20, 64), (36, 7)):
        assert checkpoint.part_ranges(1, 1 << n, parts) == split_steps(n, parts)
    # more parts than steps: empty parts are kept, the union is the range
    r = checkpoint.part_ranges(10, 13, 8)
    assert len(r) == 8 and r[0][0] == 10 and r[-1][1] == 13
    assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
    with pytest.raises(ValueError):
        checkpoint.part_ranges(1, 8, 0)


def test_resume_recomputes_only_missing_parts(oracle, tmp_path):
    m = _c1_matrix()
    mags, sgns = m.planes()
    want = oracle.chunk_counts(mags, sgns, 20, 1, 1 << 20)
    path = str(tmp_path / "c1.journal")
    calls = []
    fn = _oracle_counts(oracle, calls)
    p, q, complete = checkpoint.resumable_counts(m, path, parts=16, max_parts=5, counts_fn=fn)
    assert not complete and len(calls) == 5
    assert checkpoint.perm_mod3_resumable(m, path, parts=16, max_parts=0, counts_fn=fn) is None
    # "crash": a new session sees the five parts and computes the other eleven
    calls.clear()
    p, q, complete = checkpoint.resumable_counts(m, path, parts=16, counts_fn=fn)
    assert complete and len(calls) == 11 and (p, q) == want
    assert calls == checkpoint.part_ranges(1, 1 << 20, 16)[5:]
    # a finished journal answers without any compute
    calls.clear()
    v = checkpoint.perm_mod3_resumable(m, path, parts=16, counts_fn=fn)
    assert calls == [] and v == oracle.finalize(20, want[0] - want[1])
    # the answer does not depend on the part count or on where a session stopped
    for parts, stop in ((1, None), (3, 1), (37, 20)):
        path2 = str(tmp_path / f"c1_{parts}.journal")
        checkpoint.resumable_counts(m, path2, parts=parts, max_parts=stop, counts_fn=fn)
        assert checkpoint.resumable_counts(m, path2, parts=parts, counts_fn=fn) == (want[0], want[1], True)


def test_journal_format_and_sub_ranges(oracle, tmp_path):
    m = _c1_matrix()
    mags, sgns = m.planes()
    path = str(tmp_path / "w.journal")
    lo, hi = 12345, 678901
    seen = []
    p, q, complete = checkpoint.resumable_counts(m, path, parts=4, lo=lo, hi=hi, counts_fn=_oracle_counts(oracle),
                                                 on_part=lambda k, a, b: seen.append(k))
    assert complete and seen == [0, 1, 2, 3]
    assert (p, q) == oracle.chunk_counts(mags, sgns, 20, lo, hi)
    lines = [json.loads(ln) for ln in open(path)]
    assert lines[0] == {"schema": checkpoint.SCHEMA, "n": 20, "matrix_sha256": checkpoint.matrix_digest(m),
                        "lo": lo, "hi": hi, "parts": 4}
    assert [r["part"] for r in lines[1:]] == [0, 1, 2, 3]
    assert lines[1]["lo"] == lo and lines[-1]["hi"] == hi
    assert sum(r["plus"] for r in lines[1:]) == p and sum(r["minus"] for r in lines[1:]) == q


def test_foreign_corrupt_and_torn_journals(oracle, tmp_path):
    m = _c1_matrix()
    fn = _oracle_counts(oracle)
    path = str(tmp_path / "j")
    checkpoint.resumable_counts(m, path, parts=8, max_parts=3, counts_fn=fn)
    # another matrix, another part count, another range: refused, file untouched
    before = open(path).read()
    other = MatrixF3(np.roll(np.array(m.rows), 1, axis=0).tolist())
    for args in ((other, 8, 1, None), (m, 9, 1, None), (m, 8, 2, None), (m, 8, 1, 1 << 19)):
        with pytest.raises(ValueError, match="another job"):
            checkpoint.resumable_counts(args[0], path, parts=args[1], lo=args[2], hi=args[3], counts_fn=fn)
    assert open(path).read() == before
    # a torn last record (no newline) is dropped and recomputed
    with open(path, "a") as fh:
        fh.write('{"part": 3, "lo": 3932')
    calls = []
    out = checkpoint.resumable_counts(m, path, parts=8, counts_fn=_oracle_counts(oracle, calls))
    mags, sgns = m.planes()
    assert out == (*oracle.chunk_counts(mags, sgns, 20, 1, 1 << 20), True) and len(calls) == 5
    assert all(json.loads(ln) for ln in open(path))
    # impossible counters, a part that is not of this job, a conflicting duplicate
    good = open(path).read().splitlines()
    for bad in ('{"part": 0, "lo": 1, "hi": 2, "plus": 0, "minus": 0}',
                json.dumps({**json.loads(good[1]), "plus": 1 << 40}),
                json.dumps({**json.loads(good[1]), "minus": json.loads(good[1])["minus"] + 1}),
                "not json"):
        with open(path, "w") as fh:
            fh.write("\n".join(good + [bad]) + "\n")
        with pytest.raises(ValueError):
            checkpoint.resumable_counts(m, path, parts=8, counts_fn=fn)
    with open(path, "w") as fh:
        fh.write("garbage\n")
    with pytest.raises(ValueError, match="not a"):
        checkpoint.resumable_counts(m, path, parts=8, counts_fn=fn)
    # argument validation happens before any file or device work
    with pytest.raises(ValueError):
        checkpoint.resumable_counts(m, str(tmp_path / "x"), lo=0, counts_fn=fn)
    with pytest.raises(ValueError):
        checkpoint.resumable_counts(m, str(tmp_path / "x"), hi=(1 << 20) + 1, counts_fn=fn)
    assert not os.path.exists(str(tmp_path / "x"))


@pytest.mark.gpu
def test_c4_full_traversal_interrupted_and_resumed(gpu, tmp_path):
    g = load_golden("anchors.json")["c4_full"]
    m = MatrixF3(centred(dec(g["a"], 36)))
    path = str(tmp_path / "c4.journal")
    assert gpu.perm_mod3_resumable(m, path, parts=12, max_parts=5) is None
    assert len(open(path).read().splitlines()) == 6
    p, q, complete = gpu.resumable_counts(m, path, parts=12, max_parts=4)
    assert not complete
    v = gpu.perm_mod3_resumable(m, path, parts=12)
    p, q, complete = gpu.resumable_counts(m, path, parts=12)
    assert complete and p - q == g["partial"] and v % 3 == g["class"]
    assert v == gpu.perm_mod3_fast(m)


@pytest.mark.gpu
def test_cli_checkpoint_resumes(gpu, tmp_path, capsys):
    from paper_2407_20205_b200 import cli

    g = load_golden("anchors.json")["c1"][0]
    m = MatrixF3(centred(dec(g["a"], 20)))
    f = tmp_path / "m.txt"
    f.write_text(cli.format_matrix_text(m))
    j = str(tmp_path / "m.journal")
    assert cli.main(["perm", str(f), "--checkpoint", j, "--parts", "8", "--max-parts", "3"]) == 0
    rec = json.loads(capsys.readouterr().out.splitlines()[-1])
    assert rec["complete"] is False and rec["value"] is None
    assert cli.main(["perm", str(f), "--checkpoint", j, "--parts", "8", "--mod3-classes"]) == 0
    lines = capsys.readouterr().out.splitlines()
    assert int(lines[0]) == g["class"] and json.loads(lines[1])["checkpoint"] == j
