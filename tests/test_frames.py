"""Frame files: the reader/differ on frames the reference wrote
(tests/golden/frames_shelf_small.npz, made by tests/golden/make_golden.py),
and the header writer against the reference's header bytes."""

import numpy as np

from conftest import load_golden


def _frames():
    from paper_1803_01450_b200 import frames as F
    z = load_golden("frames_shelf_small.npz")
    return F, {k: z[k].tobytes() for k in z.files if k != "dts"}


def test_binary_and_text_frames_parse_to_the_same_fields():
    F, fr = _frames()
    for tag in ("t0", "s2"):
        a = F.parse_frame(fr[f"{tag}_bin"])
        b = F.parse_frame(fr[f"{tag}_txt"])
        assert (a.time, a.num_layers, a.domain, a.rest, a.levels) == (b.time, b.num_layers, b.domain, b.rest,
                                                                      b.levels)
        assert len(a.patches) == len(b.patches) > 0
        for p, q in zip(a.patches, b.patches):
            assert (p.level, p.box) == (q.level, q.box)
            for k in ("bathy", "h", "hu", "hv"):
                assert np.array_equal(getattr(p, k).view(np.int64), getattr(q, k).view(np.int64))


def test_header_writer_matches_reference_bytes():
    F, fr = _frames()
    for tag in ("t0", "s2"):
        for text in (False, True):
            blob = fr[f"{tag}_{'txt' if text else 'bin'}"]
            f = F.parse_frame(blob)
            head = F.header_text(f.time, f.num_layers, f.domain, f.rest, f.levels, len(f.patches), text)
            assert blob.startswith(head.encode("ascii"))


def test_l1_diff_of_identical_and_evolved_frames():
    F, fr = _frames()
    a = F.parse_frame(fr["t0_bin"])
    b = F.parse_frame(fr["s2_bin"])
    d0 = F.l1_diff(a, a)
    assert all(v == 0.0 for v in d0.values()) and "eta_1_l1" in d0 and "h_2_linf" in d0
    d1 = F.l1_diff(a, b)
    assert d1["eta_1_linf"] > 0.0
    comp = F.composite_fields(a)
    assert not np.isnan(comp["bathy"]).any()


def test_malformed_frames_raise():
    import pytest
    F, fr = _frames()
    with pytest.raises(F.FrameFormatError):
        F.parse_frame(b"NOT A FRAME\n")
    with pytest.raises(F.FrameFormatError):
        F.parse_frame(fr["t0_bin"].replace(b"end_header\n", b"end_headr\n"))
    with pytest.raises(F.FrameFormatError):
        F.parse_frame(fr["t0_bin"].replace(b"MLAMR FRAME 1", b"MLAMR FRAME 7"))
