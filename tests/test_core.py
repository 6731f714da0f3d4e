"""Core invariants through the native library: validate_program,
out_range_for and tiles_exactly (ported from test_core.cpp:31-152)."""
import random

import pytest

import paper_1805_02755_b200 as P


def spec(gws, lws, pattern=(1, 1), out_count=None):
    oi, wi = pattern
    n = gws * oi // wi if out_count is None else out_count
    return P.ProgramSpec(gws, lws, [], [P.BufferDesc("out", 4, n)], P.OutPattern(oi, wi), "synthetic", [])


def code_of(fn):
    with pytest.raises(P.Error) as e:
        fn()
    return e.value.code


def test_rejects_non_dividing_local_size():
    assert 16777216 % 255 != 0
    assert code_of(lambda: P.validate_program(spec(16777216, 255, out_count=16777216))) == \
        P.ErrorCode.NonDivisibleWorkSize


def test_derives_work_group_count():
    p = P.validate_program(spec(1024, 128))
    assert p.total_work_groups() == 8 and p.global_work_size() == 1024


def test_rejects_incompatible_out_pattern():
    assert code_of(lambda: P.validate_program(spec(1024, 256, (1, 255), out_count=1024))) == P.ErrorCode.BadOutPattern


def test_rejects_program_without_outputs():
    s = spec(1024, 128)
    s.out_buffers = []
    assert code_of(lambda: P.validate_program(s)) == P.ErrorCode.EmptyProgram


def test_rejects_out_buffer_sized_against_pattern():
    assert code_of(lambda: P.validate_program(spec(1024, 128, out_count=1000))) == P.ErrorCode.BadOutPattern


def test_rejects_zero_sizes():
    assert code_of(lambda: P.validate_program(spec(0, 1, out_count=1))) == P.ErrorCode.ConfigError


def test_out_range_identity():
    p = P.validate_program(spec(1024, 128))
    r = P.out_range_for(P.Package(offset_wg=2, size_wg=3), p)
    assert (r.offset, r.count) == (256, 384)


def test_out_range_1_255():
    p = P.validate_program(spec(1020, 255, (1, 255)))
    r = P.out_range_for(P.Package(offset_wg=0, size_wg=4), p)
    assert (r.offset, r.count) == (0, 4)


def test_out_range_4_1():
    p = P.validate_program(spec(1024, 256, (4, 1)))
    r = P.out_range_for(P.Package(offset_wg=1, size_wg=1), p)
    assert (r.offset, r.count) == (1024, 1024)


def test_out_range_indivisible():
    p = P.validate_program(spec(1024, 128, (1, 256)))
    assert code_of(lambda: P.out_range_for(P.Package(offset_wg=0, size_wg=1), p)) == P.ErrorCode.IndivisiblePackage


def random_tiling(rng, total, devices):
    out, off, seq = [], 0, 0
    while off < total:
        size = 1 + rng.randrange(total - off)
        d = rng.randrange(devices)
        out.append(P.Package(seq, d, f"d{d}", off, size))
        off += size
        seq += 1
    return out


def test_tiles_exactly_random_tilings():
    rng = random.Random(7)
    for _ in range(200):
        total = 1 + rng.randrange(500)
        pk = random_tiling(rng, total, 3)
        assert P.tiles_exactly(pk, total)
        assert not P.tiles_exactly(pk, total + 1)
        mutated = [P.Package(**vars(p)) for p in pk]
        mutated[rng.randrange(len(mutated))].offset_wg += 1
        assert not P.tiles_exactly(mutated, total)
        if len(pk) > 1:
            dropped = list(pk)
            dropped.pop(rng.randrange(len(dropped)))
            assert not P.tiles_exactly(dropped, total)
    assert P.tiles_exactly([], 0) and not P.tiles_exactly([], 1)


def test_out_range_preserves_order_and_disjointness():
    rng = random.Random(11)
    for pattern in ((1, 1), (4, 1), (1, 128), (2, 1)):
        p = P.validate_program(spec(64 * 128, 128, pattern))
        for _ in range(20):
            expected = 0
            for pkg in random_tiling(rng, 64, 3):
                r = P.out_range_for(pkg, p)
                assert r.offset == expected
                expected = r.offset + r.count
            assert expected == p.spec().out_buffers[0].element_count


def test_matches_reference_out_range(ref):
    import ctypes
    import json
    lib = ref.lib
    lib.ref_out_range.argtypes = [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_uint64,
                                  ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64)]
    rng = random.Random(3)
    for pattern in ((1, 1), (4, 1), (1, 256), (3, 2)):
        s = spec(4096 * 256, 256, pattern)
        p = P.validate_program(s)
        for _ in range(50):
            o, n = rng.randrange(4096), 1 + rng.randrange(64)
            a, b = ctypes.c_uint64(), ctypes.c_uint64()
            rc = lib.ref_out_range(json.dumps(s.to_json()).encode(), o, n, ctypes.byref(a), ctypes.byref(b))
            if rc == 0:
                r = P.out_range_for(P.Package(offset_wg=o, size_wg=n), p)
                assert (r.offset, r.count) == (a.value, b.value)
            else:
                assert code_of(lambda: P.out_range_for(P.Package(offset_wg=o, size_wg=n), p)).value == rc - 1
