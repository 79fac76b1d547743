"""Streaming `sketch` ingest: paper_2008_08654_b200/mersenne_b200_cli.

Pinned to the reference CLI's behaviour, /root/reference/proj/src/cli/commands.cpp
(parse_stream :118-155, parse_queries :157-179, do_sketch :181-232), by
  * the reference's own CLI test cases, tests/unit/test_cli.cpp:200-310
    (F2 = 14 on >= 95 of 100 seeds, a single key -> 49, empty stream, line
    numbers of malformed input, key domain, save/load and resume = combined
    pass, --input), run through the GPU binary (-m gpu);
  * the compiled reference (oracle/_ref): F2, point queries and the saved MCSK1
    bytes of long multi-block streams equal the reference CountSketch fed the
    same items (-m gpu);
  * a restatement of parse_stream below (CPU): the `parse` subcommand (grammar
    only, no device) against it on streams that cross the 32 MiB blocks and
    the per-thread pieces, with errors injected at random lines.
"""
import json
import os
import random
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2008_08654_b200", "mersenne_b200_cli")

_WS = re.compile(rb"[ \t\n\v\f\r]+")
_U64 = re.compile(rb"[0-9]+")
_I64 = re.compile(rb"-?[0-9]+")


def ref_parse_stream(data: bytes, key_bits: int):
    """commands.cpp:118-155 restated: std::getline lines, operator>> tokens,
    std::from_chars for the key (u64) and the delta (i64 after one optional '+')."""
    domain = 1 << key_bits
    items = []
    lines = data.split(b"\n")
    if lines and lines[-1] == b"":
        lines.pop()  # getline yields no line after a final '\n'
    for no, line in enumerate(lines, 1):
        toks = [t for t in _WS.split(line) if t]
        if not toks:
            continue
        if len(toks) < 2:
            raise ValueError(f"line {no}: expected 'key delta'")
        if len(toks) > 2:
            raise ValueError(f"line {no}: unexpected trailing token '{toks[2].decode()}'")
        kt, dt = toks
        if not _U64.fullmatch(kt) or int(kt) >= 1 << 64:
            raise ValueError(f"line {no}: malformed key '{kt.decode()}'")
        dv = dt[1:] if dt.startswith(b"+") else dt
        if not _I64.fullmatch(dv) or not (-(1 << 63) <= int(dv) < (1 << 63)):
            raise ValueError(f"line {no}: malformed delta '{dt.decode()}'")
        if int(kt) >= domain:
            raise ValueError(f"line {no}: key {kt.decode()} is outside the configured key domain")
        items.append((int(kt), int(dv)))
    return items


def run(args, stdin=b"", check=False):
    r = subprocess.run([CLI] + args, input=stdin, capture_output=True, timeout=600)
    if check:
        assert r.returncode == 0, r.stderr.decode()
    return r


def sums(items):
    m = (1 << 64) - 1
    return {
        "processed": len(items),
        "sum_keys": sum(k for k, _ in items) & m,
        "sum_deltas": sum(d for _, d in items) & m,
        "sum_key_delta": sum(k * d for k, d in items) & m,
    }


@pytest.fixture(scope="module")
def cli():
    if not os.path.exists(CLI):
        subprocess.check_call(["make", "-C", ROOT, "cli"])
    return CLI


def check_parse(data, key_bits=32):
    try:
        exp = sums(ref_parse_stream(data, key_bits))
        err = None
    except ValueError as e:
        exp, err = None, str(e)
    r = run(["parse", "--key-bits", str(key_bits)], data)
    if err is None:
        assert r.returncode == 0, r.stderr.decode()
        assert json.loads(r.stdout) == exp
    else:
        assert r.returncode == 1 and r.stdout == b""
        assert r.stderr.decode() == f"error: {err}\n"


@pytest.mark.parametrize(
    "data",
    [
        b"",
        b"\n\n",
        b"1 2\n3 -1\n7 3\n",
        b"1 2\n3 -1\n7 3",  # no final newline
        b"  1\t2 \r\n\v3 +4\f\n\n",  # operator>> whitespace set, CRLF
        b"5 +-7\n",  # '+' stripped once, then from_chars accepts '-'
        b"5 -0\n0 0\n18446744073709551615 9223372036854775807\n1 -9223372036854775808\n",
        b"1 2\nbogus\n",
        b"1\n",
        b"1 2 3\n",
        b"-4 2\n",
        b"+4 2\n",
        b"4 ++2\n",
        b"4 +\n",
        b"4 -\n",
        b"4 2x\n",
        b"18446744073709551616 1\n",
        b"1 9223372036854775808\n",
        b"0x10 1\n",
    ],
)
def test_parse_rules_match_reference(cli, data):
    check_parse(data, key_bits=64)


def test_parse_key_domain(cli):
    check_parse(b"15 1\n", key_bits=4)
    check_parse(b"3 1\n16 1\n", key_bits=4)


def _stream(rng, n, key_bits=32, junk=False):
    keys = rng.integers(0, 1 << key_bits, n, dtype=np.uint64)
    deltas = rng.integers(-1000, 1000, n)
    parts = []
    for i, (k, d) in enumerate(zip(keys.tolist(), deltas.tolist())):
        if junk and i % 97 == 0:
            parts.append("\n")
        sep = " \t"[i % 2] if junk else " "
        dd = f"+{d}" if (junk and d >= 0 and i % 3 == 0) else str(d)
        parts.append(f"{k}{sep}{dd}{chr(13) if junk and i % 5 == 0 else ''}\n")
    return "".join(parts).encode()


def test_parse_multi_block_stream(cli):
    # > 32 MiB: crosses ingest blocks, and every block splits into per-thread pieces
    rng = np.random.default_rng(7)
    data = _stream(rng, 2_600_000, junk=True)
    assert len(data) > 34 << 20
    check_parse(data)


def test_parse_error_line_numbers_across_blocks_and_pieces(cli):
    rng = np.random.default_rng(11)
    base = _stream(rng, 2_400_000).split(b"\n")
    r = random.Random(5)
    for bad in [b"bogus", b"1 2 3", b"7", b"1 x", b"4294967296 1"]:
        pos = r.randrange(len(base) - 1)
        lines = list(base)
        lines[pos] = bad
        data = b"\n".join(lines)
        check_parse(data)


# --------------------------------------------------------------------------- GPU


def out_json(r):
    assert r.returncode == 0, r.stderr.decode()
    return json.loads(r.stdout)


@pytest.mark.gpu
def test_cli_exact_second_moment_on_nearly_every_seed(cli, ref):
    # test_cli.cpp:200-210, and each seed's F2 equals the reference CountSketch's
    exact = 0
    keys = np.array([1, 3, 7], dtype=np.uint64)
    w = np.array([2, -1, 3], dtype=np.int64)
    for seed in range(1, 101):
        j = out_json(run(["sketch", "--width", "1024", "--rows", "1", "--prime", "2^61-1", "--seed", str(seed),
                          "--queries", "1,3,7"], b"1 2\n3 -1\n7 3\n"))
        exact += j["f2"] == "14"
        _, moments, _ = ref.cs_run(1, 1024, 61, 32, 0, seed, keys, w)
        assert j["f2"] == str(moments[0][0])
        assert [q["estimate"] for q in j["queries"]] == ref.point_query(1, 1024, 61, 32, 0, seed, keys, w,
                                                                       keys).tolist()
    assert exact >= 95


@pytest.mark.gpu
def test_cli_single_key_point_query_and_output_format(cli):
    # test_cli.cpp:212-228; the text is nlohmann::json dump(2) (sorted keys)
    r = run(["sketch", "--width", "32", "--rows", "3", "--prime", "2^61-1", "--seed", "42", "--queries", "5"],
            b"5 7\n")
    assert r.returncode == 0, r.stderr.decode()
    assert r.stdout.decode() == (
        '{\n  "b": 61,\n  "f2": "49",\n  "f2_saturated": false,\n  "processed": 1,\n  "queries": [\n'
        '    {\n      "estimate": 7,\n      "key": "5"\n    }\n  ],\n  "rows": 3,\n  "width": 32\n}\n')


@pytest.mark.gpu
def test_cli_empty_stream(cli):
    # test_cli.cpp:230-239
    r = run(["sketch", "--width", "64", "--rows", "1", "--prime", "2^61-1", "--seed", "1"], b"")
    j = out_json(r)
    assert j["f2"] == "0" and j["processed"] == 0 and j["queries"] == []
    assert '"queries": [],' in r.stdout.decode()


@pytest.mark.gpu
def test_cli_malformed_input_names_the_line(cli):
    # test_cli.cpp:241-258
    args = ["sketch", "--width", "64", "--rows", "1", "--prime", "2^61-1", "--seed", "1"]
    for data, line in [(b"1 2\nbogus\n", "line 2"), (b"1\n", "line 1"), (b"1 2 3\n", "line 1")]:
        r = run(args, data)
        assert r.returncode != 0 and line in r.stderr.decode() and r.stdout == b""
    assert run(args, b"-4 2\n").returncode != 0


@pytest.mark.gpu
def test_cli_key_domain(cli):
    # test_cli.cpp:260-270
    r = run(["sketch", "--width", "32", "--rows", "1", "--prime", "2^61-1", "--seed", "1", "--key-bits", "4"],
            b"16 1\n")
    assert r.returncode != 0 and "line 1" in r.stderr.decode()
    q = run(["sketch", "--width", "32", "--rows", "1", "--prime", "2^61-1", "--seed", "1", "--key-bits", "4",
             "--queries", "99"], b"3 1\n")
    assert q.returncode != 0
    assert q.stderr.decode() == "error: query key 99 is outside the configured key domain\n"


@pytest.mark.gpu
def test_cli_save_load_resume(cli, ref, tmp_path):
    # test_cli.cpp:272-299, and the saved bytes are the reference's serialize()
    path = str(tmp_path / "state.bin")
    a = out_json(run(["sketch", "--width", "256", "--rows", "3", "--prime", "2^61-1", "--seed", "9", "--save", path,
                      "--queries", "1,3,7"], b"1 2\n3 -1\n7 3\n"))
    assert a["saved"] == path
    keys = np.array([1, 3, 7], dtype=np.uint64)
    w = np.array([2, -1, 3], dtype=np.int64)
    assert open(path, "rb").read() == ref.serialize(3, 256, 61, 32, 0, 9, keys, w)
    b = out_json(run(["sketch", "--load", path, "--queries", "1,3,7"]))
    assert a["f2"] == b["f2"] and a["queries"] == b["queries"] and b["width"] == 256 and b["rows"] == 3
    combined = out_json(run(["sketch", "--width", "256", "--rows", "3", "--prime", "2^61-1", "--seed", "9",
                             "--queries", "1"], b"1 2\n3 -1\n7 3\n1 1\n"))
    resumed = out_json(run(["sketch", "--load", path, "--queries", "1"], b"1 1\n"))
    assert combined["f2"] == resumed["f2"] and combined["queries"] == resumed["queries"]


@pytest.mark.gpu
def test_cli_input_file_equals_stdin(cli, tmp_path):
    # test_cli.cpp:301-310
    p = tmp_path / "in.txt"
    p.write_bytes(b"1 2\n3 -1\n7 3\n")
    args = ["sketch", "--width", "128", "--rows", "1", "--prime", "2^61-1", "--seed", "4", "--queries", "3"]
    assert out_json(run(args + ["--input", str(p)])) == out_json(run(args, b"1 2\n3 -1\n7 3\n"))
    assert run(args + ["--input", str(tmp_path / "missing.txt")]).returncode == 1


@pytest.mark.gpu
@pytest.mark.parametrize("splitter,rows,key_bits,b", [("pow2", 5, 32, 61), ("uniform", 3, 60, 61),
                                                      ("mersenne", 2, 20, 61), ("pow2", 3, 64, 127),
                                                      ("uniform", 2, 64, 89)])
def test_cli_long_stream_matches_reference(cli, ref, tmp_path, splitter, rows, key_bits, b):
    """A multi-block stream (> 32 MiB of text) through the CLI equals the
    reference CountSketch fed the same items: F2 (median), point queries and the
    saved MCSK1 bytes."""
    rng = np.random.default_rng(rows + b)
    n = 2_500_000 if key_bits < 40 else 1_400_000  # > 32 MiB of text either way
    keys = rng.integers(0, 1 << key_bits, n, dtype=np.uint64)
    keys[: n // 4] = keys[n // 2: n // 2 + n // 4] % 1000  # repeats
    w = rng.integers(-(1 << 40), 1 << 40, n)
    data = "".join(f"{k} {d}\n" for k, d in zip(keys.tolist(), w.tolist())).encode()
    assert len(data) > 32 << 20
    spl = {"pow2": 0, "uniform": 1, "mersenne": 2}[splitter]
    width = 1000 if splitter != "pow2" else 4096
    path = str(tmp_path / "s.bin")
    q = keys[:5]
    j = out_json(run(["sketch", "--width", str(width), "--rows", str(rows), "--seed", "77", "--key-bits",
                      str(key_bits), "--prime", f"2^{b}-1", "--splitter", splitter, "--f2-median", "--save", path,
                      "--queries", ",".join(str(x) for x in q.tolist())], data))
    assert j["processed"] == n and j["b"] == b
    payload = ref.serialize(rows, width, b, key_bits, spl, 77, keys, w)
    assert open(path, "rb").read() == payload
    _, f2 = ref.resume(payload)
    assert j["f2"] == str(f2)
    est = ref.point_query(rows, width, b, key_bits, spl, 77, keys, w, q)
    assert [x["estimate"] for x in j["queries"]] == est.tolist()
