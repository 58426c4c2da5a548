"""On-disk formats: edge CSV, binary event file, assignment JSON.

CSV cases mirror the reference's own graph_io tests (tests/test_graph_io.cpp:13-76)
and are checked against the UNMODIFIED reference load_edges / write_edges
(oracle/_ref) on the same files: same edges, same error code and text.
The assignment document mirrors speedpart_main.cpp:110-166.
"""
import json
import os

import numpy as np
import pytest

import paper_2308_14129_b200 as sp
from oracle import ref

needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")

CSV_CASES = {
    "sorts": "src,dst,ts\n0,1,5.0\n2,0,1.0\n",
    "header_only": "src,dst,ts\n",
    "empty": "",
    "malformed": "src,dst,ts\na,b,c\n",
    "no_header": "0,1,5.0\n",
    "neg_ts": "src,dst,ts\n0,1,-2\n",
    "neg_id": "src,dst,ts\n-1,1,2\n",
    "missing": "src,dst,ts\n0,1\n",
    "extra_cols_ties": "src,dst,ts,weight\n5,6,2.0,9\n1,2,2.0,9\n3,4,1.0,9\n",
    "blank_rows_crlf": "src , dst,ts\r\n\r\n 3 ,4, 1e2\r\n\n7,8,0.5 \r\n",
    "id_range": "src,dst,ts\n4294967295,1,2\n",
    "id_max_ok": "src,dst,ts\n4294967294,1,2\n",
    "id_overflow": "src,dst,ts\n99999999999999999999999,1,2\n",
    "ts_inf": "src,dst,ts\n0,1,inf\n",
    "ts_nan": "src,dst,ts\n0,1,nan\n",
    "ts_trailing": "src,dst,ts\n0,1,2.5x\n",
    "ts_hex": "src,dst,ts\n0,1,0x1p3\n",
    "ts_empty": "src,dst,ts\n0,1,\n",
    "bad_row3": "src,dst,ts\n0,1,1\n\n1,2,2\n1,x,3\n",
    "plus_id": "src,dst,ts\n+1,2,3\n",
}


def _write(tmp_path, name, text):
    p = tmp_path / f"{name}.csv"
    p.write_bytes(text.encode())
    return str(p)


def _ours(path, sorted_=False):
    try:
        s = sp.load_edges(path, sorted_)
        return ("ok", s.edges.tobytes(), s.node_count, s.t_max)
    except sp.SpeedError as e:
        return ("err", e.code, e.detail)


def _theirs(path, sorted_=False):
    try:
        e, nc, tm = ref.load_edges(path, sorted_)
        return ("ok", e.tobytes(), nc, tm)
    except ref.RefError as e:
        return ("err", e.code, e.detail)


def test_load_edges_sorts_and_counts(tmp_path):  # test_graph_io.cpp:13-21
    s = sp.load_edges(_write(tmp_path, "a", CSV_CASES["sorts"]))
    assert [tuple(x) for x in s.edges.tolist()] == [(2, 0, 1.0), (0, 1, 5.0)]
    assert s.node_count == 3 and s.t_max == 5.0


def test_header_only_is_empty(tmp_path):  # :23-29
    s = sp.load_edges(_write(tmp_path, "a", CSV_CASES["header_only"]))
    assert s.empty() and s.node_count == 0 and s.t_max == 0.0


def test_malformed_rows_report_their_index(tmp_path):  # :31-40
    with pytest.raises(sp.DataError) as ei:
        sp.load_edges(_write(tmp_path, "a", CSV_CASES["malformed"]))
    assert ei.value.code == "ParseError" and "row 1" in ei.value.detail


@pytest.mark.parametrize("case", ["no_header", "neg_ts", "neg_id", "missing"])
def test_rejects_bad_input(tmp_path, case):  # :42-56
    with pytest.raises(sp.DataError):
        sp.load_edges(_write(tmp_path, case, CSV_CASES[case]))


def test_missing_file():
    with pytest.raises(sp.DataError) as ei:
        sp.load_edges("/nonexistent/x.csv")
    assert ei.value.code == "FileNotFound"


def test_extra_columns_and_stable_ties(tmp_path):  # :58-66
    s = sp.load_edges(_write(tmp_path, "a", CSV_CASES["extra_cols_ties"]))
    assert s.edges["src"].tolist() == [3, 5, 1]


def test_write_then_load_round_trips_bit_exactly(tmp_path):  # :68-80
    s = sp.gen_powerlaw(40, 300, 2.5, 11)
    s.edges["ts"] = s.edges["ts"] * 0.1 + 0.2  # awkward decimals
    s.t_max = float(s.edges["ts"][-1])
    p = str(tmp_path / "rt.csv")
    sp.write_edges(s, p)
    r = sp.load_edges(p, True)
    assert r.edges.tobytes() == s.edges.tobytes() and r.node_count == s.node_count


@needs_ref
@pytest.mark.parametrize("case", sorted(CSV_CASES))
@pytest.mark.parametrize("assume_sorted", [False, True])
def test_load_edges_matches_reference(tmp_path, case, assume_sorted):
    p = _write(tmp_path, case, CSV_CASES[case])
    assert _ours(p, assume_sorted) == _theirs(p, assume_sorted)


@needs_ref
def test_write_edges_bytes_match_reference(tmp_path):
    s = sp.gen_powerlaw(300, 5000, 2.5, 7)
    s.edges["ts"] = s.edges["ts"] / 3.0 + 1e-7
    a, b = tmp_path / "ours.csv", tmp_path / "theirs.csv"
    sp.write_edges(s, str(a))
    ref.write_edges(s.edges, str(b))
    assert a.read_bytes() == b.read_bytes()


@needs_ref
def test_generated_stream_csv_parity(tmp_path):
    s = sp.gen_powerlaw(2000, 60000, 2.5, 3)
    p = str(tmp_path / "g.csv")
    ref.write_edges(s.edges, p)
    assert _ours(p) == _theirs(p)
    assert _ours(p)[1] == s.edges.tobytes()


# ------------------------------------------------------------ binary file
def test_binary_round_trip(tmp_path):
    s = sp.gen_powerlaw(500, 20000, 2.5, 5)
    p = str(tmp_path / "e.bin")
    sp.write_edges_bin(s, p)
    assert os.path.getsize(p) == 32 + 16 * len(s)
    r = sp.load_edges_bin(p)
    assert r.edges.tobytes() == s.edges.tobytes()
    assert (r.node_count, r.t_max) == (s.node_count, s.t_max)
    buf = np.zeros(len(s) + 7, dtype=sp.EDGE_DTYPE)  # caller-owned (e.g. pinned) buffer
    r2 = sp.load_edges_bin(p, out=buf)
    assert buf[: len(s)].tobytes() == s.edges.tobytes() and len(r2) == len(s)


def test_binary_empty(tmp_path):
    p = str(tmp_path / "e.bin")
    sp.write_edges_bin(sp.EdgeStream(), p)
    r = sp.load_edges_bin(p)
    assert r.empty() and r.node_count == 0


def test_binary_rejects_corruption(tmp_path):
    s = sp.gen_powerlaw(50, 400, 2.5, 1)
    p = tmp_path / "e.bin"
    sp.write_edges_bin(s, str(p))
    raw = p.read_bytes()
    cases = {
        "magic": (b"X" + raw[1:], "ParseError"),
        "truncated": (raw[:-5], "ParseError"),
        "trailing": (raw + b"\0", "ParseError"),
    }
    bad_id = bytearray(raw)
    bad_id[32:36] = np.uint32(s.node_count).tobytes()  # first src == node_count
    cases["id"] = (bytes(bad_id), "ParseError")
    unsorted = bytearray(raw)
    unsorted[32 + 16 + 8: 32 + 32] = np.float64(0.5).tobytes()  # second ts below the first (1.0)
    cases["order"] = (bytes(unsorted), "UnsortedStream")
    for name, v in (("negative", -1.0), ("nan", float("nan")), ("inf", float("inf"))):
        b = bytearray(raw)  # parse_ts's rule (graph_io.cpp:60-72): finite and >= 0
        b[32 + 8: 32 + 16] = np.float64(v).tobytes()
        cases[name] = (bytes(b), "ParseError")
    for name, (blob, code) in cases.items():
        q = tmp_path / f"{name}.bin"
        q.write_bytes(blob)
        with pytest.raises(sp.DataError) as ei:
            sp.load_edges_bin(str(q))
        assert ei.value.code == code, name
    with pytest.raises(sp.DataError) as ei:
        sp.load_edges_bin(str(tmp_path / "absent.bin"))
    assert ei.value.code == "FileNotFound"


def test_binary_writer_rejects_what_the_reader_rejects(tmp_path):
    # every file the writer produces reads back: unsorted, negative-time or
    # out-of-range streams are refused before anything is written
    s = sp.gen_powerlaw(50, 400, 2.5, 1)
    for name, mutate, code in (
            ("order", ("ts", 1, 0.5), "UnsortedStream"),
            ("negative", ("ts", 0, -2.0), "ParseError"),
            ("nan", ("ts", 3, float("nan")), "ParseError"),
            ("id", ("dst", 2, s.node_count), "InvalidParams")):
        e = s.edges.copy()
        e[mutate[0]][mutate[1]] = mutate[2]
        p = tmp_path / f"w_{name}.bin"
        with pytest.raises(sp.DataError) as ei:
            sp.write_edges_bin(sp.EdgeStream(e, s.node_count, s.t_max), str(p))
        assert ei.value.code == code, name
        assert not p.exists() or p.stat().st_size == 0, name


# -------------------------------------------------------- assignment JSON
def _partitioned(parts=4, k=0.05):
    s = sp.gen_powerlaw(800, 30000, 2.5, 1)
    train = sp.chrono_split(s, 0.7, 0.15).train
    cent = sp.compute_centrality(train, 0.5)
    hubs = sp.select_hubs(cent, k)
    cfg = sp.PartitionerConfig(num_parts=parts, centrality=cent, hub_set=hubs)
    return train, sp.partition_stream(train, cfg)


CONFIG = {"subcommand": "partition", "input": "g.csv", "assume_sorted": False,
          "train_frac": 0.7, "val_frac": 0.15, "partition_on": "train", "parts": 4,
          "topk": 0.05, "beta": 0.5, "lambda": 1.0, "epsilon": 1.0, "mode": "sep"}


def test_assignment_json_document_and_round_trip(tmp_path):
    train, pa = _partitioned()
    p = tmp_path / "a.json"
    sp.write_assignment_json(pa, str(p), CONFIG)
    # the reference's ordered_json dump() of the same document (compact, ordered keys)
    want = json.dumps({"config": CONFIG, "edge_part": pa.edge_part.tolist(),
                       "node_parts": {str(i): list(v) for i, v in enumerate(pa.node_parts)},
                       "shared": pa.shared.tolist(), "discards": pa.discard_count},
                      separators=(",", ":")) + "\n"
    assert p.read_text() == want
    pb, cfg = sp.load_assignment_json(str(p))
    assert cfg == CONFIG
    assert np.array_equal(pb.edge_part, pa.edge_part)
    assert pb.node_parts == [list(v) for v in pa.node_parts]
    assert np.array_equal(pb.shared, pa.shared)
    assert (pb.discard_count, pb.num_parts, pb.k_eff) == (pa.discard_count, 4, 0.05)
    # the loaded assignment drives induction exactly like the original
    a = sp.induce_subgraphs(train, pa.node_parts, 4)
    b = sp.induce_subgraphs(train, pb.node_parts, 4)
    assert all(np.array_equal(x.edges, y.edges) for x, y in zip(a, b))


def test_assignment_json_reader_accepts_pretty_printed(tmp_path):
    _, pa = _partitioned(parts=2)
    doc = {"config": dict(CONFIG, parts=2), "edge_part": pa.edge_part.tolist(),
           "node_parts": {str(i): list(v) for i, v in enumerate(pa.node_parts)},
           "shared": pa.shared.tolist(), "discards": pa.discard_count, "extra": [1, {"x": None}]}
    p = tmp_path / "pretty.json"
    p.write_text(json.dumps(doc, indent=2))
    pb, _ = sp.load_assignment_json(str(p))
    assert np.array_equal(pb.edge_part, pa.edge_part) and pb.num_parts == 2


@pytest.mark.parametrize("key,what", [("config", "assignment"), ("node_parts", "assignment"),
                                      ("edge_part", "assignment"), ("shared", "assignment"),
                                      ("discards", "assignment"), ("parts", "assignment config"),
                                      ("topk", "assignment config")])
def test_assignment_json_missing_keys(tmp_path, key, what):  # speedpart_main.cpp:128-133
    doc = {"config": {"parts": 1, "topk": 0.0}, "edge_part": [0], "node_parts": {"0": [0], "1": [0]},
           "shared": [], "discards": 0}
    if what == "assignment":
        del doc[key]
    else:
        del doc["config"][key]
    p = tmp_path / "m.json"
    p.write_text(json.dumps(doc))
    with pytest.raises(sp.DataError) as ei:
        sp.load_assignment_json(str(p))
    assert ei.value.code == "ParseError"
    assert ei.value.detail == f"{what} is missing '{key}'"


def test_assignment_json_errors(tmp_path):
    with pytest.raises(sp.DataError) as ei:
        sp.load_assignment_json(str(tmp_path / "absent.json"))
    assert ei.value.code == "FileNotFound"
    for name, text, code in [("trunc", '{"config": {"parts": 1', "ParseError"),
                             ("key", '{"config":{"parts":1,"topk":0},"edge_part":[],'
                                     '"node_parts":{"x":[0]},"shared":[],"discards":0}', "ParseError"),
                             ("range", '{"config":{"parts":1,"topk":0},"edge_part":[3],'
                                       '"node_parts":{"0":[0]},"shared":[],"discards":0}',
                              "InvalidPartition")]:
        p = tmp_path / f"{name}.json"
        p.write_text(text)
        with pytest.raises(sp.DataError) as ei:
            sp.load_assignment_json(str(p))
        assert ei.value.code == code, name
