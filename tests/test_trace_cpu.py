"""CPU tests of the trace store (include/rvk.h rvk_trace_*; reference
trace.hpp:11-46, trace.cpp:48-104): host-only events (markers), the JSONL
keys and the Chrome export, without any device work."""
import json

from paper_2306_17801_b200 import rvk


def test_markers_jsonl_and_chrome(tmp_path):
    t = rvk.trace
    t.clear()
    t.enable(False)
    t.marker("not recorded")
    assert t.count() == 0
    t.enable(True)
    try:
        t.marker("phase \"a\"\n")  # escaped in the JSON
        t.marker("phase b")
        ev = t.events(str(tmp_path / "t.jsonl"))
        assert [e["label"] for e in ev] == ["phase \"a\"\n", "phase b"]
        for e in ev:
            assert set(e) >= {"task", "enqueue_seq", "ctx", "ctx_name", "label", "kind", "blocked",
                              "start", "end"}
            assert e["kind"] == "marker" and e["start"] == e["end"] > 0
        assert ev[0]["start"] <= ev[1]["start"]
        t.write_chrome(str(tmp_path / "t.json"))
        doc = json.load(open(tmp_path / "t.json"))
        names = [e["name"] for e in doc["traceEvents"] if e.get("ph") == "i"]
        assert names == ["phase \"a\"\n", "phase b"]
    finally:
        t.enable(False)
        t.clear()
    assert t.count() == 0


def test_write_to_bad_path_fails_loudly():
    import pytest
    with pytest.raises(rvk.RvkError):
        rvk.trace.write_jsonl("/nonexistent-dir/x.jsonl")
