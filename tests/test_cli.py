"""DSL front end + CLI reporting against the reference CLI's text:
golden cases produced by the reference itself (tests/golden/make_golden_cli.py: samples,
gen_well_declared programs, mutants, raw bodies, error paths), byte-for-byte on stdout,
stderr and exit code.  check / infer / translate are host passes (CPU tests); `run`
executes on the GPU (gpu tests)."""
import gzip
import json
import os
import random
import subprocess
import sys

import pytest

import oracle_ffi as o
from paper_1910_11110_b200.cli import run_cli

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CASES = json.load(gzip.open(os.path.join(HERE, "golden", "cli.json.gz"), "rt"))


def got(c, ctx=None):
    return run_cli(c["cmd"], c["src"], ctx, raw=bool(c["raw"]), no_overlap=bool(c["no_overlap"]), fuel=c["fuel"],
                   schedule=c["schedule"] or None, trace=bool(c.get("trace", 0)))


def want(c):
    return c["out"], c["err"], c["exit"]


def test_host_commands_match_reference():
    host = [c for c in CASES if c["cmd"] not in ("run", "trace")]
    assert len(host) > 2000
    for c in host:
        assert got(c) == want(c), (c["cmd"], c["src"])


def test_run_rejections_before_execution():
    # diagnostics (exit 1), parse / construction / schedule errors (exit 2) never reach the device
    rej = [c for c in CASES if c["cmd"] in ("run", "trace") and c["exit"] in (1, 2)]
    assert len(rej) > 200
    for c in rej:
        assert got(c) == want(c), c["src"]


def test_reference_goldens_and_samples():
    # the reference's own tests/golden outputs (write_read.translate, overlap_f123.infer)
    by = {(c["cmd"], c["src"], c["raw"], c["no_overlap"], c["fuel"], c["schedule"]): c for c in CASES}
    wr = next(c for c in CASES if c["cmd"] == "translate" and c["src"].startswith("// One variable") and not c["raw"]
              and not c["no_overlap"])
    assert got(wr)[0] == ("block 0: if (valid(x^)) { } else { pull x; pull x^; } w x^; w x;\n"
                          "block 1: if (gvalid(x^)) { } else { push x; push x^; } gr x;\n")
    inf = next(c for c in CASES if c["cmd"] == "infer" and "pv3" in c["src"] and not c["raw"] and not c["no_overlap"])
    assert "GW(pv3), GRW(pv2) /*shadow*/ {\n" in got(inf)[0]
    assert len(by) > 1000


def test_json_records():
    src = "buffer b[4]\nview v = b[0:1]\nview u = b[1:2]\nRW(v) { w v[0]; }\n"
    out, err, code = run_cli("infer", src, json=True)
    assert code == 0 and err == ""
    rec = [json.loads(x) for x in out.splitlines()]
    assert rec == [{"block": 0, "modes": [{"kind": "RW", "shadow": False, "site": "local", "view": "v"},
                                          {"kind": "RW", "shadow": True, "site": "local", "view": "u"}]}]
    assert list(rec[0]["modes"][0]) == sorted(rec[0]["modes"][0])  # nlohmann's map-ordered keys
    out, _, code = run_cli("check", "scalar x\nR(x) { w x; }\n", json=True)
    d = json.loads(out.splitlines()[0])
    assert code == 1 and d == {"col": 8, "line": 2, "message": "'x' is written locally but has no W or RW declaration there",
                               "rule": "D2-UNDECLARED-WRITE", "view": "x"}


def test_cli_module_entry(tmp_path):
    f = tmp_path / "p.coh"
    f.write_text("scalar x\nRW(x) {\n  w x;\n}\n\nGR(x) {\n  gr x;\n}\n")
    r = subprocess.run([sys.executable, "-m", "paper_1910_11110_b200.cli", "translate", str(f)], cwd=ROOT,
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert r.stdout.startswith("block 0: if (valid(x^)) { } else { pull x; pull x^; } w x^; w x;")


@pytest.mark.skipif(not o.have_ref(), reason="oracle/_ref (the compiled reference) not present")
def test_live_reference_fresh_programs():
    import ctypes as C

    from paper_1910_11110_b200.sweep import gen_program_text
    sys.path.insert(0, os.path.join(HERE, "golden"))
    from make_golden_cli import mutate, raw_of, ref_fn
    ref = ref_fn()
    rng = random.Random(7)
    for seed in range(5000, 5150):
        src = gen_program_text(seed)
        m = mutate(src, rng)
        for cmd in ("check", "infer", "translate"):
            c = ref(cmd, src)
            assert got(c) == want(c), (cmd, src)
            c = ref(cmd, m)
            assert got(c) == want(c), (cmd, m)
        c = ref("check", raw_of(src, rng), 1)
        assert got(c) == want(c)
    del C


@pytest.mark.gpu
def test_run_on_gpu_matches_reference(ctx):
    runs = [c for c in CASES if c["cmd"] in ("run", "trace")]
    assert len(runs) > 2500 and sum(1 for c in runs if c["cmd"] == "trace" or c["trace"]) > 150
    n_exec = 0
    for c in runs:
        assert got(c, ctx) == want(c), (c["src"], c["schedule"], c["fuel"], c["raw"])
        n_exec += c["exit"] in (0, 3, 4)
    assert n_exec > 2000


@pytest.mark.gpu
def test_run_json_on_gpu(ctx):
    out, err, code = run_cli("run", "scalar x\nw x;\ngr x;\n", ctx, raw=True, json=True)
    assert code == 3 and err == ""
    rec = [json.loads(x) for x in out.splitlines()]
    assert rec[0] == {"outcome": "stuck", "schedule_consumed": 0, "steps": 1,
                      "stuck": {"effect": "r", "have": "(V,I)", "key": "x", "site": "remote"}}
    assert rec[1:] == [{"key": "x", "local": "V", "remote": "I"}, {"key": "x^", "local": "V", "remote": "I"}]


WIDE = [
    # whole-view syncs over tens of thousands of cells, overlap shadows, scalars
    ("run", "scalar x\nbuffer b[65536]\nview v = b[0:40000]\nview u = b[30000:65535]\nview t = b[100:200]\n"
            "RW(v) { w v[5]; r v[39999]; }\nGR(u) { gr u[0]; }\nRW(x), R(t) { r t[3]; w x; }\n"
            "GRW(u) { gw u[7]; }\nR(v) { r v[30001]; }\n", 0, ""),
    ("run", "buffer b[70000]\nview v = b[0:69999]\nview w = b[12345:12400]\nGRW(w) { gw w[0]; }\nR(v) { r v[12345]; }\n"
            "RW(v) { w v[12345]; }\nGR(w) { gr w[3]; }\n", 0, ""),
    # raw: a stuck whole-view sync (the first failing cell, ascending) and fuel cut-offs
    ("run", "buffer b[100000]\nview v = b[5:99990]\nview u = b[50000:50010]\nw u[3];\ngw u[4];\npush v;\npull v;\n", 1, ""),
    ("run", "buffer b[4096]\nview v = b[0:4095]\nscalar s\nwhile (opaque) { push v; w s; }\npull v;\n", 1, "1101"),
    ("trace", "buffer b[300]\nview v = b[0:299]\nview u = b[250:299]\nGRW(u) { gw u[1]; }\nR(v) { r v[251]; }\n", 0, ""),
    ("trace", "scalar a\nscalar c\nbuffer b[40]\nview v = b[3:39]\nif (opaque) { push v; gw v[2]; pull v; } else { w a; }\n"
              "while (valid(a)) { gw a; }\nr c;\n", 1, "1"),
]


@pytest.mark.gpu
@pytest.mark.skipif(not o.have_ref(), reason="oracle/_ref (the compiled reference) not present")
def test_run_wide_programs_match_live_reference(ctx):
    """Programs far beyond 32 store keys (buffers up to 100000 cells) run on the bit-plane
    interpreter and match the reference CLI byte for byte, text and JSON, with and without
    the step trace, and with a small fuel."""
    sys.path.insert(0, os.path.join(HERE, "golden"))
    from make_golden_cli import ref_fn
    ref = ref_fn()
    for cmd, src, raw, sched in WIDE:
        for fuel in (10000, 7):
            c = ref(cmd, src, raw, 0, fuel, sched)
            assert got(c, ctx) == want(c), (cmd, src, fuel)
            if cmd == "run" and len(src) < 200 and "b[4096]" in src:
                c2 = dict(c, trace=1)
                r2 = ref(cmd, src, raw, 0, fuel, sched, 1)
                assert got(c2, ctx) == want(r2), (src, fuel)
        out, err, code = run_cli(cmd, src, ctx, raw=bool(raw), json=True, schedule=sched or None)
        assert code == ref(cmd, src, raw, 0, 10000, sched)["exit"]
        assert all(line.startswith("{") for line in out.splitlines())


def test_batched_host_passes_match_reference():
    """coh_cli_batch (the batched checker): every host case of the
    reference-made corpus, grouped by command and flags and evaluated on the host threads,
    gives the reference's bytes and exit codes."""
    from paper_1910_11110_b200.cli import run_cli_batch
    groups = {}
    for c in CASES:
        if c["cmd"] in ("check", "infer", "translate"):
            groups.setdefault((c["cmd"], bool(c["raw"]), bool(c["no_overlap"])), []).append(c)
    n = 0
    for (cmd, raw, no_ovl), cs in groups.items():
        got_all = run_cli_batch(cmd, [c["src"] for c in cs], raw=raw, no_overlap=no_ovl)
        for c, g in zip(cs, got_all):
            assert g == want(c), (cmd, c["src"])
        n += len(cs)
    assert n > 2000
    from paper_1910_11110_b200 import CohError
    with pytest.raises(CohError):
        run_cli_batch("run", ["scalar x\n"])
