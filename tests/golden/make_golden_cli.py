"""Regenerate the CLI golden fixtures from the REFERENCE itself (oracle/_ref ref_cli: the
reference headers compiled in place, tools/cohere_main.cpp's text reporting).  Run in the
build container (where /root/reference exists):

    make -C oracle && python tests/golden/make_golden_cli.py

Output (committed): cli.json.gz, one record per case
  {cmd, src, raw, no_overlap, fuel, schedule, trace, out, err, exit}
Corpus:
  * the reference's samples/*.coh under every command and flag combination, traces included (their
    outputs include the reference's own tests/golden/*.txt, checked here);
  * gen_well_declared programs (coh_gen_program_text, text-identical to the reference
    generator) under run (several schedules and fuels), infer, translate, check;
  * mutants of those programs (mode kinds/sites flipped, statements dropped, raw bodies
    with syncs, truncated text) for diagnostics, stuck runs and parse errors;
  * hand-written edge cases (every ParseError / ConstructionError path, overlap conflicts).
"""
import ctypes as C
import glob
import gzip
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [os.path.dirname(HERE), ROOT]

import oracle_ffi as o  # noqa: E402
from paper_1910_11110_b200.sweep import gen_program_text  # noqa: E402

REF_SAMPLES = "/root/reference/proj/samples"
REF_GOLDEN = "/root/reference/proj/tests/golden"


def ref_fn():
    R = o.reference()
    R.ref_cli.restype = C.c_int
    R.ref_cli.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_int, C.c_char_p,
                          C.c_size_t, C.c_char_p, C.c_size_t, C.POINTER(C.c_int)]

    def call(cmd, src, raw=0, no_overlap=0, fuel=10000, schedule="", trace=0):
        cap = 1 << 24
        out, err, code = C.create_string_buffer(cap), C.create_string_buffer(cap), C.c_int()
        rc = R.ref_cli(cmd.encode(), src.encode(), raw, no_overlap, fuel, schedule.encode(), trace, out, cap, err, cap,
                       C.byref(code))
        assert rc == 0
        return dict(cmd=cmd, src=src, raw=raw, no_overlap=no_overlap, fuel=fuel, schedule=schedule, trace=trace,
                    out=out.value.decode(), err=err.value.decode(), exit=code.value)
    return call


EDGE = [
    ("check", "scalar x\nscalar x\n"), ("check", "buffer b[0]\n"), ("check", "buffer b[2]\nbuffer b[3]\n"),
    ("check", "view v = b[0:1]\n"), ("check", "buffer b[4]\nview v = b[2:9]\n"), ("check", "buffer b[4]\nview v = b[3:1]\n"),
    ("check", "scalar if\n"), ("check", "scalar x\nR(x) { r x; }\nscalar y\n"), ("check", "scalar x\nR(y) { }\n"),
    ("check", "scalar x\nR(x), W(x) { r x; }\n"), ("check", "scalar x\nQ(x) { }\n"), ("check", "scalar x\nR(x) { r x }\n"),
    ("check", "scalar x\n{ r x[1]; }\n"), ("check", "buffer b[4]\nview v = b[0:3]\n{ r v; }\n"),
    ("check", "buffer b[4]\nview v = b[0:3]\n{ push v[1]; }\n"), ("check", "buffer b[4]\nview v = b[0:3]\n{ r v[4]; }\n"),
    ("check", "scalar x\n{ r z; }\n"), ("check", "scalar x\n{ if (valid(z)) { } }\n"), ("check", "scalar x\n{ if (maybe) { } }\n"),
    ("check", "scalar x\n{ r x; } /* unterminated\n"), ("check", "scalar x\n{ r x; } @\n"),
    ("check", "scalar x\nW(x) { if (opaque) { w x; } }\n"), ("check", "scalar x\nW(x) { while (opaque) { w x; } }\n"),
    ("check", "scalar x\nRW(x) { if (opaque) { w x; } else { w x; } }\n"), ("check", "scalar x\nR(x) { gr x; w x; push x; }\n"),
    ("check", "scalar x\nR(x) { }\n"), ("check", "scalar x\nGR(x) /*shadow*/ { }\n"), ("check", "scalar x\nR(x) { r x; gr x; }\n"),
    ("check", "buffer b[4]\nview v = b[0:3]\nview u = b[2:3]\nW(v) { w v[0]; w v[1]; w v[2]; w v[3]; }\n"),
    ("check", "buffer b[4]\nview v = b[0:3]\nW(v) { w v[0]; if (opaque) { w v[1]; } w v[2]; w v[3]; }\n"),
    ("check", "scalar x\n{ r x; } // trailing comment"), ("check", "scalar x\n{ r x; } /*  shadow */"),
    ("run", "buffer b[4]\nview v = b[0:1]\nview u = b[1:2]\nW(v), GW(u) { w v[0]; w v[1]; gw u[0]; gw u[1]; }\n"),
    ("run", "buffer b[4]\nview v = b[0:1]\nview u = b[1:2]\nRW(v), GRW(u) { w v[0]; gw u[1]; }\n"),
    ("run", "scalar x\nGRW(x) { gw x; }\nR(x) { r x; }\nGR(x) { gr x; }\n"),
    ("run", "buffer b[3]\nview v = b[0:2]\nGW(v) { gw v[0]; gw v[1]; gw v[2]; }\nR(v) { r v[1]; }\n"),
    ("run", "scalar x\n{ while (opaque) { } }\n"), ("run", "scalar x\nRW(x) { while (valid(x)) { w x; } }\n"),
    ("infer", "buffer b[6]\nview a = b[0:3]\nview c = b[2:5]\nview d = b[5:5]\nRW(a), GW(d) { w a[0]; gw d[0]; }\n"),
    ("translate", "buffer b[6]\nview a = b[0:3]\nview c = b[2:5]\nGRW(c), R(a) { gw c[0]; r a[1]; }\n"),
]
RAW_EDGE = [
    ("run", "scalar x\nw x;\ngr x;\n"), ("run", "scalar x\nw x;\npush x;\ngr x;\n"),
    ("run", "buffer b[3]\nview v = b[0:2]\ngw v[1];\npull v;\n"), ("run", "buffer b[3]\nview v = b[0:2]\ngw v[1];\npush v;\n"),
    ("run", "buffer b[3]\nview v = b[0:2]\nw v[0];\npush v;\npull v;\ngr v[2];\n"),
    ("run", "scalar x\nwhile (opaque) { push x; }\n"), ("run", "scalar x\nif (gvalid(x)) { gr x; } else { push x; gr x; }\n"),
    ("run", "scalar x\nif (valid(x^)) { pull x; } else { w x; }\n"), ("check", "scalar x\nw x;\ngw x;\n"),
    ("infer", "scalar x\nw x;\n"), ("translate", "scalar x\nw x;\n"), ("run", "scalar x\nR(x) { r x; }\n"),
]


def mutate(src, rng):
    lines = src.split("\n")
    k = rng.randrange(4)
    if k == 0:  # flip a mode word
        words = ["R", "W", "RW", "GR", "GW", "GRW"]
        for i, ln in enumerate(lines):
            if ln.endswith("{") and "(" in ln and rng.random() < 0.6:
                head, rest = ln.split("(", 1)
                parts = head.split(", ")
                parts[-1] = rng.choice(words)
                lines[i] = ", ".join(parts) + "(" + rest
                break
    elif k == 1:  # drop a body statement
        body = [i for i, ln in enumerate(lines) if ln.startswith("  ") and ln.strip().endswith(";")]
        if body:
            del lines[rng.choice(body)]
    elif k == 2:  # add a stray effect
        body = [i for i, ln in enumerate(lines) if ln.startswith("  ")]
        if body:
            i = rng.choice(body)
            lines.insert(i, "  " + rng.choice(["gr", "r", "w", "gw", "push", "pull"]) + " s0;")
    else:  # truncate
        cut = rng.randrange(max(1, len(src)))
        return src[:cut]
    return "\n".join(lines)


def raw_of(src, rng):
    """Declarations + all block bodies as bare statements, with random syncs added."""
    out, decls = [], True
    for ln in src.split("\n"):
        if decls and (ln.startswith("scalar") or ln.startswith("buffer") or ln.startswith("view")):
            out.append(ln)
            continue
        decls = False
        s = ln.strip()
        if not s or (s.endswith("{") and "(" in s and not s.startswith(("if", "while", "}"))) or s == "{":
            continue
        if s == "}" and not ln.startswith(" "):
            continue
        out.append(ln)
        if s.endswith(";") and rng.random() < 0.3:
            out.append(ln[: len(ln) - len(ln.lstrip())] + rng.choice(["push", "pull"]) + " s0;")
    return "\n".join(out) + "\n"


def main():
    assert o.have_ref(), "build oracle/_ref first (make -C oracle)"
    ref = ref_fn()
    cases = []
    # 1. the reference samples, every command and flag; the reference goldens must agree
    samples = sorted(glob.glob(os.path.join(REF_SAMPLES, "*.coh")))
    for f in samples:
        src = open(f).read()
        for cmd in ("check", "run", "infer", "translate"):
            for raw in (0, 1):
                for no in (0, 1):
                    cases.append(ref(cmd, src, raw, no))
        for sched in ("0", "1", "0101"):
            cases.append(ref("run", src, 0, 0, 10000, sched))
        for raw in (0, 1):
            cases.append(ref("trace", src, raw))
            cases.append(ref("run", src, raw, 0, 4, "1", 1))
        for fuel in (1, 2, 3, 5):
            cases.append(ref("run", src, 0, 0, fuel))
    for g in sorted(glob.glob(os.path.join(REF_GOLDEN, "*.txt"))):
        stem, cmd = os.path.basename(g)[:-4].rsplit(".", 1)
        src = open(os.path.join(REF_SAMPLES, stem + ".coh")).read()
        raw = 1 if stem.endswith("_raw") else 0
        got = ref(cmd, src, raw)
        assert got["out"] == open(g).read(), g  # the harness reproduces the reference goldens
    # 2. generated well-declared programs, 3. mutants and raw bodies
    rng = random.Random(1910)
    for seed in range(400):
        src = gen_program_text(seed)
        cases.append(ref("run", src))
        for _ in range(2):
            sched = "".join(rng.choice("01") for _ in range(rng.randrange(1, 9)))
            cases.append(ref("run", src, 0, 0, 10000, sched))
        cases.append(ref("run", src, 0, 0, rng.randrange(1, 12), "1" * rng.randrange(0, 4)))
        cases.append(ref("run", src, 0, 1))
        if seed % 4 == 0:
            cases.append(ref("trace", src, 0, 0, 10000, "".join(rng.choice("01") for _ in range(6))))
        for cmd in ("check", "infer", "translate"):
            cases.append(ref(cmd, src))
        m = mutate(src, rng)
        cases.append(ref("check", m))
        cases.append(ref("run", m, 0, 0, 10000, "01"))
        r = raw_of(src, rng)
        cases.append(ref("run", r, 1, 0, 10000, "10", seed % 5 == 0))
        cases.append(ref("check", r, 1))
    # 4. edge cases
    for cmd, src in EDGE:
        for no in (0, 1):
            cases.append(ref(cmd, src, 0, no))
    for cmd, src in RAW_EDGE:
        cases.append(ref(cmd, src, 1, 0, 10000, "110"))
        cases.append(ref(cmd, src, 1, 0, 10000, "110", 1))
    cases.append(ref("run", "scalar x\nR(x) { r x; }\n", 0, 0, 10000, "012"))  # bad schedule
    with gzip.open(os.path.join(HERE, "cli.json.gz"), "wt") as f:
        json.dump(cases, f)
    exits = {}
    for c in cases:
        exits[(c["cmd"], c["exit"])] = exits.get((c["cmd"], c["exit"]), 0) + 1
    print(len(cases), "cases", sorted(exits.items()))


if __name__ == "__main__":
    main()
