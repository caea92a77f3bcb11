"""Generate tests/golden/ref_cli_text.json from the REFERENCE ITSELF: the text the reference's
`ph0` CLI (proj/tools/ph0_cli.cpp) prints for each case, produced through oracle/_ref's
ref_cli_text (the unmodified read_points / generate_uniform_cloud / pipeline / kruskal_barcode
/ format_barcode / write_points of /root/reference/proj/src).  Run in the build container:

    make -C oracle ref && python tests/golden/make_text_golden.py

Each case: the argv of our `ph0b` CLI (with "{in}" standing for the input file), the input
file text (or null), and the expected stdout / stderr / exit code.
"""
from __future__ import annotations

import ctypes as C
import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT / "tests"))

import oracle_bridge as ob  # noqa: E402


def ref_text(points: str | None, mode: int, show_essential: bool = False,
             gen=(0, 0, 0)) -> tuple[int, str]:
    L = ob.ref()
    L.ref_cli_text.restype = C.c_int
    L.ref_cli_text.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, C.c_int,
                               C.c_char_p, C.c_uint64, C.POINTER(C.c_uint64)]
    n = C.c_uint64(0)
    src = points.encode() if points is not None else None
    rc = L.ref_cli_text(src, gen[0], gen[1], gen[2], mode, int(show_essential), None, 0,
                        C.byref(n))
    buf = C.create_string_buffer(n.value + 1)
    rc = L.ref_cli_text(src, gen[0], gen[1], gen[2], mode, int(show_essential), buf,
                        n.value + 1, C.byref(n))
    return rc, buf.value.decode()


def main():
    collinear = Path("/root/reference/proj/data/collinear3.txt").read_text()  # acceptance.cpp:321
    _, uniform37 = ref_text(None, 2, gen=(37, 3, 2024))  # test_point_cloud.cpp:91-97
    lattice = "".join(f"{x},{y}\n" for x in range(6) for y in range(6))
    cases = []

    def add(name, argv, points=None, mode=0, show=False, gen=(0, 0, 0), stdin_text=None):
        rc, text = ref_text(stdin_text if stdin_text is not None else points, mode, show, gen)
        cases.append({"name": name, "argv": argv, "input": points,
                      "rc": rc, "stdout": text if rc == 0 else "",
                      "stderr": text if rc != 0 else "",
                      "gpu": mode in (0, 1) and rc == 0})

    for cmd, mode in (("compute", 0), ("oracle", 1)):
        add(f"{cmd}_collinear3", [cmd, "--in", "{in}"], collinear, mode)
        add(f"{cmd}_collinear3_essential", [cmd, "--in", "{in}", "--show-essential"], collinear,
            mode, True)
        add(f"{cmd}_uniform37", [cmd, "--in", "{in}"], uniform37, mode)
        add(f"{cmd}_lattice_ties", [cmd, "--in={in}"], lattice, mode)
        add(f"{cmd}_generated", [cmd, "--n", "60", "--dim", "3", "--seed", "9"], None, mode,
            gen=(60, 3, 9), stdin_text=None)
        add(f"{cmd}_generated_defaults", [cmd, "--n", "50", "--show-essential"], None, mode, True,
            gen=(50, 2, 1))
    add("compute_mixed_separators", ["compute", "--in", "{in}"], "# comment\n 1.5\t2.5\n3,4\n\n")
    add("compute_coincident", ["compute", "--in", "{in}", "--show-essential"], "1,1\n1,1\n1,1\n",
        0, True)
    add("compute_single_point", ["compute", "--in", "{in}", "--show-essential"], "5,5\n", 0, True)
    add("compute_workers_pivot", ["compute", "--in", "{in}", "--workers", "4", "--pivot", "off"],
        uniform37)
    add("generate_37_3_2024", ["generate", "--n", "37", "--dim", "3", "--seed", "2024"], None, 2,
        gen=(37, 3, 2024))
    add("generate_defaults", ["generate", "--n", "5"], None, 2, gen=(5, 2, 1))
    add("generate_dim0", ["generate", "--n", "3", "--dim", "0"], None, 2, gen=(3, 0, 1))
    add("parse_dim_mismatch", ["compute", "--in", "{in}"], "0,0\n1,2,3\n")       # test_point_cloud.cpp:76-79
    add("parse_malformed", ["compute", "--in", "{in}"], "1,2\nx,3\n")            # :81-84
    add("parse_nonfinite", ["oracle", "--in", "{in}"], "1,inf\n")                # :86-89
    add("parse_nan", ["compute", "--in", "{in}"], "# c\n\nnan,1\n")
    add("compute_empty_input", ["compute", "--in", "{in}", "--show-essential"], "")  # :71-74
    add("oracle_comments_only", ["oracle", "--in", "{in}"], "# nothing\n\n")
    # the two messages below are the reference's literal texts (no input to run it on)
    cases.append({"name": "missing_file", "argv": ["compute", "--in", "/nonexistent/pts.txt"],
                  "input": None, "rc": 1, "stdout": "", "gpu": False,
                  "stderr": "error: cannot open point file '/nonexistent/pts.txt'\n"})  # point_cloud.cpp:94
    cases.append({"name": "missing_source", "argv": ["oracle"], "input": None, "rc": 1,
                  "stdout": "", "gpu": False,
                  "stderr": "error: either --in or --n is required\n"})  # ph0_cli.cpp:33-35
    out = HERE / "ref_cli_text.json"
    out.write_text(json.dumps({"source": "oracle/_ref ref_cli_text (reference sources)",
                               "cases": cases}, indent=1))
    print(f"wrote {out} ({len(cases)} cases)")


if __name__ == "__main__":
    main()
