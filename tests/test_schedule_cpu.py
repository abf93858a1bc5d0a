"""The contraction's lag-column schedule (csrc/cw_frame.cuh: smsp_sched) is
a constexpr function the fused kernel unrolls at compile time; this CPU test
compiles the same source with the host compiler and checks, for every
symmetric grid half-width C0 and warp count the kernel can see, that each
column pair q = 0..C0 is dealt to exactly one warp (or the schedule reports
itself unusable and the kernel falls back to round robin), and that the
default geometry gets the balanced counts DESIGN.md §5 states."""

import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_1408_3526_b200", "csrc", "cw_frame.cuh")


def _schedule_source():
    s = open(SRC).read()
    a = s.index("struct SmspSched")
    b = s.index("struct alignas(16) LagRec")
    return s[a:b]


@pytest.fixture(scope="module")
def sched_bin(tmp_path_factory):
    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("no host C++ compiler")
    d = tmp_path_factory.mktemp("sched")
    src = d / "sched.cpp"
    src.write_text(
        "#define __host__\n#define __device__\n#define CW_SMSP_FIX 1\n#include <cstdio>\n"
        + _schedule_source()
        + r"""
int main() {
    for (int nr = 2; nr <= 8; nr++)
        for (int c0 = 1; c0 <= 16; c0++) {
            SmspSched s = smsp_sched(c0, nr);
            printf("%d %d %d", c0, nr, s.ok ? 1 : 0);
            for (int w = 0; w < nr; w++) {
                printf(" |");
                unsigned code = s.code[w];
                for (int k = 0; k < 6 && (code & 31u) != 31u; k++, code >>= 5) printf(" %u", code & 31u);
            }
            printf("\n");
        }
}
""")
    exe = d / "sched"
    subprocess.run([gxx, "-std=c++17", "-O1", "-o", str(exe), str(src)], check=True)
    return exe


def _parse(exe):
    out = {}
    for line in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines():
        head, *warps = line.split("|")
        c0, nr, ok = (int(v) for v in head.split())
        out[(c0, nr)] = (ok, [[int(v) for v in w.split()] for w in warps])
    return out


def test_every_pair_is_dealt_once(sched_bin):
    res = _parse(sched_bin)
    for (c0, nr), (ok, warps) in res.items():
        if not ok:
            continue
        assert len(warps) == nr
        got = sorted(q for w in warps for q in w)
        assert got == list(range(c0 + 1)), (c0, nr, warps)
        assert all(len(w) <= 6 for w in warps)


def test_default_geometries_are_balanced(sched_bin):
    res = _parse(sched_bin)
    # 5 warps (KY = 4): 17 and 33 lags get the SM-mate-balanced counts
    assert res[(8, 5)][0] and [len(w) for w in res[(8, 5)][1]] == [1, 2, 3, 2, 1]
    assert res[(16, 5)][0] and [len(w) for w in res[(16, 5)][1]] == [2, 4, 5, 4, 2]
    # 4 warps (KY = 3): one warp per scheduler, an even deal
    counts = [len(w) for w in res[(16, 4)][1]]
    assert res[(16, 4)][0] and max(counts) - min(counts) <= 1
