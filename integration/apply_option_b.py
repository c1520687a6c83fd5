"""Apply INTEGRATION.md "Option B" to a COPY of an installed minmapcc package:
copy the package, add minmapcc/_cuda.py (integration/minmapcc_cuda.py) and
insert the maintainer's dispatch at the top of engine.run_contour
(engine.py:266) -- with MINMAPCC_DEVICE=cuda every caller of run_contour
(bench.run_experiment, cli, tests) then runs on the GPU.

    python integration/apply_option_b.py <installed minmapcc dir> <target dir>

The original package is never modified."""
import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))

DISPATCH = '''    if os.environ.get("MINMAPCC_DEVICE") == "cuda":  # Option B (INTEGRATION.md)
        if threads < 1:
            raise ValueError("threads must be >= 1")
        from ._cuda import run_contour_cuda
        return run_contour_cuda(g, schedule)
'''


def apply(src_pkg: str, dst_parent: str) -> str:
    dst = os.path.join(dst_parent, "minmapcc")
    shutil.copytree(src_pkg, dst, ignore=shutil.ignore_patterns("__pycache__", "*.nbi", "*.nbc"))
    shutil.copy(os.path.join(HERE, "minmapcc_cuda.py"), os.path.join(dst, "_cuda.py"))
    path = os.path.join(dst, "engine.py")
    with open(path) as fh:
        src = fh.read()
    head = "def run_contour("
    i = src.index(head)
    body = src.index('    if threads < 1:', i)  # first statement after the docstring
    src = src[:body] + DISPATCH + src[body:]
    if "\nimport os\n" not in src:
        src = src.replace("\nimport time\n", "\nimport os\nimport time\n", 1)
    with open(path, "w") as fh:
        fh.write(src)
    return dst


if __name__ == "__main__":
    print(apply(sys.argv[1], sys.argv[2]))
