#!/usr/bin/env python3
"""Resolve every `file.ext:N[-M]` citation of the reference in this repo's sources and docs
against /root/reference/proj: the file must exist (unique basename) and the lines must lie
inside it.  Prints the offenders; exit 1 if any.  (tests/test_cites.py runs it.)"""
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.environ.get("RW_REF_ROOT", "/root/reference/proj")
CITE = re.compile(r"\b([A-Za-z_][A-Za-z0-9_]*\.(?:cpp|hpp))[: ]+:?(\d+)(?:-(\d+))?")
SCAN_EXT = (".py", ".cpp", ".cu", ".cuh", ".h", ".c", ".md")
SKIP_DIRS = {".git", "gpurun_out", "__pycache__", "_ref", "_build", "build", "baseline"}
SKIP_FILES = {"SURVEY.md", "VERDICT.md", "ADVICE.md", "BASELINE.md", "PAPERS.md", "SNIPPETS.md"}


def ref_files():
    out = {}
    for d, _, fs in os.walk(REF):
        for f in fs:
            out.setdefault(f, []).append(os.path.join(d, f))
    return out


def main():
    files = ref_files()
    lengths = {}
    bad = []
    n = 0
    for d, dirs, fs in os.walk(ROOT):
        dirs[:] = [x for x in dirs if x not in SKIP_DIRS]
        for f in fs:
            if not f.endswith(SCAN_EXT) or f in SKIP_FILES:
                continue
            path = os.path.join(d, f)
            with open(path, errors="replace") as fh:
                for ln_no, line in enumerate(fh, 1):
                    for mm in re.finditer(r"\b([A-Za-z_][A-Za-z0-9_]*\.(?:cpp|hpp)):(\d+)(?:-(\d+))?",
                                          line):
                        name, a, b = mm.group(1), int(mm.group(2)), mm.group(3)
                        b = int(b) if b else a
                        if name not in files:
                            continue  # one of ours (rw_abi.cpp:...) or not a reference file
                        n += 1
                        if len(files[name]) != 1:
                            continue
                        ref = files[name][0]
                        if ref not in lengths:
                            with open(ref, errors="replace") as rf:
                                lengths[ref] = sum(1 for _ in rf)
                        if not (1 <= a <= b <= lengths[ref]):
                            bad.append(f"{os.path.relpath(path, ROOT)}:{ln_no}: {name}:{a}-{b} "
                                       f"(file has {lengths[ref]} lines)")
    for x in bad:
        print(x)
    print(f"{n} citations checked, {len(bad)} out of range", file=sys.stderr)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
