#!/usr/bin/env python3
"""Build step (test infrastructure): writes the public-API part of a reference
doctest file to OUT, so the reference's OWN test cases can be compiled against
the drop-in headers and library (oracle/Makefile target `dropin-tests`).

Drops (by brace matching, nothing else is changed):
  * TEST_CASEs whose name starts with one of --drop-case prefixes
    (e.g. "tile sweep": they drive tile internals sweep_tile_slice / Tensor3);
  * helper functions named by --drop-fn (their only callers are dropped cases).

The output goes to oracle/_ref/gen/ (git-ignored build output), never into the
tracked tree: reference sources are not copied into the repository.

usage: public_cases.py SRC OUT [--drop-case PREFIX ...] [--drop-fn NAME ...]
"""
import argparse
import re


def block_end(text: str, start: int) -> int:
    """Index one past the brace block whose '{' is the first at/after start."""
    i = text.index("{", start)
    depth = 0
    while True:
        ch = text[i]
        if ch == "{":
            depth += 1
        elif ch == "}":
            depth -= 1
            if depth == 0:
                return i + 1
        elif ch == '"':  # skip string literals
            i += 1
            while text[i] != '"':
                i += 2 if text[i] == "\\" else 1
        i += 1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("src")
    ap.add_argument("out")
    ap.add_argument("--drop-case", nargs="*", default=[])
    ap.add_argument("--drop-fn", nargs="*", default=[])
    a = ap.parse_args()
    text = open(a.src).read()
    cuts = []
    for m in re.finditer(r'^TEST_CASE\("([^"]*)"\)', text, re.M):
        if any(m.group(1).startswith(p) for p in a.drop_case):
            cuts.append((m.start(), block_end(text, m.end())))
    for name in a.drop_fn:
        m = re.search(r"^[^\n;{}]*\b" + re.escape(name) + r"\(", text, re.M)
        if m:
            # include the comment block right above the function
            start = m.start()
            while True:
                prev = text.rfind("\n", 0, start - 1)
                line = text[prev + 1:start - 1] if prev >= 0 else ""
                if line.lstrip().startswith("//"):
                    start = prev + 1
                else:
                    break
            cuts.append((start, block_end(text, m.end())))
    for s, e in sorted(cuts, reverse=True):
        text = text[:s] + text[e:]
    with open(a.out, "w") as f:
        f.write(f"// generated from {a.src} by oracle/public_cases.py (public-API cases only)\n")
        f.write(text)


if __name__ == "__main__":
    main()
