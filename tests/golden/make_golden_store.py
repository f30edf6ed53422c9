#!/usr/bin/env python
"""Golden files for the store-writer / word-file / CLI rows, produced by
running the UNMODIFIED Python reference (its own ``phonsim ingest`` and ``phonsim compute`` commands).

Run in the build container only:   python tests/golden/make_golden_store.py

Writes tests/golden/store_case/: the toy corpus, the reference's .words / .inventory files, the
reference's .nwedges payload and manifest for two schemes, and the text ``phonsim compute`` printed.
"""
from __future__ import annotations

import contextlib
import io
import json
import re
import sys
from pathlib import Path

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
OUT = HERE / "store_case"

from phonsim import cli  # noqa: E402

# a small French-looking corpus (word, ipa, frequency): tie bars, nasal vowels, a digraph
CORPUS = [
    ("puissance", "pɥisɑ̃s", 50.0), ("nuance", "nɥɑ̃s", 49.0), ("puisant", "pɥizɑ̃", 48.5),
    ("paysans", "peizɑ̃", 47.0), ("épuisant", "epɥizɑ̃", 46.0), ("trottoir", "tʁɔtwaʁ", 45.0),
    ("falaise", "falɛz", 44.0), ("emporter", "ɑ̃pɔʁte", 43.0), ("tchèque", "t͡ʃɛk", 42.0),
    ("djinn", "d͡ʒin", 41.0), ("chat", "ʃa", 40.0), ("chats", "ʃa", 39.0), ("eau", "o", 38.0),
    ("oiseau", "wazo", 37.0), ("anticonstitutionnellement", "ɑ̃tikɔ̃stitysjɔnɛlmɑ̃", 36.0),
    ("roi", "ʁwa", 35.0), ("loi", "lwa", 34.0), ("foi", "fwa", 33.0), ("fois", "fwa", 32.0),
    ("froid", "fʁwa", 31.0), ("droit", "dʁwa", 30.0), ("étroit", "etʁwa", 29.0),
    ("pain", "pɛ̃", 28.0), ("bain", "bɛ̃", 27.0), ("main", "mɛ̃", 26.0), ("demain", "dəmɛ̃", 25.0),
]


def run(argv):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = cli.main(argv)
    assert rc == 0, (argv, rc)
    return buf.getvalue()


def main():
    OUT.mkdir(exist_ok=True)
    corpus = OUT / "toy.tsv"
    corpus.write_text("".join(f"{w}\t{i}\t{f}\n" for w, i, f in CORPUS), encoding="utf-8")
    run(["ingest", str(corpus), "--out", str(OUT / "toy")])
    printed = {}
    for tag, (m, x, g) in {"s1": (1, -1, -1), "s2": (2, -1, -3)}.items():
        text = run(["compute", str(OUT / "toy.words"), "--match", str(m), "--mismatch", str(x), "--gap", str(g),
                    "--workers", "1", "--chunk-size", "37", "--out", str(OUT / f"toy_{tag}")])
        text = re.sub(r"in \d+\.\d+ s", "in <T> s", text).replace(str(OUT) + "/", "")
        printed[tag] = {"scheme": [m, x, g], "stdout": text}
    # a scheme FILE with per-pair overrides (cli.py:167-174, aligner.py:195-239), resolved against toy.inventory
    (OUT / "scheme_s3.txt").write_text("# nasal vowels and the two affricates count as near-matches\nmatch\t2\nmismatch\t-1\n"
                                       "gap\t-2\n\n\u0251\u0303\t\u025b\u0303\t1\nt\u0283\td\u0292\t1\n\u0283\ts\t0\n", encoding="utf-8")
    text = run(["compute", str(OUT / "toy.words"), "--scheme", str(OUT / "scheme_s3.txt"), "--workers", "2",
                "--chunk-size", "50", "--out", str(OUT / "toy_s3")])
    text = re.sub(r"in \d+\.\d+ s", "in <T> s", text).replace(str(OUT) + "/", "")
    printed["s3"] = {"scheme_file": "scheme_s3.txt", "stdout": text}
    (OUT / "compute_stdout.json").write_text(json.dumps(printed, ensure_ascii=False, indent=1), encoding="utf-8")
    for p in sorted(OUT.iterdir()):
        print(p.name, p.stat().st_size)


if __name__ == "__main__":
    main()
