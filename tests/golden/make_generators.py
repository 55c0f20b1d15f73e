#!/usr/bin/env python
"""Golden digests of the reference's dataset generators (run in the build
container, where /root/reference exists).  Compiles a tiny driver against the
UNMODIFIED reference headers (knng::gen_gaussian / gen_clustered /
save_binary, dataset.hpp:99-233), runs it into /tmp, and records the SHA-256 of
each KNNG file and labels list in tests/golden/generators.json.  The CLI's
`generate` must reproduce them byte for byte (tests/test_cli.py)."""
import hashlib
import json
import os
import subprocess
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = [("gaussian", 500, 12, 8, 5), ("gaussian-single", 300, 7, 8, 9),
         ("clustered", 2000, 8, 4, 3), ("clustered", 1000, 3, 5, 11)]
DRIVER = r'''
#include <knng/dataset.hpp>
#include <cstdio>
#include <string>
int main(int argc, char** argv) {
    const std::string kind = argv[1];
    const unsigned n = std::stoul(argv[2]), d = std::stoul(argv[3]), c = std::stoul(argv[4]);
    const unsigned long long seed = std::stoull(argv[5]);
    if (kind == "clustered") {
        auto [ds, lab] = knng::gen_clustered(n, d, c, seed);
        knng::save_binary(ds, argv[6]);
        FILE* f = std::fopen(argv[7], "w");
        for (auto l : lab.labels) std::fprintf(f, "%u\n", l);
        std::fclose(f);
    } else {
        knng::save_binary(knng::gen_gaussian(n, d, kind == "gaussian-single", seed), argv[6]);
    }
}
'''


def sha(path):
    return hashlib.sha256(open(path, "rb").read()).hexdigest()


def main():
    tmp = tempfile.mkdtemp()
    src = os.path.join(tmp, "gen.cpp")
    exe = os.path.join(tmp, "gen")
    open(src, "w").write(DRIVER)
    subprocess.run(["g++", "-std=gnu++20", "-O2", "-I/root/reference/proj/include", src, "-o", exe],
                   check=True)
    out = []
    for kind, n, d, c, seed in CASES:
        ds, lab = os.path.join(tmp, "d.knng"), os.path.join(tmp, "l.txt")
        subprocess.run([exe, kind, str(n), str(d), str(c), str(seed), ds, lab], check=True)
        rec = {"kind": kind, "n": n, "d": d, "c": c, "seed": seed, "dataset_sha256": sha(ds)}
        if kind == "clustered":
            rec["labels_sha256"] = sha(lab)
        out.append(rec)
    json.dump(out, open(os.path.join(HERE, "generators.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
