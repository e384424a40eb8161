"""Regenerates tests/golden/rng_ref.json from the REFERENCE's own rng.hpp.

Compiles oracle/ref_rng_driver.cpp with -I/root/reference/proj/include into
oracle/_ref/ref_rng_driver (git-ignored) and stores its JSON output. Needs
/root/reference (this container only); the fixture it writes is committed.
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
REF_INC = "/root/reference/proj/include"


def main() -> int:
    out_dir = os.path.join(ROOT, "oracle", "_ref")
    os.makedirs(out_dir, exist_ok=True)
    exe = os.path.join(out_dir, "ref_rng_driver")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", REF_INC,
                    os.path.join(ROOT, "oracle", "ref_rng_driver.cpp"), "-o", exe], check=True)
    text = subprocess.run([exe], check=True, capture_output=True, text=True).stdout
    with open(os.path.join(ROOT, "tests", "golden", "rng_ref.json"), "w") as f:
        f.write(text)
    print(text)
    return 0


if __name__ == "__main__":
    sys.exit(main())
