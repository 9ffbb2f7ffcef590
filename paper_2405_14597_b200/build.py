"""In-tree build of the sm_100a library and the C++ drop-in layer (nvcc/g++ cross-compile;
no GPU needed)."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))


def build(jobs: int = 8, verbose: bool = False) -> None:
    out = None if verbose else subprocess.DEVNULL
    subprocess.run(["make", "-j", str(jobs), "-C", os.path.join(HERE, "csrc")], check=True,
                   stdout=out)
    host = os.path.join(HERE, "host")
    if os.path.exists(os.path.join(host, "Makefile")):
        subprocess.run(["make", "-j", str(jobs), "-C", host], check=True, stdout=out)


if __name__ == "__main__":
    build(verbose=True)
