"""TEST INFRASTRUCTURE ONLY — the CPU checkers of the parity suite.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this package.  The product path (paper_2201_09147_b200, libnsdf_cuda.so,
libnsdf_b200.so) never does.

  oracle.refshim  ctypes over _ref/libnsdf_ref.so — the unmodified reference library
                  compiled from /root/reference/proj/src by oracle/Makefile.
  oracle.corc     ctypes over _ref/libnsdf_oracle.so — our plain-C restatement
                  (nsdf_oracle.c), pinned bit-for-bit to the reference by
                  tests/test_oracle.py.
"""
import os

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")


def build(force: bool = False) -> None:
    """Compile the checkers (the restatement always; the reference only where
    /root/reference exists — on the GPU box the prebuilt .so files travel)."""
    import subprocess

    targets = ["oracle"]
    if os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    cmd = ["make", "-C", HERE, "-j8"] + targets
    if force:
        cmd.insert(1, "-B")
    subprocess.run(cmd, check=True, stdout=subprocess.DEVNULL)
