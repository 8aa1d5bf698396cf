"""The reference's own benchmark harness (`softmpm bench`: cli.cmd_bench,
cli.py:177-207 -- the collider-free push scene, median soft_simulation ms
per frame) run twice on this box: natively (numba, all host threads) and with
the hot path re-routed to the B200 by paper_2402_01181_b200.install().  The
installed timing includes install()'s per-step upload of the reference's
fp64 numpy state (its host-buffer path).  Needs baseline/_ref
(tools/install_reference.sh)."""
import os
import sys
import types

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..")
sys.path.insert(0, ROOT)
sys.path.append(os.path.join(ROOT, "baseline", "_ref"))
sk = types.ModuleType("skimage")
sk.measure = types.ModuleType("skimage.measure")
sys.modules["skimage"], sys.modules["skimage.measure"] = sk, sk.measure
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/softmpm_numba_cache")

import softmpm  # noqa: E402
import softmpm.cli  # noqa: E402

import paper_2402_01181_b200 as b200  # noqa: E402

counts = sys.argv[1] if len(sys.argv) > 1 else "24000,96000,384000"
threads = str(os.cpu_count() or 1)
print(f"== reference softmpm bench, numba, {threads} threads")
softmpm.cli.main(["bench", "--particles", counts, "--threads", threads, "--frames", "5"])
b200.install(softmpm)
print("== the same harness with install() (B200 hot path)")
softmpm.cli.main(["bench", "--particles", counts, "--threads", threads, "--frames", "5"])
b200.uninstall(softmpm)
