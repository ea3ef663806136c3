"""Build a probe variant of libflashhe.so with extra -D flags (development only).

    python tools/build_probe.py TAG -DTC_PROBE_NOFILL ...   ->  tools/_lib_TAG.so
Load it with FLASHHE_LIB=tools/_lib_TAG.so (results of probe builds may be wrong
by construction; they only time pipeline pieces).
"""

import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2401_16732_b200 import build  # noqa: E402

tag, flags = sys.argv[1], sys.argv[2:]
out = ROOT / "tools" / f"_lib_{tag}.so"
cmd = [build.NVCC, *build.ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
       "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr", "-I", str(ROOT / "include"), *flags,
       "-o", str(out), *map(str, build.sources())]
subprocess.run(cmd, check=True)
print(out)
