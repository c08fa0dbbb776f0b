"""Build K1 experiment variants into tools/exp/ (lib_<name>.so) from -D flag sets."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_03645_b200 import build as B  # noqa: E402

EXP = os.path.join(os.path.dirname(os.path.abspath(__file__)), "exp")
for spec in sys.argv[1:]:
    name, _, flags = spec.partition("=")
    extra = [f"-D{f}" for f in flags.split(",") if f]
    B.build(lib=os.path.join(EXP, f"lib_{name}.so"), build_dir=os.path.join(EXP, f"_b_{name}"), extra=extra,
            ptxas_info=False)
    print("built", name, extra, flush=True)
