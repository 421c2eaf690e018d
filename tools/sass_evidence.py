"""Per-kernel counts of the SASS mnemonics that show how the step kernels
move data and what their arithmetic costs (cuobjdump -sass of libsw2d.so):
TMA bulk copies (UBLKCP), mbarrier ops (SYNCS.*), shared loads, 128-bit
global loads/stores, shuffles, packed FP32 (FADD2/FMUL2), fused multiply-adds
(must be 0 in the step kernels), selects/compares (FSEL/FSETP) and register
moves (IMAD.MOV, MOV).  Static counts over the whole kernel."""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1711_04471_b200/libsw2d.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
keys = ["UBLKCP", "SYNCS.ARRIVE.TRANS64", "SYNCS.PHASECHK", "LDS.128", "STG.E.128",
        "LDG.E.128", "SHFL", "FADD2", "FMUL2", "FFMA2", "FFMA", "FSEL", "FSETP", "IMAD.MOV", "MOV",
        "HMMA", "UTCHMMA"]
print(f"# cuobjdump -sass {lib.split('/')[-1]} (sm_100a); static instruction counts per kernel")
for f in re.split(r"\n\s+Function : ", sass)[1:]:
    name = f.split("\n", 1)[0].strip()
    dem = subprocess.run(["cu++filt", name], capture_output=True, text=True).stdout.strip()
    short = re.sub(r"^(void )?sw2d_dev::(\(anonymous namespace\)|<unnamed>)::", "", dem)
    short = re.sub(r"\((sw2d_dev::)?\w+\)$", "", short).replace("(int)", "").replace("(bool)", "")
    ops = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", f)
    c = collections.Counter()
    for o in ops:
        for k in keys:
            # exact mnemonic or one of its modifiers (FADD2 is not FADD, MOV not IMAD.MOV)
            if o == k or o.startswith(k + "."):
                c[k] += 1
    print(f"{short:36s} total {len(ops):5d}  " + "  ".join(f"{k}:{c[k]}" for k in keys if c[k]))
