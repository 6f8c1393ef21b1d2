"""Device-memory probe of the GPU compressor at 256^3 (sweep E1/E2 sizing): free memory around the
operator build and around each compress of the first `nd` directions (args fmt:nd ...)."""
import math, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2010_00520_b200 import fmmt
def free(tag):
    torch.cuda.synchronize(); f, t = torch.cuda.mem_get_info(); print(f"{tag}: free {f/1e9:.2f} / {t/1e9:.1f} GB", flush=True)
free("start")
ctx = fmmt.Context(0, torch.cuda.current_stream().cuda_stream); free("ctx")
L = fmmt.multipole_count(2 * math.pi, 0.5, 5); khat, _ = fmmt.direction_grid(L, 2 * L + 1)
ndmax = max(int(a.split(":")[1]) for a in sys.argv[1:])
T = torch.empty((ndmax, 256, 256, 256), dtype=torch.complex128, device="cuda"); free(f"T alloc nd={ndmax}")
ctx.build_operator(128, 128, 128, 0.5, 2 * math.pi, L, khat[:ndmax], T); ctx.sync(); free("built")
for a in sys.argv[1:]:
    fmt, nd = a.split(":"); nd = int(nd)
    try:
        op = ctx.compress(T[:nd], (256, 256, 256), nd, fmt, 1e-6); ctx.sync(); free(f"compressed {fmt} nd={nd}")
        i = op.info(); print(fmt, nd, i["rank_max"], round(100 * (1 - i["compressed_bytes"] / i["original_bytes"]), 3), flush=True)
        op.close(); free("closed")
    except Exception as e:
        print("FAILED", fmt, nd, str(e)[:200], flush=True); free("after failure")
