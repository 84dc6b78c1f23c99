"""Shared-memory bank conflicts of one tile's node-value gathers and per-node
reads, counted on the host from the tile's tables (experiment build
lib/libfemmin_ws.so: fm_debug_tile).

    python tools/bank_probe.py [--config cfg4] [--tile N] [--save out.npz]

For every chunk and element slot l: the wavefronts of the LDS.64 that reads
nv[loc_l] over each half-warp (16 rows), = the largest number of rows that hit
the same bank pair (index mod 16)."""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["FM_LIB_OVERRIDE"] = os.path.join(ROOT, "paper_2109_01158_b200", "lib",
                                             "libfemmin_ws.so")
import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--tile", type=int, default=-1)
    ap.add_argument("--save", default="")
    args = ap.parse_args()
    from paper_2109_01158_b200 import _lib, problems
    pr = problems.CONFIGS[args.config]()
    lib = _lib.load()
    st = pr.dm.stats
    t = args.tile if args.tile >= 0 else st["n_tiles"] // 2
    meta = (C.c_int * 16)()
    ctxp = pr.dm._h
    lib.fm_debug_tile.restype = C.c_int
    lib.fm_debug_tile.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.c_void_p]
    assert lib.fm_debug_tile(ctxp, t, meta, None, None, None) == 0
    m = np.array(meta[:])
    own_count, node_count, clo_count, blk_stride = int(m[1]), int(m[5]), int(m[10]), int(m[11])
    loc = np.zeros((own_count, 4), dtype=np.uint16)
    clo = np.zeros(clo_count, dtype=np.int32)
    nch = (own_count + 255) // 256
    blocks = np.zeros(nch * blk_stride, dtype=np.uint16)
    assert lib.fm_debug_tile(ctxp, t, meta, loc.ctypes.data, clo.ctypes.data,
                             blocks.ctypes.data) == 0
    print(f"tile {t}: own {own_count} nodes {node_count} closure {clo_count} chunks {nch}")
    print("closure node ids (first 24):", clo[:24])
    print("loc of rows 0..19 of chunk 0:\n", loc[:20])
    if args.save:
        np.savez(args.save, meta=m, loc=loc, closure=clo, blocks=blocks)
    nv = 4 if pr.dm.dim == 3 else 3
    tot = ideal = 0
    for c in range(nch):
        rows = loc[c * 256:(c + 1) * 256]
        for h in range(0, len(rows), 16):
            hw = rows[h:h + 16]
            for l in range(nv):
                banks = hw[:, l].astype(int) % 16
                tot += np.bincount(banks, minlength=16).max()
                ideal += 1
    print(f"node-value gathers: {tot} wavefronts for {ideal} half-warp loads = {tot / ideal:.2f} x ideal")


if __name__ == "__main__":
    main()
