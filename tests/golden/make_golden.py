"""Generate golden vectors by running the REAL reference `rsr` package.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/*.npz.  The GPU box never reads /root/reference; tests
only read these committed fixtures.  Every fixture records the reference call
that produced it.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.environ.get("RSR_REFERENCE_SRC", "/root/reference/pkg/src"))
import rsr  # noqa: E402  (the reference package)

HERE = os.path.dirname(os.path.abspath(__file__))


def pack_index(prefix: str, idx, store: dict) -> None:
    """Flatten one reference RsrIndex (indexer.py:47-139) into npz arrays."""
    store[prefix + "perms"] = np.stack([blk.permutation for blk in idx.blocks]).astype(np.uint32)
    store[prefix + "segs"] = np.asarray(idx._segs, np.int64)        # flat, each block 2^w + 1
    store[prefix + "seg_starts"] = np.asarray(idx._seg_starts, np.int64)
    store[prefix + "widths"] = np.asarray(idx._widths, np.int64)
    store[prefix + "buckets"] = np.asarray(idx._buckets).astype(np.uint32)


def worked_example() -> dict:
    """conftest.py:10-26 / test_acceptance.py:88-101 known answers."""
    B6 = np.array([[0, 1, 1, 1, 0, 1], [0, 0, 0, 1, 1, 1], [0, 1, 1, 1, 1, 0],
                   [1, 1, 0, 0, 1, 0], [0, 0, 1, 1, 0, 1], [0, 0, 0, 0, 1, 0]], np.uint8)
    V6 = np.array([3.0, 2.0, 4.0, 5.0, 9.0, 1.0])
    B = rsr.BinaryMatrix.from_dense(B6)
    idx = rsr.preprocess(B, 2)
    tidx = rsr.preprocess_ternary(rsr.TernaryMatrix(B6.astype(np.int8)), 2)
    u = rsr.segmented_sum(V6, idx.blocks[0])
    out = {"B6": B6, "V6": V6,
           "block0_perm": idx.blocks[0].permutation, "block0_seg": idx.blocks[0].segmentation,
           "block0_sums": u.sums, "block0_rsr": rsr.block_product_rsr(u),
           "block0_rsrpp": rsr.block_product_rsrpp(u),
           "product_binary": rsr.multiply_rsr(V6, idx), "product_ternary": rsr.multiply_ternary(V6, tidx),
           "naive": rsr.naive_multiply(V6, B)}
    pack_index("bidx_", idx, out)
    pack_index("tpos_", tidx.positive, out)
    pack_index("tneg_", tidx.negative, out)
    return out


def fuzz_cases(seed: int, count: int, max_dim: int, ks_cap: int) -> dict:
    """Seeded small ternary cases across k (criterion-1 style, test_acceptance.py:41-64):
    matrix, integer and float vectors, full reference index, rsr/rsrpp products."""
    rng = np.random.default_rng(seed)
    out = {"count": np.int64(count)}
    for i in range(count):
        rows = int(rng.integers(1, max_dim + 1))
        cols = int(rng.integers(1, max_dim + 1))
        A = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
        vi = rng.integers(-100, 101, size=rows).astype(np.float64)
        vf = rng.standard_normal(rows)
        kmax = min(ks_cap, rsr.max_k_for_rows(rows))
        k = int(rng.integers(1, kmax + 1))
        T = rsr.TernaryMatrix(A)
        tidx = rsr.preprocess_ternary(T, k)
        p = f"c{i}_"
        out[p + "A"] = A
        out[p + "k"] = np.int64(k)
        out[p + "vi"] = vi
        out[p + "vf"] = vf
        pack_index(p + "pos_", tidx.positive, out)
        pack_index(p + "neg_", tidx.negative, out)
        for variant in ("rsr", "rsrpp"):
            out[p + f"int_{variant}"] = rsr.multiply_ternary(vi, tidx, variant)
            out[p + f"flt_{variant}"] = rsr.multiply_ternary(vf, tidx, variant)
        out[p + "int_naive"] = rsr.naive_multiply(vi, T)
        out[p + "flt_naive"] = rsr.naive_multiply(vf, T)
        # binary multiply of the positive half (multiply_rsr, kernels.py:185-193)
        out[p + "int_pos_rsrpp"] = rsr.multiply_rsr(vi, tidx.positive, "rsrpp")
    return out


def medium_cases() -> dict:
    """The criterion-1 'big' shapes (test_acceptance.py:46-48) at tuned k, integer v:
    products only plus the seeded generator, so tests can regenerate the inputs."""
    out = {}
    for i, (rows, cols) in enumerate(((256, 256), (1024, 1024), (256, 1024), (1024, 256))):
        rng = np.random.default_rng([2411, rows, cols])
        A = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
        v = rng.integers(-100, 101, size=rows).astype(np.float64)
        k = rsr.optimal_k_rsrpp(rows)
        tidx = rsr.preprocess_ternary(rsr.TernaryMatrix(A), k)
        p = f"m{i}_"
        out[p + "shape"] = np.array([rows, cols], np.int64)
        out[p + "k"] = np.int64(k)
        out[p + "rsrpp"] = rsr.multiply_ternary(v, tidx, "rsrpp")
        out[p + "rsr"] = rsr.multiply_ternary(v, tidx, "rsr")
        out[p + "naive"] = rsr.naive_multiply(v, rsr.TernaryMatrix(A))
        out[p + "pos_perm_crc"] = np.array([int(np.bitwise_xor.reduce(
            blk.permutation.astype(np.uint64) * np.arange(1, rows + 1, dtype=np.uint64)))
            for blk in tidx.positive.blocks], np.uint64)
        out[p + "neg_seg_sum"] = np.array([int(blk.segmentation.astype(np.int64).sum())
                                           for blk in tidx.negative.blocks], np.int64)
    return out


def folds() -> dict:
    """Block products (kernels.py:104-116) on integer and float u, widths 1..10."""
    rng = np.random.default_rng(104)
    out = {}
    for w in range(1, 11):
        ui = rng.integers(-100, 101, size=1 << w).astype(np.float64)
        uf = rng.standard_normal(1 << w)
        for tag, u in (("i", ui), ("f", uf)):
            s = rsr.SegmentedSums(w, u)
            out[f"w{w}{tag}_u"] = u
            out[f"w{w}{tag}_rsr"] = rsr.block_product_rsr(s)
            out[f"w{w}{tag}_rsrpp"] = rsr.block_product_rsrpp(s)
    return out


def tuner() -> dict:
    ns = np.array(sorted(set([1, 2, 3, 6, 100, 4095, 4096, 14336, 16384, 65536]
                             + [1 << e for e in range(0, 17)]
                             + list(np.random.default_rng(8).integers(1, 1 << 17, 200)))), np.int64)
    return {"n": ns,
            "k_rsrpp": np.array([rsr.optimal_k_rsrpp(int(n)) for n in ns], np.int64),
            "k_rsr": np.array([rsr.optimal_k_rsr(int(n)) for n in ns], np.int64),
            "max_k": np.array([rsr.max_k_for_rows(int(n)) for n in ns], np.int64)}


def rsx_files() -> dict:
    """.rsx files written by the reference's save_index (store.py:31-45) and the reference's
    load_index verdict on corrupted copies (store.py:48-101): valid files carry the product
    of a fixed vector, corrupt ones the exact FormatError message."""
    import json
    import struct
    from rsr import store
    out = {}
    rsx_dir = os.path.join(HERE, "rsx")
    os.makedirs(rsx_dir, exist_ok=True)
    rng = np.random.default_rng(2024)
    A = rng.integers(-1, 2, size=(200, 77), dtype=np.int8)
    tidx = rsr.preprocess_ternary(rsr.TernaryMatrix(A), 5)
    B = (rng.integers(0, 2, size=(90, 33))).astype(np.uint8)
    bidx = rsr.preprocess(rsr.BinaryMatrix.from_dense(B), 4)
    vt = rng.integers(-50, 51, size=200).astype(np.float64)
    vb = rng.integers(-50, 51, size=90).astype(np.float64)
    store.save_index(tidx, os.path.join(rsx_dir, "ternary_200x77_k5.rsx"))
    store.save_index(bidx, os.path.join(rsx_dir, "binary_90x33_k4.rsx"))
    out["ternary_v"] = vt
    out["ternary_y"] = rsr.multiply_ternary(vt, tidx)
    out["binary_v"] = vb
    out["binary_y"] = rsr.multiply_rsr(vb, bidx)
    good = open(os.path.join(rsx_dir, "binary_90x33_k4.rsx"), "rb").read()
    hdr = store.HEADER_BYTES
    _HEADER_T = struct.Struct("<4sHBQQHI")
    first_perm = hdr + 2                       # block 0: u16 width, then perm u32 [rows]
    first_seg = first_perm + 4 * 90
    def put_u32(raw, off, val):
        raw = bytearray(raw)
        struct.pack_into("<I", raw, off, val)
        return bytes(raw)
    corrupt = {
        "bad_magic": b"RSX9" + good[4:],
        "bad_version": good[:4] + struct.pack("<H", 7) + good[6:],
        "bad_kind": good[:6] + bytes([5]) + good[7:],
        "truncated_header": good[:20],
        "truncated_payload": good[:-5],
        "trailing_bytes": good + b"\x00",
        "bad_block_count": good[:25] + struct.pack("<I", 3) + good[29:],
        "bad_width": good[:hdr] + struct.pack("<H", 3) + good[hdr + 2:],
        "perm_duplicate": put_u32(good, first_perm + 4, struct.unpack_from("<I", good, first_perm)[0]),
        "perm_range": put_u32(good, first_perm, 90),
        "seg_start": put_u32(good, first_seg, 1),
        "seg_order": put_u32(good, first_seg + 4 * 3, 0),
    }
    # ternary files: which half / block / check the reference names first (store.py:80-101
    # validates each half completely before reading the next; k is checked by from_blocks)
    tgood = open(os.path.join(rsx_dir, "ternary_200x77_k5.rsx"), "rb").read()
    nb5 = -(-77 // 5)
    half_bytes = sum(2 + 4 * 200 + 4 * (1 << min(5, 77 - 5 * b)) for b in range(nb5))
    def tblock(h, b):  # byte offset of block b of half h (its u16 width)
        return hdr + h * half_bytes + sum(2 + 4 * 200 + 4 * (1 << min(5, 77 - 5 * c)) for c in range(b))
    def dup_perm(raw, h, b):  # perm[1] := perm[0] in block b of half h
        off = tblock(h, b) + 2
        return put_u32(raw, off + 4, struct.unpack_from("<I", raw, off)[0])
    corrupt.update({
        "t_pos5_neg2": dup_perm(dup_perm(tgood, 0, 5), 1, 2),     # both halves bad: positive block 5 first
        "t_neg3": dup_perm(tgood, 1, 3),                             # only the negative half
        "t_pos1_truncneg": dup_perm(tgood, 0, 1)[:tblock(1, 4)],     # positive invariant vs negative truncation
        "t_pos4_trailing": dup_perm(tgood, 0, 4) + b"\x00",         # positive invariant vs trailing bytes
        "t_k_exceeds": tgood[:23] + struct.pack("<H", 9) + tgood[25:],  # k = 9: block count no longer matches
        "t_k_zero": tgood[:23] + struct.pack("<H", 0) + tgood[25:],
        # a well-formed binary file whose k exceeds floor(log2 rows) (from_blocks' _check_k)
        "k_exceeds_rows": (_HEADER_T.pack(b"RSX1", 1, 1, 200, 8, 8, 1) + struct.pack("<H", 8)
                           + np.arange(200, dtype="<u4").tobytes() + np.zeros(256, "<u4").tobytes()),
    })
    verdicts = {}
    for name, raw in corrupt.items():
        path = os.path.join(rsx_dir, f"corrupt_{name}.rsx")
        open(path, "wb").write(raw)
        try:
            store.load_index(path)
            verdicts[name] = None
        except rsr.FormatError as exc:
            verdicts[name] = str(exc)
        except ValueError as exc:  # not a FormatError (e.g. column_blocks on k = 0)
            verdicts[name] = "ValueError: " + str(exc)
    json.dump(verdicts, open(os.path.join(rsx_dir, "verdicts.json"), "w"), indent=1, sort_keys=True)
    return out


def counted() -> dict:
    """The reference's instrumented twins (kernels.py:240-320): products and accumulate counts."""
    from rsr import kernels as K
    out = {}
    rng = np.random.default_rng(31)
    for i, (rows, cols, k) in enumerate(((50, 23, 3), (300, 70, 6), (128, 9, 7))):
        B = rng.integers(0, 2, size=(rows, cols)).astype(np.uint8)
        idx = rsr.preprocess(rsr.BinaryMatrix.from_dense(B), k)
        v = rng.standard_normal(rows)
        out[f"c{i}_B"] = B
        out[f"c{i}_k"] = np.int64(k)
        out[f"c{i}_v"] = v
        for variant in ("rsr", "rsrpp"):
            y, total = K.multiply_counted(v, idx, variant)
            out[f"c{i}_{variant}_y"] = y
            out[f"c{i}_{variant}_total"] = np.int64(total)
        sums, adds = K.segmented_sum_counted(v, idx.blocks[0])
        out[f"c{i}_seg0_sums"] = sums.sums
        out[f"c{i}_seg0_adds"] = np.int64(adds)
        for name, fn in (("rsr", K.block_product_rsr_counted), ("rsrpp", K.block_product_rsrpp_counted)):
            prod, adds = fn(sums)
            out[f"c{i}_bp0_{name}"] = prod
            out[f"c{i}_bp0_{name}_adds"] = np.int64(adds)
    return out


def overflow() -> dict:
    """Wide-value fixtures (tests/golden/overflow_inputs.py): integer activations whose column
    sums exceed int32 (|v| = 2^20 at 16384 rows; int64 |v| up to 2^36 and 2^50),
    float64 holding integers, high-dynamic-range floats, and 70000 rows.  The reference's
    multiply_ternary / multiply_rsr (both variants) and multiply_parallel(W=3) on each; the
    inputs are regenerated from their seeds by the tests (digests recorded here)."""
    sys.path.insert(0, HERE)
    from overflow_inputs import CASES, digest, make_inputs
    out = {}
    for name, (domain, rows, cols, k, kind, bound) in CASES.items():
        A, v = make_inputs(name)
        out[name + "_A_digest"] = np.array(digest(A))
        out[name + "_v_digest"] = np.array(digest(v))
        if domain == "ternary":
            idx = rsr.preprocess_ternary(rsr.TernaryMatrix(A), k)
            mult = rsr.multiply_ternary
        else:
            idx = rsr.preprocess(rsr.BinaryMatrix.from_dense(A.astype(np.uint8)), k)
            mult = rsr.multiply_rsr
        for variant in ("rsrpp", "rsr"):
            out[f"{name}_{variant}"] = mult(v, idx, variant)
        out[name + "_par3"] = rsr.multiply_parallel(v, idx, "rsrpp", 3)
    return out


def main() -> None:
    np.savez_compressed(os.path.join(HERE, "worked_example.npz"), **worked_example())
    np.savez_compressed(os.path.join(HERE, "fuzz_small.npz"), **fuzz_cases(101, 60, 64, 8))
    np.savez_compressed(os.path.join(HERE, "medium.npz"), **medium_cases())
    np.savez_compressed(os.path.join(HERE, "folds.npz"), **folds())
    np.savez_compressed(os.path.join(HERE, "tuner.npz"), **tuner())
    np.savez_compressed(os.path.join(HERE, "rsx_products.npz"), **rsx_files())
    np.savez_compressed(os.path.join(HERE, "counted.npz"), **counted())
    np.savez_compressed(os.path.join(HERE, "overflow.npz"), **overflow())
    print("reference rsr", rsr.__version__, "golden vectors written to", HERE)


if __name__ == "__main__":
    main()
