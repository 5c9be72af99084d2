"""Shared test helpers: golden-case readers and a CPU emulation of the device
pipeline (level-by-level, rank-based classification) driven by the oracle."""

import numpy as np

from oracle import oracle as O


def conceal_case(g, i):
    d, rho, delta, gamma, iters, B = g[f"k{i}_params"].tolist()
    fft = tuple(int(x) for x in g[f"k{i}_fft"])
    return dict(
        name=str(g[f"k{i}_name"]),
        image=g[f"k{i}_image"],
        mask=g[f"k{i}_mask"],
        d=int(d), rho=rho, delta=delta, gamma=gamma, iterations=int(iters), block_size=int(B),
        fft=None if fft == (0, 0) else fft,
        order=str(g[f"k{i}_order"]),
        out_image=g[f"k{i}_out_image"],
        out_mask=g[f"k{i}_out_mask"],
        batches=csr(g[f"k{i}_batch_ptr"], g[f"k{i}_batch_blocks"]),
        unconcealed=g[f"k{i}_unconcealed"].tolist(),
        processed=int(g[f"k{i}_processed"]),
        pick_blocks=g[f"k{i}_pick_blocks"],
        picks=g[f"k{i}_picks"],
    )


def csr(ptr, blocks):
    return [blocks[ptr[k]:ptr[k + 1]].tolist() for k in range(len(ptr) - 1)]


def block_owner(H, W, B):
    rows, cols = -(-H // B), -(-W // B)
    by = np.minimum(np.arange(H) // B, rows - 1)
    bx = np.minimum(np.arange(W) // B, cols - 1)
    return by[:, None] * cols + bx[None, :]


def emulate_block(img, mask, b, ranks, owner, B, p, kernel="c"):
    """Fit block b as the device does (classes from the ORIGINAL mask + ranks)
    with the oracle kernel and write its LOST samples into img (any array with
    numpy-style slicing, e.g. a torch CPU tensor)."""
    H, W = mask.shape
    cols = -(-W // B)
    d = p.d
    r, c = divmod(b, cols)
    r0, r1, c0, c1 = r * B, min(r * B + B, H), c * B, min(c * B + B, W)
    wr0, wr1, wc0, wc1 = max(0, r0 - d), min(H, r1 + d), max(0, c0 - d), min(W, c1 + d)
    sub = mask[wr0:wr1, wc0:wc1]
    own = owner[wr0:wr1, wc0:wc1]
    lost = sub == O.LOST
    cls = np.where(sub == O.RECONSTRUCTED, O.AREA_R, O.AREA_A).astype(np.uint8)
    earlier = ranks[own] < ranks[b]
    cls[lost & (own != b) & earlier] = O.AREA_R
    cls[lost & (own != b) & ~earlier] = O.AREA_BO
    cls[lost & (own == b)] = O.AREA_BI
    vals = np.array(img[wr0:wr1, wc0:wc1], dtype=np.float64)
    blk = O.extrapolate(vals, cls, (r0 - wr0, r1 - wr0, c0 - wc0, c1 - wc0), p, kernel)
    assert blk is not None, f"plan scheduled a degenerate block {b}"
    lostb = mask[r0:r1, c0:c1] == O.LOST
    cur = np.array(img[r0:r1, c0:c1], dtype=np.float64)
    cur[lostb] = blk[lostb]
    if isinstance(img, np.ndarray):
        img[r0:r1, c0:c1] = cur
    else:  # torch CPU tensor (strip-protocol tests)
        import torch

        img[r0:r1, c0:c1] = torch.from_numpy(cur).to(img.dtype)


def emulate_levels(image, mask, B, d, rho, delta, gamma, iterations, fft, ranks, levels, kernel="c",
                   shuffle_seed=0):
    """What the device does, on the CPU: for each level, every block classifies
    its window from the ORIGINAL mask and the plan ranks (lost sample = R iff its
    owner has a smaller rank), fits with the oracle kernel and writes back
    IMMEDIATELY, in a shuffled order (emulating CTAs of one launch racing)."""
    rng = np.random.default_rng(shuffle_seed)
    img = np.array(image, dtype=np.float64, copy=True)
    H, W = img.shape
    owner = block_owner(H, W, B)
    p = O.Params(d=d, rho=rho, delta=delta, gamma=gamma, iterations=iterations, block_size=B,
                 fft_size=fft)
    for level in levels:
        for b in rng.permutation(level).tolist():
            emulate_block(img, mask, b, ranks, owner, B, p, kernel)
    out_mask = mask.copy()
    done = ranks[owner] != np.iinfo(np.int32).max
    out_mask[(mask == O.LOST) & done] = O.RECONSTRUCTED
    return img, out_mask


# ---- large golden fixtures (tests/golden/make_golden_large.py)

def large_case(g):
    """Inputs of a large golden case, regenerated from the seeded generator,
    plus its parameters (FseParams keyword arguments) and fft size."""
    from paper_2207_00233_b200 import synth

    img, mask = synth.config_scene(int(g["config"]), int(g["frame"]))
    r0, r1, c0, c1 = (int(x) for x in g["crop"])
    if r1 > r0:
        img, mask = img[r0:r1, c0:c1].copy(), mask[r0:r1, c0:c1].copy()
    assert [int(img.astype(np.int64).sum()), int(mask.astype(np.int64).sum())] == g["input_sums"].tolist()
    d, rho, delta, gamma, iters, B = g["params"].tolist()
    fft = tuple(int(x) for x in g["fft"])
    kw = dict(d=int(d), rho=rho, delta=delta, gamma=gamma, iterations=int(iters), block_size=int(B))
    return img, mask, kw, (None if fft == (0, 0) else fft)


def window_shapes(H, W, B, d, blocks):
    """(M, N) of each block's window (grid.py:108-135: block +- d, clipped)."""
    cols = -(-W // B)
    r, c = np.asarray(blocks) // cols, np.asarray(blocks) % cols
    r0, c0 = r * B, c * B
    M = np.minimum(H, np.minimum(r0 + B, H) + d) - np.maximum(0, r0 - d)
    N = np.minimum(W, np.minimum(c0 + B, W) + d) - np.maximum(0, c0 - d)
    return M, N


def canonical_fold(picks, F1, F2):
    """Vectorised reference canonical folding (tests/reference.py:59-71):
    picks [n, I, 2] with per-block DFT sizes F1[n], F2[n] (or scalars)."""
    a = picks[..., 0].astype(np.int64)
    b = picks[..., 1].astype(np.int64)
    F1 = np.broadcast_to(np.asarray(F1, dtype=np.int64).reshape(-1, 1), a.shape)
    F2 = np.broadcast_to(np.asarray(F2, dtype=np.int64).reshape(-1, 1), a.shape)
    ta, tb = (F1 - a) % F1, (F2 - b) % F2
    twin = (ta < a) | ((ta == a) & (tb < b))
    return np.stack([np.where(twin, ta, a), np.where(twin, tb, b)], axis=-1)


def pick_hash(canon):
    """64-bit FNV-1a over each row's (a, b) pairs, vectorised over rows
    (the hash make_golden_large.py stores)."""
    canon = np.asarray(canon, dtype=np.int64).reshape(len(canon), -1)
    h = np.full(len(canon), 0xCBF29CE484222325, dtype=np.uint64)
    prime = np.uint64(0x100000001B3)
    for k in range(canon.shape[1]):
        h ^= (canon[:, k] & 0xFFFF).astype(np.uint64)
        h *= prime
    return h.view(np.int64)
