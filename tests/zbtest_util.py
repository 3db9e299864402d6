import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def read_csv(name):
    rows = []
    header = None
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            if header is None:
                header = line.split(",")
                continue
            rows.append(dict(zip(header, line.split(","))))
    return rows


def ms_to_us(x: str) -> int:
    """Table 8 ms values with 3 decimals -> exact integer microseconds."""
    whole, _, frac = x.partition(".")
    frac = (frac + "000")[:3]
    return int(whole) * 1000 + int(frac)


def cuda_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def bf16_kappa(n):
    """Elementwise counterpart of the normwise rtol (DESIGN R-tol): if the N element
    errors were Gaussian at exactly the normwise tolerance (std = rtol * scale), their
    largest would be ~sqrt(2 ln N) * rtol * scale; at least 3."""
    import math
    return max(3.0, math.sqrt(2.0 * math.log(max(n, 2))))


def close_report(x, ref, rtol, bf16=False, exact_zero_rows=False):
    """SURVEY C15 / DESIGN R-tol: normwise ||x - ref||_2 / ||ref||_2 AND an elementwise
    bound |x - ref| <= rtol*|ref| + kappa*rtol*floor.
      f32 mode:  kappa = 1, floor = rms(ref)                        (SURVEY C15 as written)
      bf16 mode: kappa = bf16_kappa(N) = max(3, sqrt(2 ln N)), floor = max(rms of the
                 element's row, rms over the tensor's
                 non-zero rows)                                      (DESIGN R-tol derivation);
                 exact_zero_rows: a row the reference leaves exactly zero (an embedding
                 row no token touched) must be exactly zero
    Returns (normwise relative error, worst elementwise |x - ref| / bound)."""
    import numpy as np
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    if x.shape != ref.shape:
        x = x.reshape(ref.shape)
    diff = np.abs(x - ref)
    nrm = float(np.linalg.norm(diff) / max(np.linalg.norm(ref), 1e-30))
    if not ref.size:
        return nrm, 0.0
    if bf16:
        r2 = ref.reshape(ref.shape[0], -1) if ref.ndim >= 2 else ref.reshape(1, -1)
        row = np.sqrt(np.mean(r2 * r2, axis=1, keepdims=True))
        nz = row[:, 0] > 0
        rms_nz = float(np.sqrt(np.mean(r2[nz] * r2[nz]))) if nz.any() else 0.0
        floor = np.maximum(row, rms_nz)
        if exact_zero_rows:       # rows the reference leaves exactly zero (untouched embedding rows)
            floor = np.where(row > 0, floor, 0.0)
        floor = floor * np.ones_like(r2)
        bound = rtol * np.abs(r2) + bf16_kappa(ref.size) * rtol * floor
        d2 = diff.reshape(r2.shape)
    else:
        rms = float(np.sqrt(np.mean(ref * ref)))
        bound = rtol * np.abs(ref) + rtol * rms
        d2 = diff
    worst = float(np.max(np.where(bound > 0, d2 / np.where(bound > 0, bound, 1.0), np.where(d2 > 0, np.inf, 0.0))))
    if not np.all(np.isfinite(x)):
        worst = float("inf")
    return nrm, worst


def assert_close(x, ref, rtol, what="", bf16=False, exact_zero_rows=False):
    """Normwise <= rtol and elementwise within the C15 bound (close_report)."""
    nrm, worst = close_report(x, ref, rtol, bf16, exact_zero_rows)
    assert nrm <= rtol, f"{what}: normwise {nrm:.3e} > {rtol:.1e}"
    assert worst <= 1.0, f"{what}: elementwise error {worst:.2f}x the C15 bound (rtol {rtol:.1e}, bf16={bf16})"
    return nrm
