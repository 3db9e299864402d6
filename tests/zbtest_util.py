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


def close_report(x, ref, rtol):
    """SURVEY C15 / DESIGN R-tol: normwise ||x - ref||_2 / ||ref||_2 AND the
    elementwise bound |x - ref| <= rtol*|ref| + rtol*rms(ref).  Returns
    (normwise relative error, worst elementwise |x - ref| / bound)."""
    import numpy as np
    x = np.asarray(x, dtype=np.float64).ravel()
    ref = np.asarray(ref, dtype=np.float64).ravel()
    diff = np.abs(x - ref)
    nrm = float(np.linalg.norm(diff) / max(np.linalg.norm(ref), 1e-30))
    rms = float(np.sqrt(np.mean(ref * ref))) if ref.size else 0.0
    bound = rtol * np.abs(ref) + rtol * rms
    bound = np.where(bound > 0, bound, 1e-300)
    worst = float(np.max(diff / bound)) if ref.size else 0.0
    if not np.all(np.isfinite(x)):
        worst = float("inf")
    return nrm, worst


def assert_close(x, ref, rtol, what=""):
    """Normwise <= rtol and elementwise within rtol*|ref| + rtol*rms(ref)."""
    nrm, worst = close_report(x, ref, rtol)
    assert nrm <= rtol, f"{what}: normwise {nrm:.3e} > {rtol:.1e}"
    assert worst <= 1.0, f"{what}: elementwise error {worst:.2f}x the bound rtol*(|ref| + rms(ref)), rtol {rtol:.1e}"
    return nrm
