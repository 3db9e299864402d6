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
