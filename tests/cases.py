"""Problem builders shared by the parity tests (names match tests/golden/golden.json)."""

from paper_2111_06552_b200 import problems as P


def tri(n):
    return P.stencil_csr((n,), [(0,), (-1,), (1,)], [2.0, -1.0, -1.0])


def problem(name):
    if name == "tri120":
        return tri(120), None
    if name == "lap2d20":
        return P.laplacian_2d(20), None
    if name == "fem6":
        return P.fem_p1_cube(6)
    if name == "tri200_moving":
        return tri(200), None
    if name == "lap3d10_noshift":
        return P.laplacian_3d(10), None
    if name == "lap3d12_baseline":
        return P.laplacian_3d(12), None
    if name == "fem8_baseline":
        return P.fem_p1_cube(8)
    if name == "varcoef10_moving":
        return P.varcoef_diffusion_3d(10, seed=0), None
    if name == "cfg1_baseline":
        return P.laplacian_2d(100), None
    raise KeyError(name)


SOLVER_CASES = ["tri120", "lap2d20", "fem6", "tri200_moving", "lap3d10_noshift",
                "lap3d12_baseline", "fem8_baseline", "varcoef10_moving", "cfg1_baseline"]
