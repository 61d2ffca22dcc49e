"""Model descriptors: the device-side counterpart of the reference's model
library (/root/reference/proj/include/ivreach/models.hpp, src/models.cpp).

The reference builds ``SystemModel`` objects out of ``std::function``
evaluators (system_model.hpp:14-43); those cannot run on a GPU, so here a
``SystemModel`` is a descriptor naming which device vector field to use and
its resolved parameters.  Constructors keep the reference's names, defaults
and argument validation (messages of models.cpp ``require``).
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace
from typing import Tuple

# pirk_model_kind (include/pirk_c.h)
ZERO, SCALAR_DECAY, SCALAR_LINEAR, TRAFFIC, HEAT3D, CHAIN, LAUB_LOOMIS, ARCH_QUAD, VDP, USER = range(10)
# pirk_decomp
DECOMP_NONE, DECOMP_NATIVE, DECOMP_JACOBIAN = range(3)

_HAS_GROWTH = {ZERO, SCALAR_DECAY, SCALAR_LINEAR, TRAFFIC, HEAT3D, LAUB_LOOMIS, ARCH_QUAD, VDP}


@dataclass(frozen=True)
class SystemModel:
    """system_model.hpp:28-43.  ``decomposition``/``growth_rhs`` presence is
    expressed by ``decomp`` and the model kind."""

    kind: int
    dim: int
    input_dim: int
    params: Tuple[float, ...] = field(default_factory=tuple)
    decomp: int = DECOMP_NATIVE
    grid: int = 0
    name: str = ""
    input_affine: bool = True
    sparsity_note: str = ""
    program: object = None  # USER: the compiled evaluators (Program)

    def has_growth(self) -> bool:
        if self.kind == USER:
            return bool(self.program.flags & HAS_GROWTH)
        return self.kind in _HAS_GROWTH

    def has_decomposition(self) -> bool:
        if self.kind == USER:
            return bool(self.program.flags & HAS_DECOMPOSITION)
        return self.decomp != DECOMP_NONE


# pirk_program flags (include/pirk_c.h)
HAS_RHS, HAS_DECOMPOSITION, HAS_GROWTH, INPUT_AFFINE = 1, 2, 4, 8


class Program:
    """A user model's evaluators: CUDA source defining ``pirk_rhs`` /
    ``pirk_decomposition`` / ``pirk_growth`` (the reference's RhsFn / DecompFn /
    growth RhsFn, system_model.hpp:14-43, as device functions with the same
    arguments -- see include/pirk_c.h).  Compiled by NVRTC for sm_100a on first
    use (exact mode: --fmad=false).  ``compile(mode)`` compiles eagerly and
    raises ValueError with the NVRTC log on a bad source (no GPU needed)."""

    def __init__(self, source: str, dim: int, input_dim: int, flags: int, stencil_radius: int = 0):
        import ctypes as C

        from . import _lib

        h = C.c_void_p()
        st = _lib.lib().pirk_program_create(source.encode(), int(dim), int(input_dim), int(flags),
                                            C.byref(h))
        if st != _lib.OK:
            raise ValueError("pirk_program_create: invalid source or dimension")
        self._h = h
        if stencil_radius:
            if _lib.lib().pirk_program_set_stencil(h, int(stencil_radius)) != _lib.OK:
                raise ValueError("user model: stencil radius must lie in [1, 64]")
        self.stencil_radius = int(stencil_radius)
        self.source = source
        self.dim = int(dim)
        self.input_dim = int(input_dim)
        self.flags = int(flags)

    @property
    def handle(self):
        return self._h

    def compile(self, mode: str = "exact") -> int:
        """Compile now; returns the sm_100a image size in bytes."""
        import ctypes as C

        from . import _lib

        log = C.create_string_buffer(1 << 16)
        size = C.c_uint64()
        st = _lib.lib().pirk_program_compile(self._h, {"exact": 0, "fast": 1}[mode], log, len(log),
                                             C.byref(size))
        if st != _lib.OK:
            raise ValueError(log.value.decode(errors="replace"))
        return int(size.value)

    def cubin(self, mode: str = "exact") -> bytes:
        import ctypes as C

        from . import _lib

        n = self.compile(mode)
        buf = C.create_string_buffer(n)
        _lib.lib().pirk_program_cubin(self._h, {"exact": 0, "fast": 1}[mode], buf, n)
        return buf.raw

    def __del__(self):
        try:
            from . import _lib

            if getattr(self, "_h", None):
                _lib.lib().pirk_program_destroy(self._h)
                self._h = None
        except Exception:
            pass


def make_user_model(source: str, dim: int, input_dim: int = 0, *, rhs: bool = True,
                    decomposition: bool = False, growth: bool = False,
                    input_affine: bool = False, name: str = "user",
                    sparsity_note: str = "", stencil_radius: int = 0) -> SystemModel:
    """A SystemModel with caller-written evaluators (system_model.hpp:28-43:
    ``rhs`` always, ``decomposition`` / ``growth_rhs`` optional, the
    ``input_affine`` flag growth-bound requires).  ``source`` is CUDA C++; see
    :class:`Program`.  ``stencil_radius`` r > 0 declares a 1-D stencil (the
    evaluators read components i-r .. i+r only): MM / GB then run one fused
    RK4 step per launch (pirk_program_set_stencil)."""
    _require(dim >= 1, "user model needs at least 1 state")
    flags = ((HAS_RHS if rhs else 0) | (HAS_DECOMPOSITION if decomposition else 0)
             | (HAS_GROWTH if growth else 0) | (INPUT_AFFINE if input_affine else 0))
    prog = Program(source, dim, input_dim, flags, stencil_radius)
    return SystemModel(USER, int(dim), int(input_dim), (), DECOMP_NATIVE if decomposition else DECOMP_NONE,
                       name=name, input_affine=input_affine, sparsity_note=sparsity_note, program=prog)


def _require(ok: bool, msg: str) -> None:
    if not ok:
        raise ValueError(msg)


def _p(*vals) -> Tuple[float, ...]:
    return tuple(float(v) for v in vals)


def make_traffic(segments: int, v: float = 0.5, w: float = 1.0 / 6.0, c: float = 40.0,
                 xbar: float = 320.0, period: float = 30.0, beta: float = 0.75) -> SystemModel:
    """models.cpp:47-90 (cooperative: decomposition = cooperative(f))."""
    _require(segments >= 3, "traffic model needs at least 3 segments")
    _require(v > 0 and w > 0 and c > 0 and xbar > 0 and period > 0,
             "traffic parameters must be positive")
    _require(0 < beta <= 1, "traffic beta must lie in (0, 1]")
    return SystemModel(TRAFFIC, int(segments), 1, _p(v, w, c, xbar, period, beta),
                       DECOMP_NATIVE, name="traffic", sparsity_note="tridiagonal")


def make_heat3d(grid: int, alpha: float = 1.0, exchange: float = 1.0) -> SystemModel:
    """models.cpp:92-133 (linear, cooperative; growth_rhs == rhs)."""
    _require(grid >= 2, "heat3d model needs at least 2 grid points per axis")
    _require(alpha > 0, "heat3d alpha must be positive")
    _require(exchange >= 0, "heat3d exchange coefficient must be nonnegative")
    g = int(grid)
    return SystemModel(HEAT3D, g * g * g, 0, _p(alpha, exchange), DECOMP_NATIVE, grid=g,
                       name="heat3d", sparsity_note="7-point stencil")


def make_chain(n: int, a: float = 1.0, b: float = 0.5, c: float = 0.25) -> SystemModel:
    """Synthetic coupled (non-cooperative) chain of SURVEY.md 8(d), config 4:
    f_i = -a x_i + b s(x_{i-1}) - c s(x_{i+1}) + p, s(z) = z/(1+|z|),
    with the decomposition reading x_{i+1} from the opposite corner."""
    _require(n >= 1, "chain model needs at least 1 state")
    return SystemModel(CHAIN, int(n), 1, _p(a, b, c), DECOMP_NATIVE, name="chain",
                       input_affine=True, sparsity_note="tridiagonal, non-cooperative")


def make_laub_loomis() -> SystemModel:
    """models.cpp:463-502 (no decomposition in the catalog)."""
    return SystemModel(LAUB_LOOMIS, 7, 0, (), DECOMP_NONE, name="laub-loomis")


def make_arch_quadrotor(mass: float = 1.4, gravity: float = 9.81, jx: float = 0.054,
                        jy: float = 0.054, jz: float = 0.104) -> SystemModel:
    """models.cpp:504-613 (no decomposition in the catalog)."""
    _require(mass > 0 and gravity > 0 and jx > 0 and jy > 0 and jz > 0,
             "quadrotor physical parameters must be positive")
    return SystemModel(ARCH_QUAD, 12, 0, _p(mass, gravity, jx, jy, jz), DECOMP_NONE,
                       name="arch-quadrotor")


def make_vdp(mu: float = 1.0, op_x: float = 2.5, op_y: float = 3.0) -> SystemModel:
    """models.cpp:444-461."""
    _require(mu > 0, "van der Pol mu must be positive")
    _require(op_x > 0 and op_y > 0, "van der Pol operating box must be positive")
    return SystemModel(VDP, 2, 0, _p(mu, op_x, op_y), DECOMP_NONE, name="vdp")


def make_zero(dim: int = 2) -> SystemModel:
    """models.cpp:615-627."""
    _require(dim >= 1, "zero model needs at least 1 state")
    return SystemModel(ZERO, int(dim), 0, (), DECOMP_NATIVE, name="zero")


def make_scalar_decay() -> SystemModel:
    """models.cpp:629-641: xdot = -x + p."""
    return SystemModel(SCALAR_DECAY, 1, 1, (), DECOMP_NATIVE, name="scalar-decay")


def make_scalar_linear(a: float = 1.0) -> SystemModel:
    """models.cpp:643-655: xdot = a x."""
    return SystemModel(SCALAR_LINEAR, 1, 0, _p(a), DECOMP_NATIVE, name="scalar-linear")


def with_jacobian_decomposition(model: SystemModel) -> SystemModel:
    """Attach d_i = f_i(x) + sum_{j != i, C_ij != 0} C_ij (x_j - xh_j), where C
    is the model's growth matrix (a valid decomposition wherever C bounds
    |df_i/dx_j| -- the models' documented operating boxes).  This is the
    user-supplied decomposition the reference accepts through its public API
    (test_reach.cpp:195-205); SURVEY.md 8(d) uses it for config 1."""
    _require(model.kind in (LAUB_LOOMIS, ARCH_QUAD, VDP),
             "jacobian decomposition needs a dense growth matrix model")
    return replace(model, decomp=DECOMP_JACOBIAN)


# Catalog defaults for the configurations the hot path is benchmarked on
# (models.cpp:688-1000 default problems).
CATALOG = {
    "traffic": make_traffic,
    "heat3d": make_heat3d,
    "chain": make_chain,
    "laub-loomis": make_laub_loomis,
    "arch-quadrotor": make_arch_quadrotor,
    "vdp": make_vdp,
    "zero": make_zero,
    "scalar-decay": make_scalar_decay,
    "scalar-linear": make_scalar_linear,
}
