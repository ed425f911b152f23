"""Plug the B200 kernel into the reference package as a kernel variant.

The reference has no FFI; its plugin point is the kernel dispatch
`tersoffmd.kernels.compute(state, nl, params, variant, threads=1)`
(pkg/src/tersoffmd/kernels.py:517-527), which its callers bind by name:
ForceField.__call__ (system.py:340) and through it velocity_verlet_step /
run_nve / run_stretch, the verify suites (verify.py:97-200), the benchmark
harness (bench.py:124-129) and the CLI.  install() adds a "B200" tag:

  * "B200" joins tersoffmd.kernels.KERNEL_TAGS (KernelVariant validation,
    kernels.py:46-59) and the CLI's variant names (cli.py:92-97, `--variant b200`);
  * compute() is wrapped in every tersoffmd module that imported it: a
    variant whose tag is "B200" runs on this package's sm_100a kernel, every
    other tag on the reference's own code;
  * the reference's NeighborList is used as built (imported to the device
    once per list object, tb_nlist_import); the result is the reference's
    ForceEnergyResult with the same stats keys.

    import tersoffmd
    from paper_1710_00882_b200 import integration
    integration.install(tersoffmd)
    v = tersoffmd.kernels.make_variant("B200")                 # fp64
    v = tersoffmd.kernels.make_variant("B200", precision="single")  # mixed
    tersoffmd.system.run_nve(state, params, tersoffmd.system.RunConfig(variant=v))

This is the binding a reference maintainer would add; the
parity test tests/test_gpu_reference_dropin.py runs the reference's own
callers through it.
"""

import importlib

from . import kernels as _k

TAG = "B200"
_MODULES = ("kernels", "system", "verify", "bench", "cli")


def _b200_compute(ref_kernels, orig):
    def compute(state, nl, params, variant, threads=1):
        if getattr(variant, "tag", None) != TAG:
            return orig(state, nl, params, variant, threads)
        res = _k.compute(state, nl, params,
                         _k.KernelVariant(TAG, None, variant.precision), threads)
        out = ref_kernels.ForceEnergyResult(res.forces, res.potential_energy,
                                            res.per_atom_energy, res.stats)
        out.virial = res.virial
        return out
    compute._b200_orig = orig
    return compute


def install(tersoffmd):
    """Register the B200 variant in an imported `tersoffmd` package.
    Idempotent; returns the package."""
    kern = importlib.import_module(tersoffmd.__name__ + ".kernels")
    if TAG not in kern.KERNEL_TAGS:
        kern.KERNEL_TAGS = tuple(kern.KERNEL_TAGS) + (TAG,)
    orig = getattr(kern.compute, "_b200_orig", kern.compute)
    wrapped = _b200_compute(kern, orig)
    for name in _MODULES:
        try:
            mod = importlib.import_module(f"{tersoffmd.__name__}.{name}")
        except ImportError:
            continue
        if getattr(mod, "compute", None) is not None and \
                getattr(mod.compute, "_b200_orig", mod.compute) is orig:
            mod.compute = wrapped
        names = getattr(mod, "_VARIANT_NAMES", None)
        if isinstance(names, dict):
            names.setdefault("b200", TAG)
    return tersoffmd


def uninstall(tersoffmd):
    """Undo install() (tests)."""
    kern = importlib.import_module(tersoffmd.__name__ + ".kernels")
    orig = getattr(kern.compute, "_b200_orig", None)
    if orig is None:
        return tersoffmd
    for name in _MODULES:
        try:
            mod = importlib.import_module(f"{tersoffmd.__name__}.{name}")
        except ImportError:
            continue
        if getattr(getattr(mod, "compute", None), "_b200_orig", None) is orig:
            mod.compute = orig
        names = getattr(mod, "_VARIANT_NAMES", None)
        if isinstance(names, dict):
            names.pop("b200", None)
    kern.KERNEL_TAGS = tuple(t for t in kern.KERNEL_TAGS if t != TAG)
    return tersoffmd
