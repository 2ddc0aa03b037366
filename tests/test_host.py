"""Host-side API mirror checks (no GPU needed)."""
import pytest

import paper_2209_08189_b200 as P


def test_public_names_match_reference_surface():
    # every name velreg/__init__.py:10-33 re-exports
    for name in ["GridError", "ObjectiveError", "ResampleError", "SearchError", "TransportError", "VelregError",
                 "VolumeIOError", "Grid", "LabelMap", "ScalarField", "VectorField", "make_grid",
                 "prolong_spectral", "restrict", "RegOperators", "SpectralWorkspace", "apply_A", "apply_K",
                 "apply_inv_shifted_A", "fd8_divergence", "fd8_gradient", "Characteristics", "TransportConfig",
                 "TransportOperators", "interpolate", "jacobian_determinant", "solve_adjoint",
                 "solve_incremental_state", "solve_state", "solve_state_series", "trace_characteristics",
                 "ArmijoConfig", "ObjectiveState", "RegistrationConfig", "SolverDiagnostics",
                 "evaluate_objective", "gauss_newton_register", "hessian_matvec", "pcg_solve",
                 "reduced_gradient", "relative_residual", "make_reference", "make_velocity", "transport_labels",
                 "DiceReport", "dice", "dice_averages", "jacobian_stats", "residual_image", "register", "SearchConfig", "SearchResult",
                 "continuation_register", "in_bounds", "search_beta_v", "search_beta_w", "search_parameters",
                 "ExperimentPlan", "run_experiment", "SynthSpec", "assoc_legendre", "make_template",
                 "spherical_harmonic_magnitude", "load_nifti", "load_volume", "save_volume"]:
        assert hasattr(P, name), name


def test_grid_validation():
    with pytest.raises(P.GridError):
        P.Grid((4, 4))
    with pytest.raises(P.GridError):
        P.Grid((4, 5, 6))
    with pytest.raises(P.GridError):
        P.Grid((2, 4, 4))
    g = P.make_grid((16, 20, 24))
    assert g.num_voxels == 16 * 20 * 24
    assert abs(g.cell_volume - (2 * 3.141592653589793) ** 3 / g.num_voxels) < 1e-12


def test_config_validation():
    with pytest.raises(ValueError):
        P.TransportConfig(n_t=0)
    with pytest.raises(ValueError):
        P.TransportConfig(interp_order="quintic")
    with pytest.raises(ValueError):
        P.RegistrationConfig(gtol=1.5)
    with pytest.raises(ValueError):
        P.RegistrationConfig(max_gn_iters=0)
    assert P.TransportConfig(8).dt == 0.125
    with pytest.raises(ValueError):
        P.RegOperators(0.0, 0.0)
    with pytest.raises(ValueError):
        P.RegOperators(1e-2, -1.0)


def test_error_hierarchy():
    for e in (P.GridError, P.ResampleError, P.VolumeIOError, P.TransportError, P.ObjectiveError, P.SearchError):
        assert issubclass(e, P.VelregError)
    from paper_2209_08189_b200._lib import NativeError
    assert issubclass(NativeError, P.VelregError)


def test_grad_layout_switch():
    """runtime.set_grad_layout validates its argument; forced modes bypass the
    free-memory heuristic (which keeps the stored series on CPU tensors)."""
    import pytest
    import torch
    from paper_2209_08189_b200 import runtime
    with pytest.raises(ValueError):
        runtime.set_grad_layout("bogus")
    try:
        runtime.set_grad_layout("lean")
        assert runtime.lean_layout(1, torch.device("cpu"))
        runtime.set_grad_layout("stored")
        assert not runtime.lean_layout(1 << 60, torch.device("cpu"))
        runtime.set_grad_layout("auto")
        assert not runtime.lean_layout(1 << 60, torch.device("cpu"))
    finally:
        runtime.set_grad_layout("auto")
