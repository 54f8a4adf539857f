"""Fig.-4-shaped PSF report (SPEC fwhm_sweep S:534-538): wire
phantom at 5..25 mm through the GPU path (DAS + IQ envelope, pre-log),
lateral / axial FWHM per depth as CSV.  Dev/validation aid."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from synth import configs  # noqa: E402
from test_psf_gpu import DEPTHS, _sweep  # noqa: E402

print("aperture,depth_mm,lateral_fwhm_mm,axial_fwhm_mm,peak_lateral_mm,peak_depth_mm")
for name, w in (("F1_dynamic", configs.psf_linear()), ("fixed_full", configs.psf_linear(f_number=0.02))):
    for z, r in zip(DEPTHS, _sweep(w)):
        print(f"{name},{z:.1f},{r['lateral_fwhm']:.4f},{r['axial_fwhm']:.4f},{r['peak_lateral']:.4f},"
              f"{r['peak_depth']:.4f}")
