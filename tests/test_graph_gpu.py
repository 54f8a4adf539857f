"""CUDA-graph capture of the C-ABI calls (SURVEY 8(b) "Ownership": the
library never allocates or synchronises per call, so calls are capturable;
the paper's 2D path was "limited by CUDA management operations", P:341,
P:344 -- a captured graph removes the per-call launch work).

One graph holds beamform + scanconvert for 6 rotating raw buffers; replaying
it reproduces the eager results bitwise, and after the buffers' contents
change a replay follows the new data (the graph reads the buffers; only the
per-call tensor maps, kernel parameters, are frozen into it)."""
import pytest

from synth import configs

from gpu_util import raw_frames

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1711_06127_b200 import SupraBF  # noqa: E402


def _eager(bf, raws, F):
    lis, imgs = [], []
    for r in raws:
        li, img = bf.empty_line_img(F), bf.empty_img(F)
        bf.beamform(r, F, line_img=li)
        bf.scanconvert(li, F, img)
        lis.append(li)
        imgs.append(img)
    torch.cuda.synchronize()
    return lis, imgs


@pytest.mark.parametrize("name,F,nbuf", [("C2", 4, 6), ("C2", 3, 10), ("C1", 1, 6)])
def test_graph_capture_rotating_buffers(name, F, nbuf):
    # C2 x 4: batch kernel with row-cut maps; C2 x 3: + a remainder launch and
    # more buffers than the host map cache holds (8); C1 x 1: warp-split kernel
    w = configs.CONFIGS[name](sc_output_type=configs.T_U8)
    base = raw_frames(w, F)
    raws = [torch.roll(base, shifts=7 * i, dims=-1).contiguous() for i in range(nbuf)]
    bf = SupraBF(w, max_frames=F)
    ref_li, ref_img = _eager(bf, raws, F)

    li_g = [bf.empty_line_img(F) for _ in range(nbuf)]
    img_g = [bf.empty_img(F) for _ in range(nbuf)]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):            # warm-up on the capture stream
        bf.beamform(raws[0], F, line_img=li_g[0])
        bf.scanconvert(li_g[0], F, img_g[0])
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(nbuf):
            bf.beamform(raws[i], F, line_img=li_g[i])
            bf.scanconvert(li_g[i], F, img_g[i])
    for t in li_g + img_g:
        t.zero_()
    g.replay()
    torch.cuda.synchronize()
    for i in range(nbuf):
        assert torch.equal(li_g[i], ref_li[i]), i
        assert torch.equal(img_g[i], ref_img[i]), i
    # new contents in the same buffers: the replay follows the data
    for i in range(nbuf):
        raws[i].copy_(torch.roll(base, shifts=-5 * i - 3, dims=-1))
    new_li, new_img = _eager(bf, raws, F)
    g.replay()
    torch.cuda.synchronize()
    for i in range(nbuf):
        assert torch.equal(li_g[i], new_li[i]), i
        assert torch.equal(img_g[i], new_img[i]), i
    bf.close()
