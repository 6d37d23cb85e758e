// halo.cu -- face-trace halo of the element partition (comm.h).
//
// GLL nodes make a face trace the value at the boundary node (P:201 with
// l_i(+-1) = delta), so a rank sends, for every element along each partition
// side, the NV x (N+1) boundary-node values of each field, and receives its
// neighbour's into ghost elements (layout L, only face nodes written) that the
// operator kernels address as elements nE + g (ops.cuh nbr_elem).
//
// Gauss-Legendre nodes (no node on the edge): the sender interpolates the
// trace sum_l l_l(+-1) w_l along the line through face node k and the ghost's
// edge-node slot holds that trace (the GL kernels read ghosts directly).
//
// Buffer layout: side segments s = 0 (-x), 1 (+x), 2 (-y), 3 (+y); inside a
// segment [pos][field][var][k], pos = ey (x-sides) or ex (y-sides), k the
// node index along the face.  A field has nvf "variables" of NODES values per
// element (nvf = n_v for states; 6 x jet components for NS lifted gradients).
#include "launch.h"

namespace {

struct HaloArgs {
  const double* src[HALO_MAX_FIELDS];
  double* dst[HALO_MAX_FIELDS];
  size_t off[4];        // segment offsets (doubles)
  int nel[4];           // elements along side s (0 if the side is inactive)
  int nf, nx, ny, nE, nv, P, dim, m, nodes;
  size_t total;
  int gl;
  double lp[8], lm[8];
  int facebuf;          // BR2 face-gradient buffers [elem][face 4][nv][P]: send face s, fill ghost face s^1
};

__device__ __forceinline__ int face_node(int s, int k, int P, int dim) {
  if (dim == 1) return (s & 1) ? P - 1 : 0;
  switch (s) {
    case 0: return k * P;              // i = 0
    case 1: return k * P + P - 1;      // i = N
    case 2: return k;                  // j = 0
    default: return (P - 1) * P + k;   // j = N
  }
}

__device__ __forceinline__ void decode(const HaloArgs& H, size_t t, int& s, int& p, int& f, int& v, int& k,
                                       size_t& flat) {
  const int FN = H.dim == 2 ? H.P : 1;
  size_t acc = 0;
  s = 0;
  for (int q = 0; q < 4; ++q) {
    const size_t len = (size_t)H.nel[q] * H.nf * H.nv * FN;
    if (t < acc + len) { s = q; break; }
    acc += len;
  }
  size_t r = t - acc;
  flat = H.off[s] + r;
  k = (int)(r % FN); r /= FN;
  v = (int)(r % H.nv); r /= H.nv;
  f = (int)(r % H.nf); r /= H.nf;
  p = (int)r;
}

__global__ void halo_pack_kernel(HaloArgs H, double* __restrict__ send) {
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < H.total; t += (size_t)gridDim.x * blockDim.x) {
    int s, p, f, v, k;
    size_t flat;
    decode(H, t, s, p, f, v, k, flat);
    int e;
    switch (s) {
      case 0: e = p * H.nx; break;
      case 1: e = p * H.nx + H.nx - 1; break;
      case 2: e = p; break;
      default: e = (H.ny - 1) * H.nx + p; break;
    }
    if (H.facebuf) {
      send[flat] = H.src[f][(((size_t)e * 4 + s) * H.nv + v) * H.P + k];
      continue;
    }
    const double* base = H.src[f] + (size_t)e * H.m + v * H.nodes;
    if (H.gl) {
      // trace on face s: line through face node k across the element (x-sides: row k, y-sides: column k)
      const double* l = (s & 1) ? H.lp : H.lm;
      double acc = 0.0;
      for (int q = 0; q < H.P; ++q) {
        const int nd = H.dim == 1 ? q : (s < 2 ? k * H.P + q : q * H.P + k);
        acc = fma(l[q], base[nd], acc);
      }
      send[flat] = acc;
    } else {
      send[flat] = base[face_node(s, k, H.P, H.dim)];
    }
  }
}

__global__ void halo_unpack_kernel(HaloArgs H, const double* __restrict__ recv) {
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < H.total; t += (size_t)gridDim.x * blockDim.x) {
    int s, p, f, v, k;
    size_t flat;
    decode(H, t, s, p, f, v, k, flat);
    int gi;
    switch (s) {
      case 0: gi = p; break;
      case 1: gi = H.ny + p; break;
      case 2: gi = 2 * H.ny + p; break;
      default: gi = 2 * H.ny + H.nx + p; break;
    }
    // the neighbour across side s touches us with its face s ^ 1
    if (H.facebuf)
      H.dst[f][(((size_t)gi * 4 + (s ^ 1)) * H.nv + v) * H.P + k] = recv[flat];
    else
      H.dst[f][(size_t)gi * H.m + v * H.nodes + face_node(s ^ 1, k, H.P, H.dim)] = recv[flat];
  }
}

HaloArgs make_args(const HaloLayout& L, int nf, int nvf) {
  HaloArgs H{};
  H.nf = nf;
  H.nx = L.nx; H.ny = L.ny; H.nE = L.nx * L.ny; H.nv = nvf > 0 ? nvf : L.nv; H.P = L.P; H.dim = L.dim;
  H.nodes = L.dim == 2 ? L.P * L.P : L.P;
  H.m = H.nv * H.nodes;
  H.gl = L.gl;
  for (int q = 0; q < 8; ++q) { H.lp[q] = L.lp[q]; H.lm[q] = L.lm[q]; }
  const int FN = L.dim == 2 ? L.P : 1;
  size_t acc = 0;
  for (int s = 0; s < 4; ++s) {
    H.nel[s] = L.active[s] ? (s < 2 ? L.ny : L.nx) : 0;
    H.off[s] = acc;
    acc += (size_t)H.nel[s] * nf * H.nv * FN;
  }
  H.total = acc;
  return H;
}

}  // namespace

void halo_segments(const HaloLayout& L, int nf, size_t off[4], size_t len[4], int nvf) {
  const HaloArgs H = make_args(L, nf, nvf);
  const int FN = L.dim == 2 ? L.P : 1;
  for (int s = 0; s < 4; ++s) {
    off[s] = H.off[s];
    len[s] = (size_t)H.nel[s] * nf * H.nv * FN;
  }
}

cudaError_t launch_halo_pack(const HaloLayout& L, int nf, const double* const* src, double* send,
                             cudaStream_t st, int nvf, bool facebuf) {
  if (nf < 1 || nf > HALO_MAX_FIELDS) return cudaErrorInvalidValue;
  HaloArgs H = make_args(L, nf, nvf);
  H.facebuf = facebuf;
  for (int f = 0; f < nf; ++f) H.src[f] = src[f];
  if (H.total == 0) return cudaSuccess;
  const int grid = (int)std::min<size_t>((H.total + 255) / 256, 1184);
  halo_pack_kernel<<<grid, 256, 0, st>>>(H, send);
  hbpdc_count_launch();
  return cudaGetLastError();
}

cudaError_t launch_halo_unpack(const HaloLayout& L, int nf, const double* recv, double* const* dst,
                               cudaStream_t st, int nvf, bool facebuf) {
  if (nf < 1 || nf > HALO_MAX_FIELDS) return cudaErrorInvalidValue;
  HaloArgs H = make_args(L, nf, nvf);
  H.facebuf = facebuf;
  for (int f = 0; f < nf; ++f) H.dst[f] = dst[f];
  if (H.total == 0) return cudaSuccess;
  const int grid = (int)std::min<size_t>((H.total + 255) / 256, 1184);
  halo_unpack_kernel<<<grid, 256, 0, st>>>(H, recv);
  hbpdc_count_launch();
  return cudaGetLastError();
}

// out = c / sqrt(*sum), 0 if the sum is 0 (FD step from an all-reduced sum)
__global__ void fd_eps_from_sum_kernel(const double* __restrict__ sum, double c, double* out) {
  const double s = *sum;
  *out = s > 0.0 ? c / sqrt(s) : 0.0;
}

cudaError_t launch_fd_eps_from_sum(const double* sum, double c, double* out, cudaStream_t st) {
  fd_eps_from_sum_kernel<<<1, 1, 0, st>>>(sum, c, out);
  hbpdc_count_launch();
  return cudaGetLastError();
}
