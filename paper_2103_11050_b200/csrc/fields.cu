// fields.cu — seeded permeability fields on the device and the field file
// formats (the reference's generator and loader are
// proj/src/fields_io.cpp:25-85 and :91-116).
//
// The reference samples its Gaussian field by a dense Cholesky of the
// covariance (capped at 2^16 cells, fields_io.cpp:28-29). The BASELINE
// configs need 4096^2 cells (C5), so the generators here are the ones of
// paper_2103_11050_b200/configs.py, on the device:
//   exp_lognormal  ln K ~ GRF with covariance var exp(-r / l): circulant
//                  embedding on the doubled periodic grid, two 2-D FFTs
//                  (cuFFT), negative embedding eigenvalues clipped
//   white_noise    K = 1 + amp U(-1, 1)
//   channels       sinuous high-k channels over a low-k background
// with counter-based normals (Philox4x32-10 + Box-Muller), so a field is a
// pure function of (shape, parameters, seed) and the host restatement in
// tests/field_ref.py reproduces it.
// Files: a binary format ("MPM2PFLD", version, nx, ny, nx*ny little-endian
// doubles) and the reference's plain-matrix text ("nx ny" then rows of
// %.17g values; fields_io.cpp:91-116, 118-136), both read and written here.
#include <cufft.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/mpm2p_fields.h"
#include "common.cuh"

namespace {

thread_local std::string g_field_err;

struct FieldError : std::runtime_error {
    int code;
    FieldError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void cuda_ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw FieldError(MPM2P_FIELD_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
void fft_ok(cufftResult r, const char* what) {
    if (r != CUFFT_SUCCESS) throw FieldError(MPM2P_FIELD_ECUDA, std::string(what) + ": cuFFT error " + std::to_string((int)r));
}

template <typename F>
int guarded(F&& fn) {
    try {
        fn();
        return MPM2P_FIELD_OK;
    } catch (const FieldError& e) {
        g_field_err = e.what();
        return e.code;
    } catch (const std::bad_alloc& e) {
        g_field_err = std::string("host allocation failed: ") + e.what();
        return MPM2P_FIELD_ECAPACITY;
    } catch (const std::exception& e) {
        g_field_err = std::string("internal error: ") + e.what();
        return MPM2P_FIELD_EINTERNAL;
    }
}

template <typename T>
struct Dev {
    T* p = nullptr;
    explicit Dev(size_t n) { cuda_ok(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)), "cudaMalloc"); }
    ~Dev() { cudaFree(p); }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
};

// ---- Philox4x32-10 (Salmon et al. 2011), counter (idx, stream), key = seed
__host__ __device__ inline void philox(uint32_t c[4], uint32_t k0, uint32_t k1) {
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c[0], p1 = (uint64_t)0xCD9E8D57u * c[2];
        const uint32_t h0 = (uint32_t)(p0 >> 32), l0 = (uint32_t)p0, h1 = (uint32_t)(p1 >> 32), l1 = (uint32_t)p1;
        const uint32_t n0 = h1 ^ c[1] ^ k0, n2 = h0 ^ c[3] ^ k1;
        c[0] = n0, c[1] = l1, c[2] = n2, c[3] = l0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}
// two uniforms in (0, 1] with 53-bit resolution from one counter
__device__ inline void uniform2(uint64_t idx, uint32_t stream, uint64_t seed, double& u1, double& u2) {
    uint32_t c[4] = {(uint32_t)idx, (uint32_t)(idx >> 32), stream, 0u};
    philox(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    const double s53 = 1.0 / 9007199254740992.0;  // 2^-53
    u1 = ((double)((((uint64_t)(c[0] >> 5)) << 26) | (c[1] >> 6)) + 1.0) * s53;
    u2 = ((double)((((uint64_t)(c[2] >> 5)) << 26) | (c[3] >> 6)) + 1.0) * s53;
}
// a Box-Muller pair of standard normals
__device__ inline void normal2(uint64_t idx, uint32_t stream, uint64_t seed, double& z1, double& z2) {
    double u1, u2;
    uniform2(idx, stream, seed, u1, u2);
    const double r = sqrt(__dmul_rn(-2.0, log(u1)));
    double sn, cs;
    sincospi(2.0 * u2, &sn, &cs);
    z1 = __dmul_rn(r, cs);
    z2 = __dmul_rn(r, sn);
}

constexpr int TPB = 256;
int blocks(long long n) { return (int)std::min<long long>((n + TPB - 1) / TPB, 148LL * 32); }

// c on the doubled periodic grid (configs.py exp_covariance_lognormal)
__global__ void k_cov(int mx, int my, double hx, double hy, double corr, double var, cufftDoubleComplex* c) {
    const long long n = (long long)mx * my;
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < n; x += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(x % mx), j = (int)(x / mx);
        const double dx = (double)min(i, mx - i) * hx, dy = (double)min(j, my - j) * hy;
        const double r = sqrt(__dadd_rn(__dmul_rn(dy, dy), __dmul_rn(dx, dx)));
        c[x] = make_cuDoubleComplex(var * exp(-r / corr), 0.0);
    }
}
// w = sqrt(max(Re lam, 0) / (mx my)) * (n1 + i n2)
__global__ void k_weight(long long n, uint64_t seed, double nn, cufftDoubleComplex* c) {
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < n; x += (long long)gridDim.x * blockDim.x) {
        const double lam = fmax(c[x].x, 0.0);
        double z1, z2;
        normal2((uint64_t)x, 0u, seed, z1, z2);
        const double w = sqrt(lam / nn);
        c[x] = make_cuDoubleComplex(w * z1, w * z2);
    }
}
__global__ void k_exp_crop(int nx, int ny, int mx, const cufftDoubleComplex* __restrict__ z, double* __restrict__ K) {
    const long long n = (long long)nx * ny;
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < n; x += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(x % nx), j = (int)(x / nx);
        K[x] = exp(z[(long long)j * mx + i].x);
    }
}
__global__ void k_white(long long n, uint64_t seed, double amp, double* K) {
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < n; x += (long long)gridDim.x * blockDim.x) {
        double u1, u2;
        uniform2((uint64_t)x, 0u, seed, u1, u2);
        K[x] = __dadd_rn(1.0, __dmul_rn(amp, __dsub_rn(__dmul_rn(2.0, u1), 1.0)));
    }
}
// one channel y = y0 + a sin(2 pi x / wav + phi), half-width `half`, OR-ed into the mask; counts new cells
__global__ void k_channel(int nx, int ny, double hx, double hy, double y0, double a, double wav, double phi,
                          double half, unsigned char* mask, unsigned long long* count) {
    const long long n = (long long)nx * ny;
    unsigned long long add = 0;
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < n; x += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(x % nx), j = (int)(x / nx);
        const double X = __dmul_rn(i + 0.5, hx), Y = __dmul_rn(j + 0.5, hy);
        const double yc = __dadd_rn(y0, __dmul_rn(a, sin(__dadd_rn(__ddiv_rn(__dmul_rn(2.0 * M_PI, X), wav), phi))));
        if (!mask[x] && fabs(Y - yc) < half) {
            mask[x] = 1;
            ++add;
        }
    }
    atomicAdd(count, add);
}
__global__ void k_channel_values(long long n, uint64_t seed, const unsigned char* mask, double mc, double sc, double mb,
                                 double sb, double* K) {
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < n; x += (long long)gridDim.x * blockDim.x) {
        double z1, z2;
        normal2((uint64_t)x, 2u, seed, z1, z2);
        K[x] = mask[x] ? exp(__dadd_rn(mc, __dmul_rn(sc, z1))) : exp(__dadd_rn(mb, __dmul_rn(sb, z1)));
    }
}

void check_shape(int nx, int ny) {
    if (nx < 1 || ny < 1) throw FieldError(MPM2P_FIELD_ECONFIG, "field: cell counts must be >= 1");
}

// host Philox uniforms for the channel parameters (stream 1): the same
// mapping as the device's uniform2
void host_uniform2(uint64_t idx, uint64_t seed, double& u1, double& u2) {
    uint32_t c[4] = {(uint32_t)idx, (uint32_t)(idx >> 32), 1u, 0u};
    philox(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    const double s53 = 1.0 / 9007199254740992.0;
    u1 = ((double)((((uint64_t)(c[0] >> 5)) << 26) | (c[1] >> 6)) + 1.0) * s53;
    u2 = ((double)((((uint64_t)(c[2] >> 5)) << 26) | (c[3] >> 6)) + 1.0) * s53;
}

const char MAGIC[8] = {'M', 'P', 'M', '2', 'P', 'F', 'L', 'D'};

}  // namespace

extern "C" {

const char* mpm2p_field_error(void) { return g_field_err.c_str(); }

int mpm2p_field_exp_lognormal(int32_t nx, int32_t ny, double lx, double ly, double corr_len, double variance,
                              uint64_t seed, double* K) {
    return guarded([&] {
        check_shape(nx, ny);
        if (!(lx > 0.0) || !(ly > 0.0) || !(corr_len > 0.0) || !(variance >= 0.0))
            throw FieldError(MPM2P_FIELD_ECONFIG, "exp_lognormal: lengths and correlation length must be positive");
        const int mx = 2 * nx, my = 2 * ny;
        const long long n = (long long)mx * my;
        Dev<cufftDoubleComplex> c(n);
        Dev<double> k((size_t)nx * ny);
        k_cov<<<blocks(n), TPB>>>(mx, my, lx / nx, ly / ny, corr_len, variance, c.p);
        cuda_ok(cudaGetLastError(), "k_cov");
        cufftHandle plan;
        fft_ok(cufftPlan2d(&plan, my, mx, CUFFT_Z2Z), "cufftPlan2d");
        try {
            fft_ok(cufftExecZ2Z(plan, c.p, c.p, CUFFT_FORWARD), "fft(c)");
            k_weight<<<blocks(n), TPB>>>(n, seed, (double)n, c.p);
            cuda_ok(cudaGetLastError(), "k_weight");
            fft_ok(cufftExecZ2Z(plan, c.p, c.p, CUFFT_FORWARD), "fft(w)");
        } catch (...) {
            cufftDestroy(plan);
            throw;
        }
        cufftDestroy(plan);
        k_exp_crop<<<blocks((long long)nx * ny), TPB>>>(nx, ny, mx, c.p, k.p);
        cuda_ok(cudaGetLastError(), "k_exp_crop");
        cuda_ok(cudaMemcpy(K, k.p, (size_t)nx * ny * sizeof(double), cudaMemcpyDeviceToHost), "copy K");
    });
}

int mpm2p_field_white_noise(int32_t nx, int32_t ny, double amp, uint64_t seed, double* K) {
    return guarded([&] {
        check_shape(nx, ny);
        const long long n = (long long)nx * ny;
        Dev<double> k(n);
        k_white<<<blocks(n), TPB>>>(n, seed, amp, k.p);
        cuda_ok(cudaGetLastError(), "k_white");
        cuda_ok(cudaMemcpy(K, k.p, n * sizeof(double), cudaMemcpyDeviceToHost), "copy K");
    });
}

int mpm2p_field_channels(int32_t nx, int32_t ny, double lx, double ly, uint64_t seed, double coverage, double k_chan,
                         double sd_chan, double k_back, double sd_back, double* K) {
    return guarded([&] {
        check_shape(nx, ny);
        if (!(k_chan > 0.0) || !(k_back > 0.0)) throw FieldError(MPM2P_FIELD_ECONFIG, "channels: k values must be positive");
        const long long n = (long long)nx * ny;
        Dev<unsigned char> mask(n);
        Dev<unsigned long long> cnt(1);
        Dev<double> k(n);
        cuda_ok(cudaMemset(mask.p, 0, n), "memset");
        cuda_ok(cudaMemset(cnt.p, 0, sizeof(unsigned long long)), "memset");
        unsigned long long covered = 0;
        for (int t = 0; t < 64 && (double)covered < coverage * (double)n; ++t) {
            double u[6];
            host_uniform2(3 * (uint64_t)t, seed, u[0], u[1]);
            host_uniform2(3 * (uint64_t)t + 1, seed, u[2], u[3]);
            host_uniform2(3 * (uint64_t)t + 2, seed, u[4], u[5]);
            const double y0 = u[0] * ly, amp = (0.05 + 0.15 * u[1]) * ly, wav = (0.3 + 0.5 * u[2]) * lx;
            const double phi = 2.0 * M_PI * u[3], half = (0.03 + 0.04 * u[4]) * ly;
            k_channel<<<blocks(n), TPB>>>(nx, ny, lx / nx, ly / ny, y0, amp, wav, phi, half, mask.p, cnt.p);
            cuda_ok(cudaGetLastError(), "k_channel");
            cuda_ok(cudaMemcpy(&covered, cnt.p, sizeof(covered), cudaMemcpyDeviceToHost), "copy count");
        }
        k_channel_values<<<blocks(n), TPB>>>(n, seed, mask.p, std::log(k_chan), sd_chan, std::log(k_back), sd_back, k.p);
        cuda_ok(cudaGetLastError(), "k_channel_values");
        cuda_ok(cudaMemcpy(K, k.p, n * sizeof(double), cudaMemcpyDeviceToHost), "copy K");
    });
}

int mpm2p_field_save(const char* path, int32_t nx, int32_t ny, const double* K) {
    return guarded([&] {
        check_shape(nx, ny);
        FILE* f = std::fopen(path, "wb");
        if (!f) throw FieldError(MPM2P_FIELD_ECONFIG, std::string("field_save: cannot write ") + path);
        const uint32_t version = 1;
        bool ok = std::fwrite(MAGIC, 1, 8, f) == 8 && std::fwrite(&version, 4, 1, f) == 1 &&
                  std::fwrite(&nx, 4, 1, f) == 1 && std::fwrite(&ny, 4, 1, f) == 1 &&
                  std::fwrite(K, sizeof(double), (size_t)nx * ny, f) == (size_t)nx * ny;
        ok = (std::fclose(f) == 0) && ok;
        if (!ok) throw FieldError(MPM2P_FIELD_ECONFIG, std::string("field_save: I/O failure writing ") + path);
    });
}

int mpm2p_field_load(const char* path, int32_t nx, int32_t ny, double* K) {
    return guarded([&] {
        check_shape(nx, ny);
        FILE* f = std::fopen(path, "rb");
        if (!f) throw FieldError(MPM2P_FIELD_ECONFIG, std::string("load_field: cannot open ") + path);
        char head[8] = {0};
        const size_t got = std::fread(head, 1, 8, f);
        const size_t n = (size_t)nx * ny;
        if (got == 8 && std::memcmp(head, MAGIC, 8) == 0) {  // binary
            uint32_t version = 0;
            int32_t fx = -1, fy = -1;
            if (std::fread(&version, 4, 1, f) != 1 || std::fread(&fx, 4, 1, f) != 1 || std::fread(&fy, 4, 1, f) != 1 ||
                version != 1) {
                std::fclose(f);
                throw FieldError(MPM2P_FIELD_ECONFIG, std::string("load_field: bad header in ") + path);
            }
            if (fx != nx || fy != ny) {
                std::fclose(f);
                throw FieldError(MPM2P_FIELD_ECONFIG, std::string("load_field: ") + path + " holds a " +
                                                          std::to_string(fx) + "x" + std::to_string(fy) +
                                                          " field, expected " + std::to_string(nx) + "x" +
                                                          std::to_string(ny));
            }
            const size_t r = std::fread(K, sizeof(double), n, f);
            std::fclose(f);
            if (r != n) throw FieldError(MPM2P_FIELD_ECONFIG, std::string("load_field: truncated ") + path);
            return;
        }
        // the reference's plain-matrix text (fields_io.cpp:91-116): "nx ny", then ny rows of nx values
        std::fseek(f, 0, SEEK_END);
        const long len = std::ftell(f);
        std::fseek(f, 0, SEEK_SET);
        std::vector<char> buf((size_t)len + 1, 0);
        const size_t rd = std::fread(buf.data(), 1, (size_t)len, f);
        std::fclose(f);
        buf[rd] = 0;
        char* p = buf.data();
        char* e = nullptr;
        const long fx = std::strtol(p, &e, 10);
        if (e == p) throw FieldError(MPM2P_FIELD_ECONFIG, std::string("load_field: bad header in ") + path);
        p = e;
        const long fy = std::strtol(p, &e, 10);
        if (e == p) throw FieldError(MPM2P_FIELD_ECONFIG, std::string("load_field: bad header in ") + path);
        p = e;
        if (fx != nx || fy != ny)
            throw FieldError(MPM2P_FIELD_ECONFIG, std::string("load_field: ") + path + " holds a " + std::to_string(fx) +
                                                      "x" + std::to_string(fy) + " field, expected " +
                                                      std::to_string(nx) + "x" + std::to_string(ny));
        for (size_t x = 0; x < n; ++x) {
            const double v = std::strtod(p, &e);
            if (e == p)
                throw FieldError(MPM2P_FIELD_ECONFIG, std::string("load_field: parse failure in ") + path + " at row " +
                                                          std::to_string(x / nx + 1) + " column " +
                                                          std::to_string(x % nx + 1));
            K[x] = v;
            p = e;
        }
    });
}

int mpm2p_field_save_text(const char* path, int32_t nx, int32_t ny, const double* K) {
    return guarded([&] {
        check_shape(nx, ny);
        FILE* f = std::fopen(path, "w");
        if (!f) throw FieldError(MPM2P_FIELD_ECONFIG, std::string("save_cell_field: cannot write ") + path);
        bool ok = std::fprintf(f, "%d %d\n", nx, ny) > 0;
        for (int j = 0; j < ny && ok; ++j)
            for (int i = 0; i < nx && ok; ++i) ok = std::fprintf(f, i + 1 < nx ? "%.17g " : "%.17g\n", K[(size_t)j * nx + i]) > 0;
        ok = (std::fclose(f) == 0) && ok;
        if (!ok) throw FieldError(MPM2P_FIELD_ECONFIG, std::string("save_cell_field: I/O failure writing ") + path);
    });
}

}  // extern "C"
