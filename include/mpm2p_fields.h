/*
 * mpm2p_fields.h — seeded permeability fields generated on the device, and
 * the field file formats. Library: libmpm2p_fields.so
 * (csrc/fields.cu; links cuFFT).
 *
 * Reference counterparts (proj/include/mrcmflow/fields_io.hpp):
 *   generate_gaussian / GaussianSampler (fields_io.cpp:25-85) samples by a
 *   dense Cholesky of the covariance and refuses grids above 2^16 cells; the
 *   generators below are the BASELINE configs' own at any
 *   size: exponential-covariance log-normal by FFT circulant embedding,
 *   K = 1 + amp U(-1,1), and sinuous channels. Normals are counter-based
 *   (Philox4x32-10 + Box-Muller): a field is a pure function of its shape,
 *   parameters and seed.
 *   load_cell_field (fields_io.cpp:91-116) and save_cell_field(PlainMatrix)
 *   (:118-136): mpm2p_field_load reads the reference's plain-matrix text or
 *   the binary format ("MPM2PFLD", uint32 version 1, int32 nx, int32 ny,
 *   nx*ny little-endian doubles, row-major j*nx+i), detected by its magic.
 * All K pointers are host arrays of nx*ny doubles (row-major).
 */
#ifndef MPM2P_FIELDS_H
#define MPM2P_FIELDS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    MPM2P_FIELD_OK = 0,
    MPM2P_FIELD_ECONFIG = 2,   /* ConfigError (bad shape / parameters / file) */
    MPM2P_FIELD_ECAPACITY = 4, /* CapacityError */
    MPM2P_FIELD_ECUDA = 5,
    MPM2P_FIELD_EINTERNAL = 6
};

const char* mpm2p_field_error(void);
/* ln K ~ GRF, covariance variance * exp(-|x - y| / corr_len), on the cell centres */
int mpm2p_field_exp_lognormal(int32_t nx, int32_t ny, double lx, double ly, double corr_len, double variance,
                              uint64_t seed, double* K);
/* K = 1 + amp U(-1, 1) */
int mpm2p_field_white_noise(int32_t nx, int32_t ny, double amp, uint64_t seed, double* K);
/* channels y = y0 + A sin(2 pi x / L + phi) added until `coverage` of the cells;
 * ln K ~ N(ln k_chan, sd_chan^2) in channels, N(ln k_back, sd_back^2) elsewhere */
int mpm2p_field_channels(int32_t nx, int32_t ny, double lx, double ly, uint64_t seed, double coverage, double k_chan,
                         double sd_chan, double k_back, double sd_back, double* K);
int mpm2p_field_save(const char* path, int32_t nx, int32_t ny, const double* K);      /* binary */
int mpm2p_field_save_text(const char* path, int32_t nx, int32_t ny, const double* K); /* plain matrix %.17g */
int mpm2p_field_load(const char* path, int32_t nx, int32_t ny, double* K);            /* either format */

#ifdef __cplusplus
}
#endif

#endif /* MPM2P_FIELDS_H */
