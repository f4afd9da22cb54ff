// The reduced (macromodel) system of the paper:
//
//   ( D - G^(E^,J^) T A^-1 B ) E^ = V^            eq. finalsystem
//
// solved by GMRES, which needs the product (eq. MV_product1)
//
//   ( D - G T A^-1 B ) Y,
//
// "T, A and B are block-diagonal matrices with M blocks ... D is also a
// block-diagonal matrix", and "matrices T_m, A_m and B_m
// only need to be calculated once for each distinct element" (PAPER.md:
// 422-425).  G is the AIM-accelerated exterior EFIE operator; with the sign
// convention of reading D1, G = -Z_eq, so the product is D Y + Z_eq (K Y) with
// K_m = T_m A_m^-1 B_m.
//
// The macromodel blocks (D_m, T_m, A_m, B_m) come from the interior problem of
// each element's scatterer and its dual-basis testing (§III-IV), which
// this build does not construct (the paper's element geometries are not
// available): the caller supplies them per element TYPE.  At
// set-up the library inverts every A_m on the device (Gauss-Jordan) and forms
// K_m = T_m (A_m^-1 B_m) with two GEMMs; each product then applies K and D as
// GEMMs over the elements of a type (FP64, many right-hand sides) around one
// aim_matvec.
#include <algorithm>
#include <vector>

#include "aim_internal.cuh"

namespace aim {

void free_reduced(aim_plan* p) {
    free_blocks(p, p->rd_D);
    free_blocks(p, p->rd_K);
    p->release(p->rd_t);
    p->rd_t = nullptr;
    p->rd_on = 0;
}

void reduced_set(aim_plan* p, int ntypes, const int32_t* nhat, const int32_t* nint, const double2* D,
                 const double2* T, const double2* A, const double2* B, const int32_t* elem_type, int nelem) {
    cudaStream_t s = p->stream;
    free_reduced(p);
    ensure_elements(p, s);
    if (nelem != p->el_count)
        throw Error(AIM_E_ARG, "n_elements " + std::to_string(nelem) + " != " + std::to_string(p->el_count) +
                                   " connected surfaces of the mesh");
    for (int d = 0; d < ntypes; ++d)
        if (nhat[d] < 1 || nint[d] < 1) throw Error(AIM_E_ARG, "block sizes must be >= 1");
    for (int e = 0; e < nelem; ++e) {
        const int d = elem_type[e];
        if (d < 0 || d >= ntypes) throw Error(AIM_E_ARG, "element type out of range");
        if (p->el_rptr_h[e + 1] - p->el_rptr_h[e] != nhat[d])
            throw Error(AIM_E_ARG, "element " + std::to_string(e) + " has " +
                                       std::to_string(p->el_rptr_h[e + 1] - p->el_rptr_h[e]) +
                                       " RWGs, its type declares " + std::to_string(nhat[d]));
    }
    std::vector<int> sizes(nhat, nhat + ntypes);
    std::vector<int64_t> off(ntypes + 1, 0);
    for (int d = 0; d < ntypes; ++d) off[d + 1] = off[d] + (int64_t)nhat[d] * nhat[d];
    try {
        for (BlockSet* b : {&p->rd_D, &p->rd_K}) {
            b->mats = p->alloc<double2>(off[ntypes]);
            b->off = p->alloc<int64_t>(ntypes + 1);
            h2d(b->off, off.data(), sizeof(int64_t) * (ntypes + 1), s);
        }
        h2d(p->rd_D.mats, D, sizeof(double2) * off[ntypes], s);
        // K_d = T_d (A_d^-1 B_d)
        const double2 *Td = T, *Ad = A, *Bd = B;
        for (int d = 0; d < ntypes; ++d) {
            const long long nh = nhat[d], ni = nint[d];
            double2 *dA = nullptr, *dB = nullptr, *dT = nullptr, *dW = nullptr;
            AIM_CUDA(cudaMalloc(&dA, sizeof(double2) * ni * ni));
            AIM_CUDA(cudaMalloc(&dB, sizeof(double2) * ni * nh));
            AIM_CUDA(cudaMalloc(&dT, sizeof(double2) * nh * ni));
            AIM_CUDA(cudaMalloc(&dW, sizeof(double2) * ni * nh));
            h2d(dA, Ad, sizeof(double2) * ni * ni, s);
            h2d(dB, Bd, sizeof(double2) * ni * nh, s);
            h2d(dT, Td, sizeof(double2) * nh * ni, s);
            try {
                invert_blocks(dA, std::vector<int64_t>{0}, std::vector<int>{(int)ni}, s);
            } catch (...) {
                cudaFree(dA); cudaFree(dB); cudaFree(dT); cudaFree(dW);
                throw;
            }
            zgemm_rm(dA, dB, dW, (int)ni, (int)nh, (int)ni, s);
            zgemm_rm(dT, dW, p->rd_K.mats + off[d], (int)nh, (int)nh, (int)ni, s);
            AIM_CUDA(cudaStreamSynchronize(s));
            cudaFree(dA); cudaFree(dB); cudaFree(dT); cudaFree(dW);
            Td += nh * ni;
            Ad += ni * ni;
            Bd += ni * nh;
        }
        std::vector<int32_t> map(elem_type, elem_type + nelem);
        setup_block_apply(p, p->rd_D, map, sizes, s);
        setup_block_apply(p, p->rd_K, map, sizes, s);
        p->rd_t = p->alloc<double2>(p->N);
        AIM_CUDA(cudaStreamSynchronize(s));
    } catch (...) {
        free_reduced(p);
        throw;
    }
    p->rd_on = 1;
}

// out = D Y - G (K Y) = D Y + Z_eq (K Y)   (D1: G = -Z_eq)
void reduced_matvec(aim_plan* p, const double2* Y, double2* out, cudaStream_t s) {
    if (!p->rd_on) throw Error(AIM_E_ARG, "no reduced system set (aim_reduced_set)");
    apply_blocks(p, p->rd_K, Y, p->rd_t, false, s);
    matvec(p, p->rd_t, out, 1, s);
    apply_blocks(p, p->rd_D, Y, out, true, s);
}

}  // namespace aim
