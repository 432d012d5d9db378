// kernels.cuh — launch wrappers of the hand-written sm_100a kernels (kernels.cu).
// Every wrapper enqueues on the given stream and returns immediately.
#pragma once

#include <cstdint>

#include <vector>

#include <cuda_runtime.h>

namespace slabgpu {
	struct Decomp;
	struct Sell;
	struct BoxTile;
	namespace kern {

		// ---- vector ops (operations.hpp:49-106)
		void fill( cudaStream_t st, double * v, uint64_t n, double value );
		void waxpby( cudaStream_t st, double * w, double alpha, const double * x, double beta, const double * y,
			uint64_t n );
		// dot, exact: 4096-chunk ordered (operations.hpp:61-91). partials needs ceil(n/4096) doubles.
		void dot_exact_prepare(); // function attributes; call outside stream capture
		void dot_exact( cudaStream_t st, const double * x, const double * y, uint64_t n, double * partials,
			unsigned int * counter, double * out );
		// dot, fixed-shape tree. partials needs dot_tree_blocks(n, sms) doubles.
		uint64_t dot_tree_blocks( uint64_t n, int sm_count );
		void dot_tree( cudaStream_t st, const double * x, const double * y, uint64_t n, int sm_count, double * partials,
			unsigned int * counter, double * out );

		// ---- SELL-32 matrix-vector products (operations.hpp:116-125, :164-174)
		// dot_out != nullptr additionally reduces x'(A x) in the tree-dot shape (cg.hpp:122-123 in one pass);
		// dot_partials then needs spmv_dot_blocks(nrows) doubles
		// Every matrix entry point takes the SELL and runs from its dictionary-coded copy (packed.cu) when
		// one exists and g_use_packed is set; the arithmetic and its order are the same either way.
		void spmv( cudaStream_t st, const Sell & S, const double * x, double * y, int64_t nrows,
			double * dot_partials = nullptr, unsigned int * dot_counter = nullptr, double * dot_out = nullptr );
		uint64_t spmv_dot_blocks( int64_t nrows );
		void spmv_masked( cudaStream_t st, const Sell & S, const double * x, double * y, const int32_t * members,
			int64_t count );
		// out = fold of `count` block partials in a fixed order
		void sum_partials( cudaStream_t st, const double * partials, uint64_t count, double * out );

		// ---- fused Gauss-Seidel colour step (smoother.hpp:60-72) on the colour-major SELL
		// flags bit 0: prolongation fused in front (z[i] += src[k], multigrid.hpp:71-81); bit 1: residual +
		// restriction fused behind (out[k], zero[k] = 0; multigrid.hpp:100-104); both only on colour-0 steps of
		// stencil levels. Bit 2: the step is applied twice in a row (turnaround of a symmetric sweep,
		// smoother.hpp:108-111). Bits 1 and 2 only where gs_color_step_can_fuse_residual(S, pos_count).
		void gs_color_step( cudaStream_t st, const Sell & S, const int32_t * rows, int64_t pos_begin, int64_t pos_count, double * z, const double * r, int flags = 0,
			const double * src = nullptr, double * out = nullptr, double * zero = nullptr, size_t window_bytes = 0,
			const int32_t * pos_list = nullptr, const uint8_t * skip = nullptr );
		// pos_list: cover exactly these positions (pos_count = their number); skip: leave flagged positions out
		// window_bytes > 0: size of z; many-wave launches then ask the L2 to keep z in its persisting carve-out
		bool gs_color_step_can_fuse_residual( const Sell & S, int64_t pos_count );
		// sweep_cluster.cu: one forward + one backward sweep of a small level in ONE launch (a thread-block cluster that
		// separates the colours with its hardware barrier); first_flags / last_flags as the flags of gs_color_step on
		// the first and the last step. Usable when the level has a coded copy and no colour above g_cluster_rows rows.
		bool gs_sweep_cluster_usable( const Sell & S, const std::vector< int64_t > & color_pos, const std::vector< uint64_t > & color_size,
			uint64_t n );
		void gs_sweep_cluster( cudaStream_t st, const Sell & S, const int32_t * rows, const std::vector< int64_t > & color_pos,
			const std::vector< uint64_t > & color_size, uint64_t n, double * z, const double * r, int first_flags, int last_flags,
			const double * src, double * out, double * zero );

		// ---- fused grid transfers (multigrid.hpp:100-104 and :71-81)
		// r_c[p] = 0 + 1*( 1*r[i] + (-1)*(A z)[i] ),  i = rows[p], p in the colour-0 block = injected rows
		void residual_restrict( cudaStream_t st, const Sell & S, const int32_t * rows, int64_t n_coarse, const double * z, const double * r, double * r_c,
			double * zero = nullptr ); // zero: the coarse guess, cleared by the same threads (multigrid.hpp:104)
		// z[i] = 1*z[i] + 1*(0 + 1*z_c[p]) at the injected rows
		void prolong_add( cudaStream_t st, const int32_t * rows, int64_t n_coarse, double * z, const double * z_c );

		// ---- the same entry points on the dictionary-coded copy (packed.cu); S.packed must be usable
		void spmv_packed( cudaStream_t st, const Sell & S, const double * x, double * y, const int32_t * members,
			int64_t count, double * dot_partials, double * dot_out );
		void gs_color_step_packed( cudaStream_t st, const Sell & S, const int32_t * rows, int64_t pos_begin,
			int64_t pos_count, double * z, const double * r, int flags, const double * src, double * out, double * zero,
			const int32_t * pos_list, const uint8_t * skip );
		void residual_restrict_packed( cudaStream_t st, const Sell & S, const int32_t * rows, int64_t n_coarse,
			const double * z, const double * r, double * r_c, double * zero );

		// ---- tile.cu: shared-memory-staged kernels for matrices on a 3D box (BoxTile, common.hpp)
		// the colours (2 pair, 2 pair + 1) of a stencil level in ONE launch; mode 0: forward order, 1: backward,
		// 2: the turnaround of a symmetric sweep (even, odd, odd, even). flags as gs_color_step, on colour 0 only:
		// bit 0 with mode 0, bit 1 with mode 1. Bit-identical to the colour-by-colour steps.
		bool gs_pair_tile_usable( const BoxTile & T, int64_t pair_rows );
		void gs_pair_tile( cudaStream_t st, int sm_count, const BoxTile & T, const std::vector< int64_t > & color_pos, int pair, int mode,
			double * z, const double * r, int flags, const double * src, double * out, double * zero );

		// ---- plane.cu: a symmetric sweep of a regular box level as three plane phases (even planes: colours 0-3; odd
		// planes: colours 4-7 and 7-4; even planes: colours 3-0), every phase out of place, the vector staged through
		// shared memory by bulk-async copies. kind: 0 = colours 0..3, 1 = 4..7,7..4, 2 = 3..0, 3 = 4..7, 4 = 7..4.
		// own_in / nb_in: where the planes of the phase's parity / their neighbour planes are read from; own_out: where
		// the updated planes go (not own_in); pass (bit 0: plane z+1, bit 1: plane z-1, bit 2: plane z+1 if it is the
		// last of the box): neighbour planes copied through to pass_out. flags / src / out / zero as gs_color_step,
		// bit 0 with kind 0, bit 1 with kind 2. Bit-identical to the colour-by-colour steps.
		bool gs_planes_usable( const BoxTile & T, int64_t rows, int sm_count );
		void gs_planes_prepare(); // function attributes; call outside stream capture
		void gs_planes( cudaStream_t st, int sm_count, const BoxTile & T, int kind, int pass, const double * own_in, const double * nb_in,
			double * own_out, double * pass_out, const double * r, int flags, const double * src, double * out, double * zero,
			double * dot_partials = nullptr ); // flags bit 4: one partial of r'z per block (kinds 1 and 2)
		uint64_t gs_planes_blocks( const BoxTile & T, int kind, int sm_count );
		// times the tile shapes the cost models propose and keeps the fastest in T (z, zs, r: scratch vectors, overwritten)
		void gs_planes_tune( cudaStream_t st, int sm_count, BoxTile & T, double * z, double * zs, double * r );

		// ---- plane_spmv.cu: y = A x of a regular box matrix, x staged through shared memory (every staged value read once
		// per thread); dot_out != nullptr: x'(A x) in a fixed tree (dot_partials: spmv_planes_blocks doubles)
		bool spmv_planes_usable( const BoxTile & T, int64_t rows, int sm_count );
		void spmv_planes_prepare(); // function attributes; call outside stream capture
		uint64_t spmv_planes_blocks( const BoxTile & T, int sm_count );
		void spmv_planes( cudaStream_t st, int sm_count, const BoxTile & T, const double * x, double * y, double * dot_partials, double * dot_out );

		// ---- CG vector updates with device-resident scalars (cg.hpp:116-132)
		// p = 1*z + (rho/rho_prev)*p   (when *iter_counter == 0: p = 1*z + 0*z)
		// hist_rr != nullptr: also hist_rr/pq[it - 1] = the previous iteration's r'r / p'Ap (it > 0)
		void cg_update_p( cudaStream_t st, double * p, const double * z, const double * scalars,
			const unsigned int * iter_counter, uint64_t n, double * hist_rr = nullptr, double * hist_pq = nullptr );
		// alpha = rho/pq; x = 1*x + alpha*p; r = 1*r + (-alpha)*q; rho_prev <- rho, S_ALPHA <- alpha
		// x == nullptr (both shapes): the x update is left to cg_update_x
		// bump != nullptr (both shapes): ++*bump (the iteration counter, with the history written by cg_update_p)
		void cg_update_xr( cudaStream_t st, double * x, double * r, const double * p, const double * q, double * scalars,
			uint64_t n, unsigned int * bump = nullptr );
		// the same plus r'r -> scalars[S_RR] (cg.hpp:132) in the tree-dot shape; partials: dot_tree_blocks doubles
		void cg_update_xr_dot( cudaStream_t st, double * x, double * r, const double * p, const double * q, double * scalars,
			uint64_t n, int sm_count, double * partials, unsigned int * counter, unsigned int * bump = nullptr );
		// x = 1*x + scalars[S_ALPHA]*p unless *iter_counter == 0 (cg.hpp:128 one iteration late, cg.cu lazy x)
		void cg_update_x( cudaStream_t st, double * x, const double * p, const double * scalars, const unsigned int * iter_counter,
			uint64_t n, int sm_count );
		// hist_rr[it] = rr, hist_pq[it] = pq, ++it
		// iteration k-1's bookkeeping inside iteration k (it > 0 only; last: after the final iteration, no increment)
		void cg_record_deferred( cudaStream_t st, const double * scalars, double * hist_rr, double * hist_pq, unsigned int * iter_counter, bool last );
		void cg_record( cudaStream_t st, const double * scalars, double * hist_rr, double * hist_pq,
			unsigned int * iter_counter );

		// ---- setup: 27-point stencil straight into SELL (problem.hpp:90-131), colour row lists
		void stencil_widths( cudaStream_t st, const Decomp & D, const int32_t * rows, int64_t npos, int64_t nslices,
			int32_t * widths );
		void stencil_fill( cudaStream_t st, const Decomp & D, const int32_t * rows, int64_t npos, int64_t nslices,
			const int64_t * slice_off, double * vals, int32_t * cols );
		// rows[pos0 + q] = local index of the q-th owned member of global parity class `color`, -1 beyond `size`
		void color_rows( cudaStream_t st, const Decomp & D, int color, int64_t pos0, int64_t size, int64_t padded,
			int32_t * rows );
		// halo pack: buf[dst[k]] = v[src[k]]
		void halo_pack( cudaStream_t st, const int32_t * src, const int32_t * dst, int64_t count, const double * v,
			double * buf );
		// fine[c] = linear index of (2cx,2cy,2cz) (problem.hpp:189-195)
		void injection_cols( cudaStream_t st, int nx, int ny, int nz, int32_t * fine );
		// widths/cols/vals of a one-entry-per-row SELL from a column list
		void sell_single_entry( cudaStream_t st, const int32_t * col_of_row, int64_t nrows, int64_t nslices,
			double * vals, int32_t * cols );
		// SELL -> row counts / CSR (download path)
		void sell_row_counts( cudaStream_t st, const int64_t * slice_off, const int32_t * cols, int64_t nrows,
			int64_t * counts );
		void sell_to_csr( cudaStream_t st, const int64_t * slice_off, const double * vals, const int32_t * cols,
			int64_t nrows, const int64_t * row_off, int64_t * out_cols, double * out_vals );

	} // namespace kern
} // namespace slabgpu
